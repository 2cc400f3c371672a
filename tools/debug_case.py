import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import ctis_synth as syn
import paper_2006_01573_b200 as ctis
geom = syn.Geometry(128, 32, 5, 200, 33)
taps = syn.random_taps(geom, (1, 13), seed=15, region="any")
print("taps per band", np.diff(taps.ptr))
plan = ctis.Plan.from_geometry(geom, taps)
f = torch.rand(geom.m, device="cuda")
g = plan.forward(f); torch.cuda.synchronize(); print("fwd ok")
z = plan.backproject(torch.rand(geom.n, device="cuda")); torch.cuda.synchronize(); print("back ok")
