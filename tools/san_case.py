"""Small MLEM on the element-loader (non-TMA) path for compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import ctis_synth as syn
import paper_2006_01573_b200 as ctis
geom = syn.Geometry(33, 17, 6, 70, 45)
taps = syn.random_taps(geom, (2, 9), seed=77, region="any")
plan = ctis.Plan.from_geometry(geom, taps)
plan.set_option = getattr(plan, "set_option", None)
g = plan.forward(torch.rand(geom.m, device="cuda") + 0.1)
f = torch.ones(geom.m, device="cuda")
plan.mlem(g, f, 2)
torch.cuda.synchronize()
print("ok", float(f.sum()))
