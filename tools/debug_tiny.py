import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import ctis_synth as syn
import paper_2006_01573_b200 as ctis
name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
which = sys.argv[2] if len(sys.argv) > 2 else "both"
cfg = syn.config(name)
plan = ctis.Plan.from_geometry(cfg.geom, syn.paper_taps(cfg))
f = torch.from_numpy(syn.scene_blobs(cfg.geom).reshape(-1)).cuda()
if which in ("fwd", "both"):
    g = plan.forward(f); torch.cuda.synchronize(); print("forward ok", float(g.sum()))
if which in ("back", "both"):
    r = torch.rand(cfg.geom.n, device="cuda")
    z = plan.backproject(r); torch.cuda.synchronize(); print("back ok", float(z.sum()))
