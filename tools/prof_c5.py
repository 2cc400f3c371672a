"""ncu driver for the snapshot-video layout: a C3 plan, 32 frames in one batched MLEM iteration
(throughput layout: classic forward, NB = 12 back)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import ctis_synth as syn
import paper_2006_01573_b200 as ctis
F = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cfg = syn.config("C3")
geom = cfg.geom
plan = ctis.Plan.from_geometry(geom, syn.paper_taps(cfg))
plan.set_option(ctis.OPT_USE_GRAPH, 0)
scenes = torch.from_numpy(np.stack([syn.frame_scene(geom, i).reshape(-1) for i in range(F)])).cuda()
g = plan.forward(scenes.view(F, geom.m))
f = torch.ones(F, geom.m, device="cuda")
ws = plan.workspace(F)
for _ in range(3):
    plan.mlem(g, f, 1, ws=ws)
torch.cuda.synchronize()
print("ok", plan.info())
