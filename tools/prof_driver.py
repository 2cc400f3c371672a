"""Small driver for ncu captures: builds a plan and launches forward_ratio / back_update a few times."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ctis_synth as syn  # noqa: E402
import paper_2006_01573_b200 as ctis  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C4")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
cfg = syn.config(args.workload)
geom = cfg.geom
taps = syn.paper_taps(cfg)
plan = ctis.Plan.from_geometry(geom, taps)
dev = torch.device("cuda:0")
ftrue = torch.from_numpy(syn.scene_blobs(geom).reshape(-1)).to(dev)
g = plan.forward(ftrue)
f = torch.ones(geom.m, device=dev)
r = torch.empty(geom.n, device=dev)
for _ in range(args.reps):
    plan.forward_ratio(f, g, r)
    plan.back_update(r, f)
torch.cuda.synchronize()
print("ok", float(f.sum()))
