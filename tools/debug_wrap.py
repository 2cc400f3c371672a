"""Debug: MLEM on the random wrapping case (33,17,6,70,45), repeated, errors per iteration count."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import ctis_synth as syn, oracle
import paper_2006_01573_b200 as ctis
geom = syn.Geometry(33, 17, 6, 70, 45)
taps = syn.random_taps(geom, (2, 9), seed=77, region="any")
ftrue = syn.scene_random(geom, seed=3, lo=0.1, zero_frac=0.1)
g = oracle.forward(geom, taps, ftrue).astype(np.float32)
def rel(a, b): return float(np.linalg.norm(np.float64(a).ravel() - b.ravel()) / np.linalg.norm(b))
plan = ctis.Plan.from_geometry(geom, taps)
f = ftrue.reshape(-1).astype(np.float32)
for rep in range(3):
    print("fwd", rel(plan.forward(torch.from_numpy(f).cuda()).cpu().numpy(), oracle.forward(geom, taps, f)),
          "back", rel(plan.backproject(torch.from_numpy(g).cuda()).cpu().numpy(), oracle.backproject(geom, taps, g)))
for K in (1, 2, 5, 10, 30):
    want = oracle.mlem(geom, taps, g.astype(np.float64), np.ones(geom.m), K)
    errs = []
    for rep in range(3):
        fd = torch.ones(geom.m, device="cuda")
        plan.mlem(torch.from_numpy(g).cuda(), fd, K)
        errs.append(rel(fd.cpu().numpy(), want))
    print("K", K, errs)
