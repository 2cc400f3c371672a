"""Stress: repeat the random-wrapping MLEM case (tests/test_gpu_parity.py::test_mlem_random_wrapping)
with fresh plans, optionally after a C4 run, and report every relative error above 1e-4."""
import gc, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import ctis_synth as syn, oracle
import paper_2006_01573_b200 as ctis
geom = syn.Geometry(33, 17, 6, 70, 45)
taps = syn.random_taps(geom, (2, 9), seed=77, region="any")
ftrue = syn.scene_random(geom, seed=3, lo=0.1, zero_frac=0.1)
g = oracle.forward(geom, taps, ftrue).astype(np.float32)
want = oracle.mlem(geom, taps, g.astype(np.float64), np.ones(geom.m), 30)
def rel(a, b): return float(np.linalg.norm(np.float64(a).ravel() - b.ravel()) / np.linalg.norm(b))
c4 = syn.config("C4")
big = None
bad = 0
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    if rep % 4 == 1:
        big = ctis.Plan.from_geometry(c4.geom, syn.paper_taps(c4))
        gb = big.forward(torch.ones(c4.geom.m, device="cuda"))
        fb = torch.ones(c4.geom.m, device="cuda")
        big.mlem(gb, fb, 5)
    if rep % 4 == 3:
        big = None; gc.collect()
    junk = torch.full((64 << 20,), float("nan"), device="cuda")  # dirty the caching allocator's blocks
    del junk
    plan = ctis.Plan.from_geometry(geom, taps)
    gd = torch.from_numpy(g).cuda()
    fd = torch.ones(geom.m, device="cuda")
    plan.mlem(gd, fd, 30)
    e = rel(fd.cpu().numpy(), want)
    if e > 1e-4:
        bad += 1
        print("rep", rep, "err", e, flush=True)
print("bad", bad)
