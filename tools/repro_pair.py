"""Repro: tests C4_full_run_invariants followed by mlem_random_wrapping, repeated in one process."""
import gc, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import ctis_synth as syn, oracle
import paper_2006_01573_b200 as ctis
mode = sys.argv[1] if len(sys.argv) > 1 else "graph"
geom = syn.Geometry(33, 17, 6, 70, 45)
taps = syn.random_taps(geom, (2, 9), seed=77, region="any")
ftrue = syn.scene_random(geom, seed=3, lo=0.1, zero_frac=0.1)
g = oracle.forward(geom, taps, ftrue).astype(np.float32)
want = oracle.mlem(geom, taps, g.astype(np.float64), np.ones(geom.m), 30)
def rel(a, b): return float(np.linalg.norm(np.float64(a).ravel() - b.ravel()) / np.linalg.norm(b))
cfg = syn.config("C4")
bad = 0
for rep in range(int(os.environ.get("REPS", "8"))):
    if mode != "nobig":
        plan = ctis.Plan.from_geometry(cfg.geom, syn.paper_taps(cfg))
        gb = plan.forward(torch.from_numpy(syn.scene_blobs(cfg.geom).reshape(-1)).cuda())
        f = torch.ones(cfg.geom.m, device="cuda")
        plan.mlem(gb, f, cfg.K)
        gh = plan.forward(f)
        assert bool((f >= 0).all())
        del plan, gb, f, gh
        if mode == "gc": gc.collect()
    p2 = ctis.Plan.from_geometry(geom, taps)
    if mode == "nograph": p2.set_option(2, 0)
    gd = torch.from_numpy(g).cuda()
    fd = torch.ones(geom.m, device="cuda")
    p2.mlem(gd, fd, 30)
    e = rel(fd.cpu().numpy(), want)
    # per-iteration check: run 1 iteration at a time on a fresh f
    print(mode, "rep", rep, "err %.3e" % e, flush=True)
    bad += e > 1e-4
    del p2
print(mode, "bad", bad)
