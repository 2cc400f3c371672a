"""Subprocess body of test_gpu_parity.py::test_no_stale_shared_memory_reads (run with CTIS_DEBUG=8:
every projection kernel fills its shared-memory window ring with NaN before it starts, so a read of a
slot the kernel did not load in this launch poisons the result)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ctis_synth as syn  # noqa: E402
import oracle  # noqa: E402
import paper_2006_01573_b200 as ctis  # noqa: E402


def rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


worst = 0.0
cases = [
    (syn.Geometry(33, 17, 6, 70, 45), "any"),      # element-loader kernels, wrapping taps, multi-pass
    (syn.Geometry(128, 32, 5, 200, 33), "any"),    # TMA forward, element-loader back
    (syn.Geometry(64, 48, 7, 160, 120), "nowrap"),  # TMA forward and back
]
for gi, (geom, region) in enumerate(cases):
    taps = syn.random_taps(geom, (2, 13), seed=40 + gi, region=region)
    plan = ctis.Plan.from_geometry(geom, taps)
    f = syn.scene_random(geom, seed=gi, lo=0.1, zero_frac=0.1).astype(np.float32)
    g = oracle.forward(geom, taps, f).astype(np.float32)
    e1 = rel(plan.forward(torch.from_numpy(f.ravel()).cuda()).cpu().numpy(), oracle.forward(geom, taps, f))
    u = np.random.default_rng(gi).uniform(0.5, 1.5, geom.n).astype(np.float32)
    e2 = rel(plan.backproject(torch.from_numpy(u).cuda()).cpu().numpy(), oracle.backproject(geom, taps, u))
    fd = torch.ones(geom.m, device="cuda")
    plan.mlem(torch.from_numpy(g).cuda(), fd, 10)
    e3 = rel(fd.cpu().numpy(), oracle.mlem(geom, taps, g, np.ones(geom.m), 10))
    print(gi, e1, e2, e3)
    worst = max(worst, e1 / 1e-5, e2 / 1e-5, e3 / 1e-3)
if len(sys.argv) > 1 and sys.argv[1] == "solvers":
    # C2 (TMA forward + persistent TMA back) and a wrapping case: MLEM / SMART / monitored MLEM
    cfg = syn.config("C2")
    for geom, taps, ft in [(cfg.geom, syn.paper_taps(cfg), syn.scene_blobs(cfg.geom)),
                           (syn.Geometry(33, 17, 6, 70, 45), syn.random_taps(syn.Geometry(33, 17, 6, 70, 45), (2, 9),
                                                                               seed=77, region="any"),
                            syn.scene_random(syn.Geometry(33, 17, 6, 70, 45), seed=3, lo=0.1))]:
        plan = ctis.Plan.from_geometry(geom, taps)
        g = oracle.forward(geom, taps, ft).astype(np.float32)
        gd = torch.from_numpy(g).cuda()
        fd = torch.ones(geom.m, device="cuda")
        plan.mlem(gd, fd, 30)
        e4 = rel(fd.cpu().numpy(), oracle.mlem(geom, taps, g, np.ones(geom.m), 30))
        fs = torch.ones(geom.m, device="cuda")
        plan.smart(gd, fs, 10)
        e5 = rel(fs.cpu().numpy(), oracle.smart(geom, taps, g, np.ones(geom.m), 10))
        fm = torch.ones(geom.m, device="cuda")
        plan.mlem_monitored(gd, fm, 15, 0.0)
        e6 = rel(fm.cpu().numpy(), oracle.mlem(geom, taps, g, np.ones(geom.m), 15))
        print("solvers", geom, e4, e5, e6)
        worst = max(worst, e4 / 1e-3, e5 / 1e-3, e6 / 1e-3)
print("WORST", worst)
sys.exit(0 if worst <= 1.0 else 1)
