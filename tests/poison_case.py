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
print("WORST", worst)
sys.exit(0 if worst <= 1.0 else 1)
