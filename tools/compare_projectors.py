"""Tap projector vs the paper's Fourier (WBH) route on B200: MLEM ms per iteration at the paper-shaped
configs (CUDA events around a captured 10-iteration ctis_mlem graph, after warm-up).  Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ctis_synth as syn  # noqa: E402
import paper_2006_01573_b200 as ctis  # noqa: E402

K = 10
out = {}
for name in sys.argv[1:] or ["C2", "C3", "C4"]:
    cfg = syn.config(name)
    plan = ctis.Plan.from_geometry(cfg.geom, syn.paper_taps(cfg))
    plan.set_option(ctis.OPT_VALIDATE_DATA, 0)
    g = plan.forward(torch.from_numpy(syn.scene_blobs(cfg.geom).reshape(-1)).cuda())
    row = {}
    for proj, label in ((0, "taps"), (1, "fft")):
        plan.set_option(ctis.OPT_PROJECTOR, proj)
        f = torch.ones(cfg.geom.m, device="cuda")
        for _ in range(2):
            plan.mlem(g, f, K)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            f.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            plan.mlem(g, f, K)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / K)
        row[label + "_ms_per_iteration"] = sorted(ts)[len(ts) // 2]
    row["fft_over_taps"] = row["fft_ms_per_iteration"] / row["taps_ms_per_iteration"]
    out[name] = row
    print(name, row, flush=True)
print(json.dumps(out))
