"""Bench-style step timing diagnostics: one K-iteration ctis_mlem per step between CUDA events, with and
without the L2 flush (and with the GPU kept busy while the host enqueues), plus the host time of the call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ctis_synth as syn
import paper_2006_01573_b200 as ctis
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = syn.config(name)
plan = ctis.Plan.from_geometry(cfg.geom, syn.paper_taps(cfg))
plan.set_option(ctis.OPT_VALIDATE_DATA, 0)
g = plan.forward(torch.from_numpy(syn.scene_blobs(cfg.geom).reshape(-1)).cuda())
f = torch.ones(cfg.geom.m, device="cuda")
ws = plan.workspace(1)
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
s = torch.cuda.current_stream()
for mode in ("noflush", "flush", "flush+sleep"):
    res, host = [], []
    for i in range(6):
        f.fill_(1.0)
        if mode != "noflush":
            flush.zero_()
        if mode == "flush+sleep":
            torch.cuda._sleep(2_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        t0 = time.perf_counter()
        plan.mlem(g, f, cfg.K, ws=ws)
        host.append((time.perf_counter() - t0) * 1e6)
        b.record(s)
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) * 1e3 / cfg.K)
    print(name, mode, "us/iter", " ".join(f"{x:.1f}" for x in res[2:]), "host us/call", " ".join(f"{x:.0f}" for x in host[2:]), flush=True)
