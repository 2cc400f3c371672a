"""Time the forward / back_update kernels in isolation (CUDA events), for quick experiments."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ctis_synth as syn
import paper_2006_01573_b200 as ctis
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = syn.config(name)
plan = ctis.Plan.from_geometry(cfg.geom, syn.paper_taps(cfg))
f = torch.from_numpy(syn.scene_blobs(cfg.geom).reshape(-1)).cuda()
g = torch.zeros(cfg.geom.n, device="cuda")
r = torch.rand(cfg.geom.n, device="cuda") + 0.5
fu = torch.ones(cfg.geom.m, device="cuda")
out = {}
for nm, fn in (("forward", lambda: plan.forward_accumulate(f, g)), ("back", lambda: plan.back_update(r, fu))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    # 30 back-to-back launches between two events: the host runs ahead, so the average is device time
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(30): fn()
    b.record()
    torch.cuda.synchronize()
    out[nm] = a.elapsed_time(b) / 30 * 1e3
print(name, "dbg=%s" % os.environ.get("CTIS_DEBUG", "0"), " ".join(f"{k}={v:.1f}us" for k, v in out.items()))
