"""Time the forward / back_update kernels in isolation (CUDA events), for quick experiments.
usage: kernel_times.py [config] [frames]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import ctis_synth as syn
import paper_2006_01573_b200 as ctis
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
F = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = syn.config(name)
geom = cfg.geom
plan = ctis.Plan.from_geometry(geom, syn.paper_taps(cfg))
scenes = np.stack([syn.frame_scene(geom, i).reshape(-1) for i in range(F)]) if F > 1 else syn.scene_blobs(geom).reshape(1, -1)
f = torch.from_numpy(scenes).cuda().view(F, geom.m) if F > 1 else torch.from_numpy(scenes).cuda().view(-1)
g = torch.zeros((F, geom.n) if F > 1 else (geom.n,), device="cuda")
r = torch.rand((F, geom.n) if F > 1 else (geom.n,), device="cuda") + 0.5
fu = torch.ones((F, geom.m) if F > 1 else (geom.m,), device="cuda")
ws = plan.workspace(F)
out = {}
def back():
    if F == 1:
        plan.back_update(r, fu)
    else:   # batched back update through the batched MLEM's back half is not exposed: time mlem K=1 instead
        plan.mlem(r, fu, 1, ws=ws)
for nm, fn in (("forward", lambda: plan.forward_accumulate(f, g)), ("back" if F == 1 else "mlem1", back)):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    # back-to-back launches between two events: the host runs ahead, so the average is device time
    reps = 30 if F == 1 else 5
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record()
    torch.cuda.synchronize()
    out[nm] = a.elapsed_time(b) / reps * 1e3
info = plan.info()
print(name, f"F={F}", "dbg=%s" % os.environ.get("CTIS_DEBUG", "0"), " ".join(f"{k}={v:.1f}us" for k, v in out.items()),
      " ".join(f"{k}/frame={v / F:.2f}us" for k, v in out.items()) if F > 1 else "", info)
