"""C5 (256 C3 frames, K = 100): one batched ctis_mlem call vs sub-batches of B frames (L2-sized)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import ctis_synth as syn
import paper_2006_01573_b200 as ctis
cfg = syn.config("C5")
geom = cfg.geom
plan = ctis.Plan.from_geometry(geom, syn.paper_taps(cfg))
plan.set_option(ctis.OPT_VALIDATE_DATA, 0)
F = cfg.frames
scenes = torch.from_numpy(np.stack([syn.frame_scene(geom, i).reshape(-1) for i in range(F)])).cuda()
g = plan.forward(scenes.view(F, geom.m)).view(F, geom.n)
del scenes
f = torch.ones(F, geom.m, device="cuda")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for B in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "256,32,16,8,4").split(",")]:
    ws = plan.workspace(B)
    def run():
        for s in range(0, F, B):
            plan.mlem(g[s:s + B], f[s:s + B], K, ws=ws)
    f.fill_(1.0); run(); torch.cuda.synchronize()
    f.fill_(1.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); run(); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"B={B}: {ms:.1f} ms per C5 reconstruction set, {F / (ms / 1e3):.1f} recon/s, {ms * 1e3 / (F * K):.2f} us/frame-iter", flush=True)
