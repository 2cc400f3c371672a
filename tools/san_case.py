"""Workloads for compute-sanitizer runs (memcheck / racecheck / synccheck) of the projection kernels.

Cases (argv[1], default "bench"):
  bench    the kernels the benchmark runs: tiny and C2 (TMA forward ctis_fwd_g2_*_t, back ctis_back2/4_*_t),
           and 8 C3 frames in one batched launch (persistent CTAs walking many work items);
  loader   the element-loader kernels (wrapping taps: ctis_fwd_g1_*_s, ctis_back_b*_s).
Direct launches (no CUDA graph) so the tools see every kernel; 2 MLEM iterations each.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ctis_synth as syn  # noqa: E402
import paper_2006_01573_b200 as ctis  # noqa: E402


def run(geom, taps, frames=1, iters=2, solvers=False):
    plan = ctis.Plan.from_geometry(geom, taps)
    plan.set_option(ctis.OPT_USE_GRAPH, 0)
    print("plan", geom, plan.info(), flush=True)
    scenes = torch.from_numpy(np.stack([syn.frame_scene(geom, i).reshape(-1) for i in range(frames)])).cuda()
    g = plan.forward(scenes.view(frames, geom.m) if frames > 1 else scenes.view(-1))
    f = torch.ones((frames, geom.m) if frames > 1 else (geom.m,), device="cuda")
    plan.mlem(g, f, iters)
    if solvers and frames == 1:
        fs = torch.ones(geom.m, device="cuda")
        plan.smart(g, fs, iters)
        fm = torch.ones(geom.m, device="cuda")
        plan.mlem_monitored(g, fm, iters, 0.0)
    torch.cuda.synchronize()
    print("ok", geom, frames, float(f.sum()), flush=True)


case = sys.argv[1] if len(sys.argv) > 1 else "bench"
if case == "loader":  # odd field stops otherwise take the repacked TMA forward (which racecheck cannot run)
    os.environ["CTIS_FWD_REPACK"] = "0"
if case == "bench":
    for name in ("tiny", "C2"):
        cfg = syn.config(name)
        run(cfg.geom, syn.paper_taps(cfg), solvers=True)
    cfg = syn.config("C3")
    run(cfg.geom, syn.paper_taps(cfg), frames=8)
else:
    geom = syn.Geometry(33, 17, 6, 70, 45)
    run(geom, syn.random_taps(geom, (2, 9), seed=77, region="any"), solvers=True)
print("done")
