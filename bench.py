#!/usr/bin/env python
"""Benchmark of the CTIS MLEM hot path on B200 (BASELINE.json metric).

Metric: MLEM iterations/s (and reconstructions/s of K = 100 iterations).
A "step" is one full reconstruction: ctis_mlem(K = 100) from f0 = ones over one
synthetic measurement g (all §8(a) rows: forward, ratio, back-projection,
update, iteration control).  Default workload: C4 (256x256 field stop, w = 100,
2048x2048 FPA, 7x7 orders) — the largest paper-shaped datacube that BASELINE's
target names.  N > 1 (torchrun): throughput mode, each rank reconstructs its own
frame, no collective (weak scaling); --mode bands runs the latency mode
(band-sharded with an NCCL all-reduce of g_hat per iteration).

--impl reference times the CPU oracle (oracle/, the reference arm of this tier)
on the same workload, one MLEM iteration per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import ctis_synth as syn  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
SM_COUNT = 148
FP32_LANES_PER_SM = 128


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C4", choices=list(syn.CONFIGS))
    ap.add_argument("--mode", default="frames", choices=["frames", "bands"])
    ap.add_argument("--iters", type=int, default=None, help="MLEM iterations per reconstruction (default: config K)")
    ap.add_argument("--frames", type=int, default=None, help="frames per rank (default: 1; C5: 256/N)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "fused"],
                    help="--mode bands: NCCL reduce-scatter/all-gather or the fused NVLink exchange kernel")
    ap.add_argument("--extra", default="C5,C3,T1w75",
                    help="N = 1: also time these workloads (same rules) under 'extra_workloads' ('' = none)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# PAPER.md Table 1, WBH + EM + P4000: seconds / K at K = 25 (w = 75: 3.8 s, 24: 1.2 s, 3: 0.2 s)
PAPER_T1_MS = {"T1w75": 3800.0 / 25, "T1w24": 1200.0 / 25, "T1w3": 200.0 / 25}


def time_extra(name, dev, steps=2, warmup=1):
    """One secondary workload measured like the headline (f0 = 1 reset and 512 MB L2 flush outside the
    CUDA events, K iterations per reconstruction, all frames of the config in one batched call)."""
    import torch

    import paper_2006_01573_b200 as ctis
    cfg = syn.config(name)
    geom = cfg.geom
    taps = syn.paper_taps(cfg)
    plan = ctis.Plan.from_geometry(geom, taps, device=dev.index or 0)
    plan.set_option(ctis.OPT_VALIDATE_DATA, 0)
    F = cfg.frames
    scenes = torch.from_numpy(np.stack([syn.frame_scene(geom, i).reshape(-1) for i in range(F)]) if F > 1
                              else syn.scene_blobs(geom).reshape(1, -1)).to(dev)
    g = plan.forward(scenes.view(F, geom.m) if F > 1 else scenes.view(-1))
    del scenes
    f = torch.ones((F, geom.m) if F > 1 else (geom.m,), dtype=torch.float32, device=dev)
    ws = plan.workspace(F)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        f.fill_(1.0)
        plan.mlem(g, f, cfg.K, ws=ws)
    launches = plan.last_launch_count()
    ms = []
    for _ in range(steps):
        f.fill_(1.0)
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.mlem(g, f, cfg.K, ws=ws)
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    t = sum(ms) / len(ms)
    ctx = None
    if name in PAPER_T1_MS:  # the paper's own Table 1 row for this geometry (other hardware: context only)
        ctx = {"paper_ms_per_iteration_P4000": PAPER_T1_MS[name],
               "source": "PAPER.md P:245-262 Table 1, WBH + EM on a Quadro P4000, fp32 (t/K); the paper's "
                         "measured system matrix is not available, taps follow ctis_synth's recipe"}
    return {"value": F * cfg.K / (t / 1e3), "unit": "iterations/s", "recon_per_s": F / (t / 1e3),
            "paper_context": ctx,
            "ms_per_step": t, "steps": steps, "warmup": warmup, "frames": F, "iterations_per_step": cfg.K,
            "us_per_frame_iteration": t * 1e3 / (F * cfg.K), "gpu_launches_per_step": launches,
            "config": {"workload": name, "a": geom.a, "alpha": geom.alpha, "w": geom.w, "gamma": geom.gamma,
                       "xi": geom.xi, "taps_per_band": int(taps.ptr[1])}}


def load_peaks():
    try:
        with open(PEAKS_PATH) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), float(pk.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, 1965.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic(cfg, taps):
    """Per-iteration algorithmic work: bytes and FLOPs of each kernel."""
    g = cfg.geom
    m, n = g.m, g.n
    mT = int(taps.ptr[-1]) * g.ell            # sum over bands of T_lam * l = incidences per projection
    return {
        "forward": {"bytes": 4 * m + 4 * n, "flops": 2 * mT},          # read f, write g_hat
        "back": {"bytes": 4 * n + 8 * m, "flops": 2 * mT + 2 * m},     # read r, read+write f
        "iteration": {"bytes": 12 * m + 12 * n, "flops": 4 * mT + n + 3 * m},
        "incidences": mT,
    }


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_oracle_iterations(cfg, taps, g, iters, threads=1):
    """Time `iters` MLEM iterations of the fp64 oracle as it stands (oracle/; OpenMP over `threads`)."""
    import oracle
    f0 = np.ones(cfg.geom.m)
    with oracle.threads(threads):
        t0 = time.perf_counter()
        oracle.mlem(cfg.geom, taps, g, f0, iters)
        return time.perf_counter() - t0


def cpu_baseline(cfg, taps, g, K, workload, budget_s=12.0):
    """The oracle on the host's cores (rank 0, N = 1): a bounded sample of the benchmarked workload on
    every core, the same on one core, and full-K reconstructions of the small configs (tiny, C2)."""
    import oracle
    cores = host_cores()
    t1 = cpu_oracle_iterations(cfg, taps, g, 1, cores)              # probe (includes h = H^T 1)
    iters = int(max(1, min(K, budget_s / max(t1, 1e-3))))
    t = cpu_oracle_iterations(cfg, taps, g, iters, cores)
    t_single = cpu_oracle_iterations(cfg, taps, g, 1, 1)
    small = {}
    for name in ("tiny", "C2"):
        c = syn.config(name)
        tp = syn.paper_taps(c)
        gs = oracle.forward(c.geom, tp, syn.scene_blobs(c.geom)).astype(np.float32).astype(np.float64)
        small[name] = {"K": c.K, "s_per_recon_1_thread": cpu_oracle_iterations(c, tp, gs, c.K, 1),
                       f"s_per_recon_{cores}_threads": cpu_oracle_iterations(c, tp, gs, c.K, cores)}
    return {"value": iters / t, "unit": "iterations/s", "cores": cores, "kind": "oracle",
            "cpu": cpu_model(),
            "sample": f"{workload}: {iters} MLEM iterations (of K={K}) on {cores} threads, {t:.1f} s; "
                      f"recon/s = value/{K} (extrapolated from the sample)",
            "single_thread": {"value": 1.0 / t_single, "unit": "iterations/s", "sample": f"{workload}: 1 iteration"},
            "full_K_small_configs": small}


def run_reference(args):
    """--impl reference: the fp64 CPU oracle (oracle/) as it stands, 1 MLEM iteration per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    cfg = syn.config(args.workload)
    geom = cfg.geom
    taps = syn.paper_taps(cfg)
    g = oracle.forward(geom, taps, syn.scene_blobs(geom)).astype(np.float32).astype(np.float64)
    cores = host_cores()
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_oracle_iterations(cfg, taps, g, 1, cores)
    times = [cpu_oracle_iterations(cfg, taps, g, 1, cores) for _ in range(args.steps)]
    total = sum(times)
    value = args.steps / total
    line = {
        "impl": "reference", "metric": "MLEM iterations/s", "value": value, "unit": "iterations/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "a": geom.a, "alpha": geom.alpha, "w": geom.w, "gamma": geom.gamma,
                   "xi": geom.xi, "taps_per_band": int(taps.ptr[1]), "iterations_per_step": 1,
                   "recon_iterations": cfg.K, "l2": "inputs resident in host RAM; CPU run"},
        "recon_per_s": value / cfg.K,
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": cores, "kind": "oracle", "cpu": cpu_model(),
                         "sample": f"{args.workload}: {args.steps} single MLEM iterations (of K={cfg.K}), 1 frame, "
                                   f"{cores} OpenMP threads"},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def self_launch(args) -> int:
    """`python bench.py --gpus N` (N > 1) outside torchrun: start N ranks with torch.distributed.run on
    127.0.0.1 so that the line reports what N GPUs did (never a silent single-GPU run)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2006_01573_b200 as ctis
    from paper_2006_01573_b200 import distributed as dmod

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        return 2
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)

    cfg = syn.config(args.workload)
    geom = cfg.geom
    K = cfg.K if args.iters is None else args.iters
    taps = syn.paper_taps(cfg)
    mode = args.mode
    if args.frames is not None:
        frames = args.frames
    elif cfg.frames > 1:
        frames = dmod.frame_partition(cfg.frames, world)[rank][1] - dmod.frame_partition(cfg.frames, world)[rank][0]
    else:
        frames = 1
    if mode == "bands":
        frames = 1
        b0, b1 = dmod.band_partition(geom.w, world)[rank]
        plan = ctis.Plan.from_geometry(geom, taps, device=local, band_range=(b0, b1))
        full = None
    else:
        b0, b1 = 0, geom.w
        plan = ctis.Plan.from_geometry(geom, taps, device=local)
    plan.set_option(ctis.OPT_VALIDATE_DATA, 0)

    # ---- synthetic measurement g = H f_true per frame (our forward; bench is not a parity check)
    fullplan = plan if mode == "frames" else ctis.Plan.from_geometry(geom, taps, device=local)
    fidx0 = rank * frames if mode == "frames" else 0
    scenes = torch.from_numpy(np.stack([syn.frame_scene(geom, fidx0 + i).reshape(-1) if frames > 1 or cfg.frames > 1
                                        else syn.scene_blobs(geom).reshape(-1) for i in range(frames)])).to(dev)
    g = fullplan.forward(scenes.view(frames, geom.m) if frames > 1 else scenes.view(-1))
    g = g.view(frames, geom.n) if frames > 1 else g.view(-1)
    if mode == "bands":
        del fullplan
    torch.cuda.synchronize()

    m_loc = plan.m
    # one f buffer, reset to f0 = 1 before every step (outside the events): ctis_mlem caches its CUDA
    # graph per (g, f, ws) pointers, so a fresh buffer per step would put a host-side graph capture
    # inside the timed region
    fbuf = torch.ones((frames, m_loc) if frames > 1 else (m_loc,), dtype=torch.float32, device=dev)
    fbufs = [fbuf] * (args.warmup + args.steps)
    ws = plan.workspace(frames)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)     # > 126 MB L2
    stream = torch.cuda.current_stream()

    comm = ws_sh = None
    if mode == "bands":
        comm = dmod.make_comm(local)                      # NCCL communicator owned by libctis
        ws_sh = plan.band_sharded_workspace(comm)
        plan.set_option(ctis.OPT_EXCHANGE, 1 if args.exchange == "fused" else 0)

    def one_step(fb):
        if mode == "bands":
            # partial forward -> reduce-scatter -> slice ratio -> all-gather -> back update, K times, one graph
            dmod.mlem_band_sharded_nccl(plan, comm, g, fb, K, ws=ws_sh)
        else:
            plan.mlem(g, fb, K, ws=ws)

    for i in range(args.warmup):
        flush.zero_()
        fbufs[i].fill_(1.0)
        one_step(fbufs[i])
    launches_per_step = plan.last_launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    sampler = ClockSampler(local)
    sampler.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for i in range(args.steps):
        fbufs[args.warmup + i].fill_(1.0)                 # f0 = 1 (outside events)
        flush.zero_()                                     # L2 flush between timed steps (outside events)
        evs[i][0].record(stream)
        one_step(fbufs[args.warmup + i])
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    recon_total = args.steps * (frames * world if mode == "frames" else 1)
    iters_total = recon_total * K
    value = iters_total / (total_ms / 1e3)
    launches = args.steps * launches_per_step

    # ---- per-kernel live timing for the roofline (CUDA events on the launching stream)
    alg = algorithmic(cfg, taps)
    hbm_peak, sm_max, peak_src = load_peaks()
    fp32_peak = SM_COUNT * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
    kern = {}
    if rank == 0:
        reps = 20
        fk = fbufs[-1].view(-1)[:m_loc] if frames == 1 else fbufs[-1][0]
        half = (geom.n * frames + 3) // 4 * 4                 # workspace = [g_hat accumulator | r]
        rk = ws.view(-1)[half:half + geom.n]
        scratch = torch.zeros(geom.n, dtype=torch.float32, device=dev)
        fu = fbufs[0].view(-1)[:m_loc]
        for name, fn in (("forward", lambda: plan.forward_accumulate(fk, scratch)),
                         ("back_update", lambda: plan.back_update(rk, fu))):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            # `reps` back-to-back launches between two events on the launching stream: the host runs
            # ahead (per-launch tensor-map encoding overlaps the previous launch), so the average is the
            # kernel's device duration
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                fn()
            b.record(stream)
            torch.cuda.synchronize()
            kern[name] = a.elapsed_time(b) / reps * 1e-3
    line = None
    if rank == 0:
        frac_w = (b1 - b0) / geom.w
        work = {"forward": (alg["forward"]["bytes"], alg["forward"]["flops"] * frac_w),
                "back_update": (alg["back"]["bytes"], alg["back"]["flops"] * frac_w)}
        dom = max(kern, key=kern.get)
        t_dom = kern[dom]
        dom_bytes, dom_flops = work[dom]
        t_hbm, t_alu = dom_bytes / (hbm_peak * 1e9), dom_flops / (fp32_peak * 1e12)
        if t_hbm >= t_alu:
            roof = {"bound": "hbm", "achieved": dom_bytes / t_dom / 1e9, "peak": hbm_peak, "unit": "GB/s"}
        else:
            roof = {"bound": "alu", "achieved": dom_flops / t_dom / 1e12, "peak": fp32_peak, "unit": "TFLOP/s"}
        roof["frac"] = roof["achieved"] / roof["peak"]
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get(args.workload, {}).get(dom)
            except Exception:
                traffic = None
        it_ms = total_ms / (args.steps * K)
        t_it_roof = max(alg["iteration"]["bytes"] / (hbm_peak * 1e9), alg["iteration"]["flops"] / (fp32_peak * 1e12))
        roof.update({
            "kernel": dom, "traffic": traffic, "peak_source": peak_src,
            "alg_bytes_per_launch": dom_bytes, "alg_flops_per_launch": dom_flops,
            "fp32_tflops_achieved": dom_flops / t_dom / 1e12, "fp32_peak_tflops": fp32_peak,
            "hbm_gbs_achieved": dom_bytes / t_dom / 1e9,
            "smem_operand_frac": (alg["incidences"] * frac_w * 4 / t_dom) / (SM_COUNT * 128 * sm_max * 1e6),
            "iteration_roof_us": t_it_roof * 1e6,
            "iteration_frac": (t_it_roof / (it_ms * 1e-3)) if mode == "frames" and frames == 1 else None})
        line = {
            "metric": "MLEM iterations/s", "value": value, "unit": "iterations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak" if mode == "frames" else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload, "mode": mode, "a": geom.a, "alpha": geom.alpha, "w": geom.w,
                       "gamma": geom.gamma, "xi": geom.xi, "taps_per_band": int(taps.ptr[1]),
                       "iterations_per_step": K, "frames_per_rank": frames,
                       "exchange": args.exchange if mode == "bands" else None, "parallelism":
                       f"{'frames' if mode == 'frames' else 'bands'}{world}",
                       "l2": "flushed between timed steps (512 MB write, outside the step events)"},
            "recon_per_s": recon_total / (total_ms / 1e3),
            "ms_per_iteration": it_ms,
            "kernels_ms": {k: v * 1e3 for k, v in kern.items()},
            "roofline": roof,
            "clocks": clocks,
            "gpu_launches": launches,
        }

    # ---- end to end through the public API with HOST buffers (ctis_mlem_host)
    if not args.no_e2e and mode == "frames":
        gh = g.cpu().pin_memory().contiguous()
        fh = [torch.ones(g.shape[:-1] + (m_loc,), dtype=torch.float32).pin_memory() for _ in range(2)]
        plan.mlem_host_ptr(gh.data_ptr(), fh[0].data_ptr(), frames, K)          # warm-up (allocations)
        if world > 1:
            dist.barrier()
        e2e_ms = 0.0
        for i in range(args.steps):
            fh[1].fill_(1.0)
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            plan.mlem_host_ptr(gh.data_ptr(), fh[1].data_ptr(), frames, K)
            e2e_ms += (time.perf_counter() - t0) * 1e3
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        if line is not None:
            line["e2e"] = {"value": iters_total / (e2e_ms / 1e3), "unit": "iterations/s",
                           "h2d_bytes_per_step": 4 * frames * (geom.n + m_loc),
                           "d2h_bytes_per_step": 4 * frames * m_loc,
                           "api": "ctis_mlem_host (pinned host buffers, wall clock incl. copies)"}

    # ---- CPU oracle beside it (rank 0, N = 1 only, bounded sample)
    if line is not None and world == 1 and not args.no_cpu_baseline:
        gnp = (g if frames == 1 else g[0]).double().cpu().numpy()
        line["cpu_baseline"] = cpu_baseline(cfg, taps, gnp, K, args.workload)
    if line is not None and world == 1 and mode == "frames" and args.extra:
        import torch as _t
        extra = {}
        for name in [x for x in args.extra.split(",") if x and x != args.workload]:
            try:
                extra[name] = time_extra(name, dev)
            except Exception as exc:  # report, never hide the headline line
                extra[name] = {"error": str(exc)[:200]}
            _t.cuda.empty_cache()
        line["extra_workloads"] = extra
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
