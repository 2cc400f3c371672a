"""Multi-GPU orchestration of the MLEM hot path (one process per GPU, torch.distributed).

Two partitions of the work:

* throughput mode — frames are independent reconstructions sharing one plan, so
  each rank runs ctis_mlem_batched on its own frames; there is NO collective on
  the data path (weak scaling).
* latency mode — bands: H = (H_1 ... H_w) (Eq. 3), so
  g_hat = H f = sum over band shards of H_shard f_shard.  Each iteration every rank
  computes its partial g_hat (ctis_forward on a shard plan), one all-reduce(SUM)
  forms the full g_hat (NCCL over NVLink/NVSwitch), then each rank computes
  r = g / g_hat and updates its own bands (ctis_back_update_from_ghat).  This is
  the only exchange the method has.

The functions take the collective as a callable so the orchestration can be
tested on CPU with gloo and a stand-in projector (tests/test_distributed_gloo.py).
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple


def band_partition(w: int, parts: int) -> List[Tuple[int, int]]:
    """Contiguous, balanced band ranges [b0, b1) for `parts` shards (first w % parts get one more)."""
    if parts < 1 or parts > w:
        raise ValueError(f"cannot split {w} bands into {parts} non-empty shards")
    base, extra = divmod(w, parts)
    out, b = [], 0
    for p in range(parts):
        e = b + base + (1 if p < extra else 0)
        out.append((b, e))
        b = e
    return out


def frame_partition(frames: int, parts: int) -> List[Tuple[int, int]]:
    """Contiguous, balanced frame ranges (throughput mode)."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    base, extra = divmod(frames, parts)
    out, b = [], 0
    for p in range(parts):
        e = b + base + (1 if p < extra else 0)
        out.append((b, e))
        b = e
    return out


def mlem_band_sharded(plan, g, f_local, iters: int, all_reduce: Callable, ghat=None, ws=None, stream=None):
    """Latency-mode MLEM on this rank's band shard.

    plan:       a shard plan (Plan(..., band_range=(b0, b1)))
    g:          full measured FPA image (n floats), replicated on every rank
    f_local:    this rank's bands of f (plan.m floats), updated in place
    all_reduce: callable(tensor) summing the tensor over all ranks in place
                (torch.distributed.all_reduce on the NCCL group)
    """
    if ghat is None:
        ghat = g.new_empty(plan.n)
    import contextlib
    # all_reduce (torch.distributed) is ordered against the CURRENT stream: run the whole iteration on
    # `stream` so the collective sees the finished partial g_hat and back_update sees the reduced one
    ctx = contextlib.nullcontext()
    if stream is not None and getattr(g, "is_cuda", False):
        import torch
        ctx = torch.cuda.stream(stream)
    with ctx:
        for _ in range(int(iters)):
            plan.forward(f_local, out=ghat, stream=stream)        # partial H_shard f_shard
            all_reduce(ghat)                                      # g_hat = sum over shards (Eq. 3)
            plan.back_update_from_ghat(g, ghat, f_local, ws=ws, stream=stream)
    return f_local


def make_comm(device: int, group=None):
    """A libctis NCCL communicator over the torch.distributed group: rank 0 creates the unique id,
    the group broadcasts it (the side channel NCCL needs), every rank calls ctis_comm_create."""
    import torch.distributed as dist

    import paper_2006_01573_b200 as ctis
    if not dist.is_initialized():  # a single process: a one-rank communicator, no side channel needed
        return ctis.Comm(1, 0, ctis.comm_unique_id(), device)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [ctis.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return ctis.Comm(world, rank, obj[0], device)


def mlem_band_sharded_nccl(plan, comm, g, f_local, iters: int, ws=None, stream=None):
    """Latency mode with the exchange inside libctis (ctis_mlem_band_sharded): per iteration partial
    forward -> reduce-scatter of g_hat -> ratio on this rank's slice -> all-gather of r -> back update,
    all `iters` iterations replayed as one CUDA graph (NCCL calls captured with the kernels)."""
    return plan.mlem_band_sharded(comm, g, f_local, iters, ws=ws, stream=stream)


def exchange_slices(lo: int, hi: int, n: int, parts: int) -> Tuple[int, int, int]:
    """The exchange layout of ctis_mlem_band_sharded (include/ctis.h): base (16-byte aligned), per-rank
    slice (floats, multiple of 4) covering [lo, hi], and the exchange buffer length in floats."""
    base = lo & ~3
    length = hi + 1 - base
    slice_ = ((length + parts - 1) // parts + 3) & ~3
    floats = (max(n, base + slice_ * parts) + 3) & ~3
    return base, slice_, floats


def mlem_band_sharded_exchange(forward_partial: Callable, ratio_slice: Callable, back_update: Callable, g, f_local,
                               iters: int, lo: int, hi: int, rank: int, parts: int,
                               reduce_scatter: Callable, all_gather: Callable, X):
    """The exchange schedule of ctis_mlem_band_sharded written with pluggable steps and collectives —
    the host-level specification the C implementation follows, exercised on CPU with gloo
    (tests/test_distributed_gloo.py).  X: exchange buffer of exchange_slices(...)[2] elements.

    per iteration: X[base:base+P*S] = 0; X += partial forward; reduce-scatter -> own slice;
    slice <- g_slice (/) slice; all-gather -> r on the whole range; f_local <- back_update(r)."""
    n = g.shape[0]
    base, S, floats = exchange_slices(lo, hi, n, parts)
    assert X.shape[0] >= floats
    s0 = base + rank * S
    cnt = 0 if s0 >= n else min(S, n - s0)
    X.zero_()
    for _ in range(int(iters)):
        X[base:base + S * parts].zero_()
        forward_partial(f_local, X)
        mine = X[s0:s0 + S]
        reduce_scatter(mine, X[base:base + S * parts])
        if cnt:
            ratio_slice(g[s0:s0 + cnt], mine[:cnt])
        all_gather(X[base:base + S * parts], mine)
        back_update(X[:n], f_local)
    return f_local


def mlem_band_sharded_local(plans: Sequence, g, f_locals: Sequence, iters: int):
    """All shards of a latency-mode run on ONE device: the all-reduce is a plain on-device sum.

    Used to test the sharding maths without a cluster (tier T2v)."""
    ghat_parts = [g.new_empty(p.n) for p in plans]
    for _ in range(int(iters)):
        for p, fl, gp in zip(plans, f_locals, ghat_parts):
            p.forward(fl, out=gp)
        total = ghat_parts[0].clone()
        for gp in ghat_parts[1:]:
            total += gp
        for p, fl in zip(plans, f_locals):
            p.back_update_from_ghat(g, total, fl)
    return list(f_locals)


def mlem_frame_sharded(plan, g_frames, f_frames, iters: int, ws=None, stream=None):
    """Throughput mode: this rank's frames [F_local, n] / [F_local, m]; no collective."""
    return plan.mlem(g_frames, f_frames, iters, ws=ws, stream=stream)
