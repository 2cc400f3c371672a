"""N > 1 orchestration on CPU: world_size 2 over gloo with a stand-in projector.

The stand-in ("OracleShard") computes the shard's partial forward and its
back-update with the fp64 oracle, so the test exercises exactly the host logic
of paper_2006_01573_b200.distributed (band partition, per-iteration all-reduce
of the partial g_hat, ratio + update on each shard; frame partition) and checks
it against a single-process oracle MLEM.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ctis_synth as syn


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleShard:
    """Host stand-in with the Plan interface used by mlem_band_sharded (test-only)."""

    def __init__(self, geom, taps, b0, b1):
        import oracle
        self.o = oracle
        self.geom = syn.Geometry(geom.a, geom.alpha, b1 - b0, geom.gamma, geom.xi)
        ptr = taps.ptr[b0:b1 + 1] - taps.ptr[b0]
        s, e = int(taps.ptr[b0]), int(taps.ptr[b1])
        self.taps = syn.Taps(ptr, taps.offset[s:e], taps.weight[s:e])
        self.n, self.m = geom.n, self.geom.m
        self.h = oracle.sensitivity(self.geom, self.taps)

    def forward(self, f, out, stream=None):
        out.copy_(torch.from_numpy(self.o.forward(self.geom, self.taps, f.numpy())))
        return out

    def back_update_from_ghat(self, g, ghat, f, ws=None, stream=None):
        gh = ghat.numpy()
        r = np.where(gh > 0, g.numpy() / np.where(gh > 0, gh, 1.0), 0.0)
        z = self.o.backproject(self.geom, self.taps, r)
        f.copy_(torch.from_numpy(f.numpy() * z / self.h))
        return f


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2006_01573_b200 import distributed as dm
    geom = syn.Geometry(8, 6, 5, 40, 30)
    taps = syn.paper_taps(geom, R=1, seed=2)
    import oracle
    g = torch.from_numpy(oracle.forward(geom, taps, syn.scene_blobs(geom)))
    b0, b1 = dm.band_partition(geom.w, world)[rank]
    shard = OracleShard(geom, taps, b0, b1)
    f = torch.ones(shard.m, dtype=torch.float64)
    dm.mlem_band_sharded(shard, g, f, 15, all_reduce=lambda t: dist.all_reduce(t), ghat=torch.empty(geom.n, dtype=torch.float64))
    parts = [None] * world
    dist.all_gather_object(parts, f.numpy())
    if rank == 0:
        results.put(np.concatenate(parts))
    # throughput mode: frame partition covers every frame exactly once
    fr = dm.frame_partition(7, world)
    mine = torch.tensor([fr[rank][1] - fr[rank][0]])
    dist.all_reduce(mine)
    if rank == 0:
        results.put(int(mine.item()))
    dist.destroy_process_group()


def test_band_sharded_mlem_gloo_world2_matches_single_process(oracle_lib):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, q), nprocs=2, start_method="spawn", join=True)
    f_sharded = q.get()
    assert q.get() == 7
    geom = syn.Geometry(8, 6, 5, 40, 30)
    taps = syn.paper_taps(geom, R=1, seed=2)
    g = oracle_lib.forward(geom, taps, syn.scene_blobs(geom))
    want = oracle_lib.mlem(geom, taps, g, np.ones(geom.m), 15)
    np.testing.assert_allclose(f_sharded, want, rtol=1e-12, atol=1e-14)


def _exchange_worker(rank, world, port, region, results):
    """The reduce-scatter / slice-ratio / all-gather schedule of ctis_mlem_band_sharded with real gloo
    collectives and the oracle as the shard projector."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2006_01573_b200 import distributed as dm
    geom = syn.Geometry(9, 7, 5, 40, 30)
    taps = (syn.paper_taps(geom, R=1, seed=2) if region == "paper"
            else syn.random_taps(geom, (2, 6), seed=8, region=region))
    g = torch.from_numpy(oracle.forward(geom, taps, syn.scene_blobs(geom)))
    emax = (geom.a - 1) + geom.gamma * (geom.alpha - 1)
    lo, hi = int(taps.offset.min()), int(taps.offset.max()) + emax
    if hi >= geom.n:
        lo, hi = 0, geom.n - 1
    b0, b1 = dm.band_partition(geom.w, world)[rank]
    shard = OracleShard(geom, taps, b0, b1)
    X = torch.empty(dm.exchange_slices(lo, hi, geom.n, world)[2], dtype=torch.float64)

    def forward_partial(f, X):
        X[:geom.n] += torch.from_numpy(oracle.forward(shard.geom, shard.taps, f.numpy()))

    def ratio_slice(gs, xs):
        gh = xs.numpy().copy()
        xs.copy_(torch.from_numpy(np.where(gh > 0, gs.numpy() / np.where(gh > 0, gh, 1.0), 0.0)))

    def back_update(r, f):
        z = oracle.backproject(shard.geom, shard.taps, r.numpy())
        f.copy_(torch.from_numpy(f.numpy() * z / shard.h))

    f = torch.ones(shard.m, dtype=torch.float64)
    dm.mlem_band_sharded_exchange(forward_partial, ratio_slice, back_update, g, f, 12, lo, hi, rank, world,
                                  reduce_scatter=lambda out, inp: dist.reduce_scatter_tensor(out, inp),
                                  all_gather=lambda out, inp: dist.all_gather_into_tensor(out, inp), X=X)
    parts = [None] * world
    dist.all_gather_object(parts, f.numpy())
    if rank == 0:
        results.put(np.concatenate(parts))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,region", [(2, "paper"), (3, "any"), (2, "nowrap")])
def test_reduce_scatter_exchange_gloo_matches_single_process(oracle_lib, world, region):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_exchange_worker, args=(world, _free_port(), region, q), nprocs=world, start_method="spawn",
                       join=True)
    f_sharded = q.get()
    geom = syn.Geometry(9, 7, 5, 40, 30)
    taps = (syn.paper_taps(geom, R=1, seed=2) if region == "paper"
            else syn.random_taps(geom, (2, 6), seed=8, region=region))
    g = oracle_lib.forward(geom, taps, syn.scene_blobs(geom))
    want = oracle_lib.mlem(geom, taps, g, np.ones(geom.m), 12)
    np.testing.assert_allclose(f_sharded, want, rtol=1e-12, atol=1e-14)


def test_exchange_layout():
    from paper_2006_01573_b200 import distributed as dm
    base, S, floats = dm.exchange_slices(5, 4_194_303, 4_194_304, 8)
    assert base == 4 and S % 4 == 0 and base + 8 * S >= 4_194_304 and floats >= 4_194_304 and floats % 4 == 0
    base, S, floats = dm.exchange_slices(0, 99, 100, 3)
    assert (base, S, floats) == (0, 36, 108)


def test_partitions():
    from paper_2006_01573_b200 import distributed as dm
    assert dm.band_partition(100, 8) == [(0, 13), (13, 26), (26, 39), (39, 52), (52, 64), (64, 76), (76, 88), (88, 100)]
    assert dm.band_partition(50, 4) == [(0, 13), (13, 26), (26, 38), (38, 50)]
    assert dm.frame_partition(256, 8)[-1] == (224, 256)
    with pytest.raises(ValueError):
        dm.band_partition(3, 4)
