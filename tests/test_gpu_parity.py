"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle.

Tolerances (BASELINE.json north_star): relative L2 <= 1e-5 for one forward or
back projection, <= 1e-3 on f after the configuration's MLEM iterations.
A single unit tap at offset 0 must be bit-exact (H is then a 0/1 selection).
"""
import os

import numpy as np
import pytest

import ctis_synth as syn

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PROJ_TOL = 1e-5
MLEM_TOL = 1e-3


ELEM_FACTOR = 1        # per-element bound = ELEM_FACTOR x the L2 tolerance (see check())


def rel(a, b):
    a = np.asarray(a, np.float64).reshape(-1)
    b = np.asarray(b, np.float64).reshape(-1)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def elem_rel(a, b):
    """Largest per-element relative error |a_i - b_i| / (|b_i| + 1e-3 max|b|): a single corrupted
    element shows here even when the global relative L2 is inside its tolerance."""
    a = np.asarray(a, np.float64).reshape(-1)
    b = np.asarray(b, np.float64).reshape(-1)
    if b.size == 0:
        return 0.0
    e = np.abs(a - b) / (np.abs(b) + 1e-3 * max(float(np.abs(b).max()), 1e-300))
    return float(e.max())


def check(got, want, tol, what=""):
    """Relative L2 <= tol (north_star) AND every element within ELEM_FACTOR x tol (relative, floored at
    1e-3 of the largest |want|); both numbers are printed (pytest -s / the GPU logs)."""
    r, e = rel(got, want), elem_rel(got, want)
    print(f"[parity] {what}: rel L2 = {r:.3e}, max elem rel = {e:.3e} (tol {tol:g})")
    assert r <= tol, (what, r)
    assert e <= ELEM_FACTOR * tol, (what, e)
    return r


@pytest.fixture(scope="module", autouse=True)
def oracle_threads(oracle_lib):
    """The oracle on every host core for this module (bit-identical to the serial oracle:
    tests/test_oracle_pins.py::test_parallel_oracle_*), so full-size runs finish in seconds."""
    prev = oracle_lib.get_threads()
    oracle_lib.set_threads(os.cpu_count() or 1)
    yield
    oracle_lib.set_threads(prev)


@pytest.fixture(scope="module")
def ctis():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2006_01573_b200 as m
    return m


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda:0")


def cuda(x, dev):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, np.float32).reshape(-1))).to(dev)


# ------------------------------------------------------------------ single projections at every config size
@pytest.mark.parametrize("name", ["tiny", "C2", "C3", "C4"])
def test_forward_back_paper_configs(ctis, oracle_lib, dev, name):
    cfg = syn.config(name)
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    plan = ctis.Plan.from_geometry(geom, taps)
    f = syn.scene_blobs(geom)
    gh = plan.forward(cuda(f, dev))
    want = oracle_lib.forward(geom, taps, f)
    check(gh.cpu().numpy(), want, PROJ_TOL, f"{name} forward")
    u = np.random.default_rng(1).uniform(0.5, 1.5, geom.n).astype(np.float32)
    z = plan.backproject(cuda(u, dev))
    check(z.cpu().numpy(), oracle_lib.backproject(geom, taps, u), PROJ_TOL, f"{name} back")
    h = plan.sensitivity()
    check(h.cpu().numpy(), oracle_lib.sensitivity(geom, taps), 1e-6, f"{name} sensitivity")


GEOMS = [
    syn.Geometry(1, 1, 1, 1, 1),            # degenerate: n = 1
    syn.Geometry(3, 5, 2, 3, 5),            # field stop fills the FPA
    syn.Geometry(7, 5, 3, 40, 29),          # ragged everything
    syn.Geometry(33, 17, 6, 70, 45),        # several tiles + ragged tails
    syn.Geometry(65, 40, 9, 130, 100),      # > 2 forward tiles in both directions
    syn.Geometry(128, 32, 5, 200, 33),
]


@pytest.mark.parametrize("gi", range(len(GEOMS)))
@pytest.mark.parametrize("region", ["any", "nowrap"])
def test_forward_back_random_wrapping_taps(ctis, oracle_lib, dev, gi, region):
    geom = GEOMS[gi]
    taps = syn.random_taps(geom, (1, 13), seed=10 + gi, region=region)
    plan = ctis.Plan.from_geometry(geom, taps)
    rng = np.random.default_rng(gi)
    f = rng.random(geom.m).astype(np.float32)
    u = rng.random(geom.n).astype(np.float32)
    assert rel(plan.forward(cuda(f, dev)).cpu().numpy(), oracle_lib.forward(geom, taps, f)) <= PROJ_TOL
    assert rel(plan.backproject(cuda(u, dev)).cpu().numpy(), oracle_lib.backproject(geom, taps, u)) <= PROJ_TOL


def test_unit_tap_is_bit_exact_embed_extract(ctis, oracle_lib, dev):
    """Unit taps whose shifted field stops do not overlap: H is a 0/1 selection, every g pixel
    has at most one term and every z voxel exactly one -> bit-exact (embed / extract)."""
    geom = syn.Geometry(37, 21, 2, 100, 50)
    taps = syn.Taps(np.array([0, 1, 2]), np.array([0, 100 * 21 + 3]), np.ones(2, np.float32))
    plan = ctis.Plan.from_geometry(geom, taps)
    f = np.random.default_rng(3).random(geom.m).astype(np.float32)
    got = plan.forward(cuda(f, dev)).cpu().numpy()
    assert np.array_equal(got, oracle_lib.forward(geom, taps, f).astype(np.float32))
    u = np.random.default_rng(4).random(geom.n).astype(np.float32)
    z = plan.backproject(cuda(u, dev)).cpu().numpy()
    assert np.array_equal(z, oracle_lib.backproject(geom, taps, u).astype(np.float32))


def test_full_wrap_taps_bit_exact_single_tap_per_band(ctis, oracle_lib, dev):
    """One tap per band at offsets that carry and wrap: still a permutation -> bit-exact."""
    for off in (9 * 11 * 2 - 1, 18, 9 * 11 * 2 - 9 * 3 + 5, 9 * 11 * 2 - 3):
        geom = syn.Geometry(9, 6, 1, 18, 11)
        taps = syn.Taps(np.array([0, 1]), np.array([off]), np.ones(1, np.float32))
        plan = ctis.Plan.from_geometry(geom, taps)
        f = np.random.default_rng(5).random(geom.m).astype(np.float32)
        assert np.array_equal(plan.forward(cuda(f, dev)).cpu().numpy(),
                              oracle_lib.forward(geom, taps, f).astype(np.float32))
        u = np.random.default_rng(6).random(geom.n).astype(np.float32)
        assert np.array_equal(plan.backproject(cuda(u, dev)).cpu().numpy(),
                              oracle_lib.backproject(geom, taps, u).astype(np.float32))


# ------------------------------------------------------------------ MLEM
def _mlem_case(ctis, oracle_lib, dev, geom, taps, K, ftrue, tol=MLEM_TOL, what="mlem"):
    g = oracle_lib.forward(geom, taps, ftrue).astype(np.float32)
    want = oracle_lib.mlem(geom, taps, g, np.ones(geom.m), K)
    plan = ctis.Plan.from_geometry(geom, taps)
    gd = cuda(g, dev)
    fd = torch.ones(geom.m, dtype=torch.float32, device=dev)
    plan.mlem(gd, fd, K)
    return check(fd.cpu().numpy(), want, tol, what), plan, gd, fd


@pytest.mark.parametrize("name", ["tiny", "C2", "C3"])
def test_mlem_paper_configs(ctis, oracle_lib, dev, name):
    cfg = syn.config(name)
    _mlem_case(ctis, oracle_lib, dev, cfg.geom, syn.paper_taps(cfg), cfg.K, syn.scene_blobs(cfg.geom),
               what=f"{name} MLEM K={cfg.K}")


def test_mlem_C4_first_iterations_vs_oracle(ctis, oracle_lib, dev):
    """Full C4 size, 2 iterations: still at projection-level agreement."""
    cfg = syn.config("C4")
    _mlem_case(ctis, oracle_lib, dev, cfg.geom, syn.paper_taps(cfg), 2, syn.scene_blobs(cfg.geom), tol=1e-5,
               what="C4 MLEM K=2")


def test_mlem_C4_headline_100_iterations_vs_oracle(ctis, oracle_lib, dev):
    """The benchmarked configuration itself: C4, K = 100 (north_star: 1e-3 on f after 100 iterations,
    PAPER.md P:203-212), the GPU in the bench's launch configuration (one CUDA graph of 100 iterations)
    against the fp64 oracle on every host core."""
    cfg = syn.config("C4")
    assert cfg.K == 100
    _mlem_case(ctis, oracle_lib, dev, cfg.geom, syn.paper_taps(cfg), cfg.K, syn.scene_blobs(cfg.geom),
               what="C4 MLEM K=100")


def test_mlem_C4_full_run_invariants(ctis, dev):
    """Full C4 run (K=100) in the bench's launch configuration: properties that hold at any size —
    nonnegativity and count conservation sum(H f^(k+1)) = sum_{ghat^(k)>0} g."""
    cfg = syn.config("C4")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    plan = ctis.Plan.from_geometry(geom, taps)
    g = plan.forward(cuda(syn.scene_blobs(geom), dev))
    f = torch.ones(geom.m, dtype=torch.float32, device=dev)
    plan.mlem(g, f, cfg.K)
    gh = plan.forward(f)
    assert bool((f >= 0).all())
    s_g, s_gh = g.double().sum().item(), gh.double().sum().item()
    assert abs(s_gh - s_g) <= 1e-4 * s_g


def test_mlem_random_wrapping(ctis, oracle_lib, dev):
    geom = syn.Geometry(33, 17, 6, 70, 45)
    taps = syn.random_taps(geom, (2, 9), seed=77, region="any")
    r, *_ = _mlem_case(ctis, oracle_lib, dev, geom, taps, 30, syn.scene_random(geom, seed=3, lo=0.1, zero_frac=0.1))
    assert r <= MLEM_TOL, r


def test_mlem_iters_zero_and_fixed_point(ctis, oracle_lib, dev):
    cfg = syn.config("tiny")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    plan = ctis.Plan.from_geometry(geom, taps)
    f = torch.rand(geom.m, device=dev) + 0.5
    f0 = f.clone()
    g = plan.forward(f)
    plan.mlem(g, f, 0)
    assert torch.equal(f, f0)
    plan.mlem(g, f, 5)      # H f0 = g exactly up to fp32 -> stays put
    assert rel(f.cpu().numpy(), f0.cpu().numpy()) <= 1e-5


def test_mlem_zero_image_gives_zero(ctis, dev):
    cfg = syn.config("tiny")
    plan = ctis.Plan.from_geometry(cfg.geom, syn.paper_taps(cfg))
    f = torch.ones(cfg.geom.m, device=dev)
    plan.mlem(torch.zeros(cfg.geom.n, device=dev), f, 1)
    assert bool((f == 0).all())


def test_graph_and_direct_launch_identical(ctis, dev):
    cfg = syn.config("C2")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    plan = ctis.Plan.from_geometry(geom, taps)
    g = plan.forward(cuda(syn.scene_blobs(geom), dev))
    f1 = torch.ones(geom.m, device=dev)
    f2 = torch.ones(geom.m, device=dev)
    plan.mlem(g, f1, 10)
    plan.set_option(ctis.OPT_USE_GRAPH, 0)
    plan.mlem(g, f2, 10)
    # the forward accumulates chunk partials with red.add: equal up to fp32 summation order
    assert rel(f1.cpu().numpy(), f2.cpu().numpy()) <= 1e-6


# ------------------------------------------------------------------ batched frames (snapshot video)
def test_batched_frames_equal_single_frame_runs(ctis, oracle_lib, dev):
    cfg = syn.config("C2")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    plan = ctis.Plan.from_geometry(geom, taps)
    F = 5
    scenes = np.stack([syn.frame_scene(geom, i).reshape(-1) for i in range(F)])
    g = plan.forward(cuda(scenes, dev).view(F, geom.m))
    fb = torch.ones(F, geom.m, device=dev)
    plan.mlem(g, fb, 20)
    for i in range(F):
        fi = torch.ones(geom.m, device=dev)
        plan.mlem(g[i].contiguous(), fi, 20)
        assert rel(fi.cpu().numpy(), fb[i].cpu().numpy()) <= 1e-6
    want = oracle_lib.mlem(geom, taps, g[2].cpu().numpy(), np.ones(geom.m), 20)
    assert rel(fb[2].cpu().numpy(), want) <= MLEM_TOL


# ------------------------------------------------------------------ latency mode on one device (virtual shards)
def test_band_shards_sum_to_full_forward_and_mlem(ctis, oracle_lib, dev):
    from paper_2006_01573_b200 import distributed as dist_mod
    cfg = syn.config("C2")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    full = ctis.Plan.from_geometry(geom, taps)
    ftrue = syn.scene_blobs(geom)
    f = cuda(ftrue, dev)
    parts = dist_mod.band_partition(geom.w, 3)
    shards = [ctis.Plan.from_geometry(geom, taps, band_range=p) for p in parts]
    ghat = sum(s.forward(f[p[0] * geom.ell:p[1] * geom.ell].contiguous()) for s, p in zip(shards, parts))
    check(ghat.cpu().numpy(), oracle_lib.forward(geom, taps, ftrue), PROJ_TOL, "C2 band-shard forward sum")
    # MLEM with the all-reduce replaced by an on-device sum of the partials, against the oracle
    g_np = oracle_lib.forward(geom, taps, ftrue).astype(np.float32)
    g = cuda(g_np, dev)
    f_loc = [torch.ones(s.m, device=dev) for s in shards]
    out = dist_mod.mlem_band_sharded_local(shards, g, f_loc, cfg.K)
    want = oracle_lib.mlem(geom, taps, g_np, np.ones(geom.m), cfg.K)
    check(torch.cat(out).cpu().numpy(), want, MLEM_TOL, f"C2 band-sharded MLEM K={cfg.K} (3 virtual shards)")
    with pytest.raises(ctis.CtisError):
        shards[0].mlem(g, f_loc[0], 1)


@pytest.mark.parametrize("nshards", [2, 5])
def test_band_shards_wrapping_taps_vs_oracle(ctis, oracle_lib, dev, nshards):
    """Latency-mode maths on uneven shards with wrapping taps (element-loader kernels) against the oracle."""
    from paper_2006_01573_b200 import distributed as dist_mod
    geom = syn.Geometry(33, 17, 7, 70, 45)
    taps = syn.random_taps(geom, (2, 9), seed=91, region="any")
    ftrue = syn.scene_random(geom, seed=5, lo=0.1, zero_frac=0.1)
    g_np = oracle_lib.forward(geom, taps, ftrue).astype(np.float32)
    g = cuda(g_np, dev)
    parts = dist_mod.band_partition(geom.w, nshards)
    shards = [ctis.Plan.from_geometry(geom, taps, band_range=p) for p in parts]
    out = dist_mod.mlem_band_sharded_local(shards, g, [torch.ones(s.m, device=dev) for s in shards], 25)
    want = oracle_lib.mlem(geom, taps, g_np, np.ones(geom.m), 25)
    check(torch.cat(out).cpu().numpy(), want, MLEM_TOL, f"wrapping band-sharded MLEM ({nshards} shards)")


# ------------------------------------------------------------------ fused ratio (CTIS_OPT_FUSED_RATIO = 1)
@pytest.mark.parametrize("name", ["C2", "C3"])
def test_fused_ratio_option_vs_oracle(ctis, oracle_lib, dev, name):
    """Two kernels per iteration: the cooperative forward turns g_hat into r after a grid barrier, the
    back kernel zeroes the other workspace half.  MLEM (single and batched) and SMART vs the oracle."""
    cfg = syn.config(name)
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    plan = ctis.Plan.from_geometry(geom, taps)
    plan.set_option(ctis.OPT_FUSED_RATIO, 1)
    g_np = oracle_lib.forward(geom, taps, syn.scene_blobs(geom)).astype(np.float32)
    g = cuda(g_np, dev)
    f = torch.ones(geom.m, device=dev)
    plan.mlem(g, f, 30)
    assert plan.last_launch_count() == 2 + 30 * (plan.info()["fwd_pages"] + plan.info()["back_pages"])  # + validation
    check(f.cpu().numpy(), oracle_lib.mlem(geom, taps, g_np, np.ones(geom.m), 30), MLEM_TOL, f"{name} fused MLEM K=30")
    fs = torch.ones(geom.m, device=dev)
    plan.smart(g, fs, 10)
    check(fs.cpu().numpy(), oracle_lib.smart(geom, taps, g_np, np.ones(geom.m), 10), MLEM_TOL, f"{name} fused SMART")
    F = 3
    gb = torch.stack([g, g * 0.5, g * 2.0]).contiguous()
    fb = torch.ones(F, geom.m, device=dev)
    plan.mlem(gb, fb, 12)
    for i, sc in enumerate((1.0, 0.5, 2.0)):
        want = oracle_lib.mlem(geom, taps, g_np.astype(np.float64) * sc, np.ones(geom.m), 12)
        check(fb[i].cpu().numpy(), want, MLEM_TOL, f"{name} fused batched frame {i}")


# ------------------------------------------------------------------ latency mode through libctis + NCCL
@pytest.mark.parametrize("case", ["C2", "C3", "wrap"])
def test_band_sharded_nccl_single_rank_vs_oracle(ctis, oracle_lib, dev, case):
    """ctis_mlem_band_sharded on a one-rank NCCL communicator (this box has one GPU): the whole
    schedule — exchange-range slicing, reduce-scatter, slice ratio, all-gather, back update, captured
    with the NCCL calls in one CUDA graph — against the oracle."""
    if case == "wrap":
        geom = syn.Geometry(33, 17, 6, 70, 45)
        taps = syn.random_taps(geom, (2, 9), seed=77, region="any")
        K, ftrue = 25, syn.scene_random(geom, seed=3, lo=0.1)
    else:
        cfg = syn.config(case)
        geom, taps, K, ftrue = cfg.geom, syn.paper_taps(cfg), cfg.K, syn.scene_blobs(cfg.geom)
    g_np = oracle_lib.forward(geom, taps, ftrue).astype(np.float32)
    try:
        comm = ctis.Comm(1, 0, ctis.comm_unique_id(), 0)
    except ctis.CtisError as e:
        pytest.skip(f"NCCL unavailable: {e}")
    shard = ctis.Plan.from_geometry(geom, taps, band_range=(0, geom.w))
    f = torch.ones(geom.m, device=dev)
    shard.mlem_band_sharded(comm, cuda(g_np, dev), f, K)
    launches = shard.last_launch_count()
    want = oracle_lib.mlem(geom, taps, g_np, np.ones(geom.m), K)
    check(f.cpu().numpy(), want, MLEM_TOL, f"{case} band-sharded NCCL (1 rank) K={K}")
    assert launches >= 3 * K
    f2 = torch.ones(geom.m, device=dev)          # replay of the cached graph
    shard.mlem_band_sharded(comm, cuda(g_np, dev), f2, K)
    assert rel(f2.cpu().numpy(), f.cpu().numpy()) <= 1e-6
    f3 = torch.ones(geom.m, device=dev)
    shard.mlem_band_sharded(comm, cuda(g_np, dev), f3, 0)
    assert bool((f3 == 1).all())
    comm.close()


@pytest.mark.parametrize("case", ["C2", "wrap"])
def test_fused_nvlink_exchange_single_rank_vs_oracle(ctis, oracle_lib, dev, case):
    """CTIS_OPT_EXCHANGE = 1: the exchange buffer is an NCCL symmetric-memory window
    and ONE kernel reduces each rank's pixel slice over all ranks, forms r and stores it to every rank.
    On this one-GPU box the team has one rank (peer-pointer path; NVLS multimem needs >= 2 GPUs on
    NVSwitch): the slicing, the LSA barriers and the ratio are exercised, against the oracle."""
    if case == "wrap":
        geom = syn.Geometry(33, 17, 6, 70, 45)
        taps = syn.random_taps(geom, (2, 9), seed=77, region="any")
        K, ftrue = 25, syn.scene_random(geom, seed=3, lo=0.1)
    else:
        cfg = syn.config(case)
        geom, taps, K, ftrue = cfg.geom, syn.paper_taps(cfg), cfg.K, syn.scene_blobs(cfg.geom)
    g_np = oracle_lib.forward(geom, taps, ftrue).astype(np.float32)
    try:
        comm = ctis.Comm(1, 0, ctis.comm_unique_id(), 0)
    except ctis.CtisError as e:
        pytest.skip(f"NCCL unavailable: {e}")
    shard = ctis.Plan.from_geometry(geom, taps, band_range=(0, geom.w))
    shard.set_option(ctis.OPT_EXCHANGE, 1)
    f = torch.ones(geom.m, device=dev)
    try:
        shard.mlem_band_sharded(comm, cuda(g_np, dev), f, K)
    except ctis.CtisError as e:
        if e.status == ctis.ERR_UNSUPPORTED:
            pytest.skip(f"NCCL symmetric memory unavailable: {e}")
        raise
    torch.cuda.synchronize()
    want = oracle_lib.mlem(geom, taps, g_np, np.ones(geom.m), K)
    check(f.cpu().numpy(), want, MLEM_TOL, f"{case} fused NVLink exchange (1 rank) K={K}")
    f2 = torch.ones(geom.m, device=dev)
    shard.set_option(ctis.OPT_EXCHANGE, 0)
    shard.mlem_band_sharded(comm, cuda(g_np, dev), f2, K)
    assert rel(f2.cpu().numpy(), f.cpu().numpy()) <= 1e-5
    comm.close()


def _nccl_worker(rank, world, port, q, exchange=0):
    import os as _os
    import torch.distributed as tdist
    _os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    tdist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device(f"cuda:{rank}"))
    import paper_2006_01573_b200 as m
    from paper_2006_01573_b200 import distributed as dm
    import oracle
    cfg = syn.config("C2")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    g_np = oracle.forward(geom, taps, syn.scene_blobs(geom)).astype(np.float32)
    b0, b1 = dm.band_partition(geom.w, world)[rank]
    shard = m.Plan.from_geometry(geom, taps, device=rank, band_range=(b0, b1))
    shard.set_option(m.OPT_EXCHANGE, exchange)
    comm = dm.make_comm(rank)
    f = torch.ones(shard.m, device=f"cuda:{rank}")
    shard.mlem_band_sharded(comm, torch.from_numpy(g_np).cuda(rank), f, cfg.K)
    parts = [None] * world
    tdist.all_gather_object(parts, f.cpu().numpy())
    if rank == 0:
        q.put(np.concatenate(parts))
    tdist.destroy_process_group()


@pytest.mark.parametrize("exchange", [0, 1])
def test_band_sharded_nccl_multi_gpu_vs_oracle(ctis, oracle_lib, exchange):
    """Two ranks on two GPUs (runs only where >= 2 GPUs are visible): NCCL collectives (0) and the fused
    NVLink exchange kernel (1)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (this gpurun box exposes one)")
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    q = mp.get_context("spawn").SimpleQueue()
    mp.start_processes(_nccl_worker, args=(2, port, q, exchange), nprocs=2, start_method="spawn", join=True)
    cfg = syn.config("C2")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    g_np = oracle_lib.forward(geom, taps, syn.scene_blobs(geom)).astype(np.float32)
    check(q.get(), oracle_lib.mlem(geom, taps, g_np, np.ones(geom.m), cfg.K), MLEM_TOL, "C2 band-sharded NCCL 2 GPUs")


# ------------------------------------------------------------------ end-to-end host path
def test_mlem_host_path_matches_device_path(ctis, dev):
    cfg = syn.config("C2")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    plan = ctis.Plan.from_geometry(geom, taps)
    g = plan.forward(cuda(syn.scene_blobs(geom), dev))
    fd = torch.ones(geom.m, device=dev)
    plan.mlem(g, fd, 15)
    fh = np.ones(geom.m, np.float32)
    plan.mlem_host(g.cpu().numpy(), fh, 15)
    assert rel(fh, fd.cpu().numpy()) <= 1e-6


# ------------------------------------------------------------------ error behaviour
def test_error_codes(ctis, dev):
    geom = syn.Geometry(8, 8, 2, 32, 32)
    good = syn.random_taps(geom, 3, seed=1)

    def make(**kw):
        args = dict(tap_ptr=good.ptr, tap_offset=good.offset, tap_weight=good.weight)
        args.update(kw)
        return ctis.Plan(geom.a, geom.alpha, geom.w, geom.gamma, geom.xi, **args)

    for kw, code in [
        (dict(tap_offset=np.where(np.arange(6) == 0, geom.n, good.offset)), ctis.ERR_TAP),
        (dict(tap_weight=np.where(np.arange(6) == 1, -1.0, good.weight).astype(np.float32)), ctis.ERR_TAP),
        (dict(tap_weight=np.where(np.arange(6) == 1, np.nan, good.weight).astype(np.float32)), ctis.ERR_TAP),
        (dict(tap_offset=np.array([5, 5, 7, 1, 2, 3])), ctis.ERR_TAP),
        (dict(tap_ptr=np.array([0, 0, 6])), ctis.ERR_TAP),
    ]:
        with pytest.raises(ctis.CtisError) as ei:
            make(**kw)
        assert ei.value.status == code
    with pytest.raises(ctis.CtisError) as ei:
        ctis.Plan(8, 8, 2, 4, 32, good)
    assert ei.value.status == ctis.ERR_DIMENSION
    with pytest.raises(ctis.CtisError) as ei:
        ctis.Plan(8, 8, 2, 32, 32, good, band_range=(1, 1))
    assert ei.value.status == ctis.ERR_DIMENSION
    plan = make()
    g = torch.ones(geom.n, device=dev)
    g[7] = float("nan")
    with pytest.raises(ctis.CtisError) as ei:
        plan.mlem(g, torch.ones(geom.m, device=dev), 3)
    assert ei.value.status == ctis.ERR_DATA
    f = torch.ones(geom.m, device=dev)
    f[0] = -1
    with pytest.raises(ctis.CtisError) as ei:
        plan.mlem(torch.ones(geom.n, device=dev), f, 3)
    assert ei.value.status == ctis.ERR_DATA
    with pytest.raises(ctis.CtisError) as ei:
        plan.mlem(torch.ones(geom.n, device=dev), torch.ones(geom.m, device=dev), -1)
    assert ei.value.status == ctis.ERR_INVALID_ARGUMENT


@pytest.mark.parametrize("variant", ["default", "loader", "strip", "split"])
def test_no_stale_shared_memory_reads(ctis, variant):
    """Every projection kernel with CTIS_DEBUG=8 NaN-fills its window ring first: results must not
    change (a band without taps in a forward pass once read a slot it never loaded).  Variants: the
    default kernel choice (odd field stops take the repacked TMA forward), the element-loader forward
    (CTIS_FWD_REPACK=0), the strip forward forced on every TMA plan (CTIS_FWD_STRIP=1) and the mode-split
    back projection forced on every plan with the persistent back kernel (CTIS_BACK_SPLIT=4)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, CTIS_DEBUG="8")
    if variant == "loader":
        env["CTIS_FWD_REPACK"] = "0"
    if variant == "strip":
        env["CTIS_FWD_STRIP"] = "1"
    if variant == "split":  # mode-split back projection (partial z red.add + update pass) on every plan
        env["CTIS_BACK_SPLIT"] = "4"
    r = subprocess.run([sys.executable, os.path.join(here, "poison_case.py"), "solvers"], env=env,
                       capture_output=True, text=True, timeout=900)
    print(r.stdout[-2000:])
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("name", ["T1w3", "T1w24"])
def test_paper_table1_geometry_vs_oracle(ctis, oracle_lib, dev, name):
    """The paper's own benchmark geometry (89 x 80 field stop on a 2048^2 FPA, w = 3 / 24): the odd
    field stop (a % 4 != 0) runs the repacked TMA forward and the reachable-box ratio pass.  Single
    projections at 1e-5 and MLEM K = 25 (Table 1's K) at 1e-3 against the oracle."""
    cfg = syn.config(name)
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    plan = ctis.Plan.from_geometry(geom, taps)
    ft = syn.scene_constant(geom)                       # fully illuminated field stop, f = 100
    g_np = oracle_lib.forward(geom, taps, ft).astype(np.float32)
    check(plan.forward(cuda(ft.ravel(), dev)).cpu().numpy(), oracle_lib.forward(geom, taps, ft), PROJ_TOL,
          f"{name} forward")
    u = np.random.default_rng(5).uniform(0.5, 1.5, geom.n).astype(np.float32)
    check(plan.backproject(cuda(u, dev)).cpu().numpy(), oracle_lib.backproject(geom, taps, u), PROJ_TOL,
          f"{name} back")
    f = torch.ones(geom.m, device=dev)
    plan.mlem(cuda(g_np, dev), f, cfg.K)
    check(f.cpu().numpy(), oracle_lib.mlem(geom, taps, g_np, np.ones(geom.m), cfg.K), MLEM_TOL, f"{name} MLEM K={cfg.K}")


# ------------------------------------------------------------------ §8(f) f-3: log-likelihood, early stop, H^T g init
@pytest.mark.parametrize("name,photons,tol", [("tiny", 1.0, 1e-4), ("C2", 4.0, 1e-5), ("C3", 2.0, 3e-6)])
def test_mlem_monitored_vs_oracle(ctis, oracle_lib, dev, name, photons, tol):
    """Poisson-count frames: the device-side loop's log-likelihood trace matches the oracle's, the
    GPU stops exactly where its own trace satisfies the rule (R16, decided in the kernel's
    fp64), and f equals the oracle's plain MLEM iterate after that many updates."""
    cfg = syn.config(name)
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    g = syn.poisson_counts(oracle_lib.forward(geom, taps, syn.scene_blobs(geom)), seed=11, photons=photons)
    plan = ctis.Plan.from_geometry(geom, taps)
    fd = torch.ones(geom.m, dtype=torch.float32, device=dev)
    ll, done = plan.mlem_monitored(cuda(g, dev), fd, cfg.K, tol)
    k = int(done.item())
    ll = ll.cpu().numpy()
    assert 2 <= k <= cfg.K and np.all(ll[k:] == 0.0)
    _, ll_o, k_o = oracle_lib.mlem_monitored(geom, taps, g, np.ones(geom.m), cfg.K, -1.0)
    assert np.all(np.abs(ll[:k] - ll_o[:k]) <= 1e-5 * np.abs(ll_o[:k]))
    gains = (ll[1:k] - ll[:k - 1]) <= tol * np.abs(ll[1:k])
    want_k = 2 + int(np.argmax(gains)) if gains.any() else cfg.K
    assert k == want_k
    assert rel(fd.cpu().numpy(), oracle_lib.mlem(geom, taps, g, np.ones(geom.m), k)) <= MLEM_TOL


def test_mlem_monitored_runs_all_iterations_and_zero(ctis, oracle_lib, dev):
    cfg = syn.config("tiny")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    g = oracle_lib.forward(geom, taps, syn.scene_blobs(geom)).astype(np.float32)
    plan = ctis.Plan.from_geometry(geom, taps)
    fd = torch.ones(geom.m, dtype=torch.float32, device=dev)
    ll, done = plan.mlem_monitored(cuda(g, dev), fd, 25, -1.0)
    assert int(done.item()) == 25 and np.all(np.diff(ll.cpu().numpy()) > 0)
    f2 = torch.ones(geom.m, dtype=torch.float32, device=dev)
    plan.mlem(cuda(g, dev), f2, 25)
    assert rel(fd.cpu().numpy(), f2.cpu().numpy()) <= 1e-6  # same kernels as ctis_mlem (atomic order aside)
    f3 = torch.ones(geom.m, dtype=torch.float32, device=dev)
    _, done0 = plan.mlem_monitored(cuda(g, dev), f3, 0, 1e-3)
    assert int(done0.item()) == 0 and bool((f3 == 1).all())


def test_mlem_from_backprojection_init(ctis, oracle_lib, dev):
    """f^(1) = H^T g, the paper's other initial guess: ctis_backproject then ctis_mlem."""
    cfg = syn.config("C2")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    g = oracle_lib.forward(geom, taps, syn.scene_blobs(geom)).astype(np.float32)
    plan = ctis.Plan.from_geometry(geom, taps)
    f0 = plan.backproject(cuda(g, dev))
    assert rel(f0.cpu().numpy(), oracle_lib.backproject(geom, taps, g)) <= PROJ_TOL
    plan.mlem(cuda(g, dev), f0, 30)
    want = oracle_lib.mlem(geom, taps, g, oracle_lib.backproject(geom, taps, g), 30)
    assert rel(f0.cpu().numpy(), want) <= MLEM_TOL


# ------------------------------------------------------------------ §8(f) f-2: the paper's FFT projector (comparator)
@pytest.mark.parametrize("name", ["tiny", "C2"])
def test_fft_projector_vs_oracle(ctis, oracle_lib, dev, name):
    """CTIS_OPT_PROJECTOR = 1 (Eqs. 13/17 with cuFFT) computes the same H as the taps (fp32 FFT
    round-off: relative L2 <= 1e-5 per projection, <= 1e-3 on f after K iterations)."""
    cfg = syn.config(name)
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    plan = ctis.Plan.from_geometry(geom, taps)
    plan.set_option(ctis.OPT_PROJECTOR, 1)
    f = syn.scene_blobs(geom)
    g = oracle_lib.forward(geom, taps, f)
    assert rel(plan.forward(cuda(f, dev)).cpu().numpy(), g) <= PROJ_TOL
    u = np.random.default_rng(1).uniform(0.5, 1.5, geom.n).astype(np.float32)
    assert rel(plan.backproject(cuda(u, dev)).cpu().numpy(), oracle_lib.backproject(geom, taps, u)) <= PROJ_TOL
    g32 = g.astype(np.float32)
    fd = torch.ones(geom.m, dtype=torch.float32, device=dev)
    plan.mlem(cuda(g32, dev), fd, cfg.K)
    assert rel(fd.cpu().numpy(), oracle_lib.mlem(geom, taps, g32, np.ones(geom.m), cfg.K)) <= MLEM_TOL


def test_fft_projector_wrapping_taps_and_switch_back(ctis, oracle_lib, dev):
    """The Fourier route is the 1-D circulant of Eq. 7, wrap included; switching back to the taps
    (option 0) restores the tap kernels (graphs are re-captured)."""
    geom = syn.Geometry(33, 17, 6, 70, 45)
    taps = syn.random_taps(geom, (2, 9), seed=77, region="any")
    plan = ctis.Plan.from_geometry(geom, taps)
    f = syn.scene_random(geom, seed=3, lo=0.1, zero_frac=0.1)
    g = oracle_lib.forward(geom, taps, f).astype(np.float32)
    for proj in (1, 0, 1):
        plan.set_option(ctis.OPT_PROJECTOR, proj)
        assert rel(plan.forward(cuda(f, dev)).cpu().numpy(), oracle_lib.forward(geom, taps, f)) <= PROJ_TOL
        fd = torch.ones(geom.m, dtype=torch.float32, device=dev)
        plan.mlem(cuda(g, dev), fd, 10)
        assert rel(fd.cpu().numpy(), oracle_lib.mlem(geom, taps, g, np.ones(geom.m), 10)) <= MLEM_TOL


# ------------------------------------------------------------------ §8(f) f-4: SMART on the same projector
@pytest.mark.parametrize("name", ["tiny", "C2", "C3"])
def test_smart_vs_oracle(ctis, oracle_lib, dev, name):
    cfg = syn.config(name)
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    K = min(cfg.K, 30)
    g = oracle_lib.forward(geom, taps, syn.scene_blobs(geom)).astype(np.float32)
    plan = ctis.Plan.from_geometry(geom, taps)
    fd = torch.ones(geom.m, dtype=torch.float32, device=dev)
    plan.smart(cuda(g, dev), fd, K)
    assert rel(fd.cpu().numpy(), oracle_lib.smart(geom, taps, g, np.ones(geom.m), K)) <= MLEM_TOL


def test_smart_wrapping_batched_and_fft_projector(ctis, oracle_lib, dev):
    """Wrapping taps (element-loader kernels), two frames in one call, and the Fourier projector."""
    geom = syn.Geometry(33, 17, 6, 70, 45)
    taps = syn.random_taps(geom, (2, 9), seed=77, region="any")
    gs = [oracle_lib.forward(geom, taps, syn.scene_random(geom, seed=s, lo=0.1, zero_frac=0.1)).astype(np.float32)
          for s in (3, 4)]
    want = [oracle_lib.smart(geom, taps, g, np.ones(geom.m), 12) for g in gs]
    plan = ctis.Plan.from_geometry(geom, taps)
    for proj in (0, 1):
        plan.set_option(ctis.OPT_PROJECTOR, proj)
        fd = torch.ones((2, geom.m), dtype=torch.float32, device=dev)
        plan.smart(torch.from_numpy(np.stack(gs)).to(dev), fd, 12)
        for i in range(2):
            assert rel(fd[i].cpu().numpy(), want[i]) <= MLEM_TOL


def test_batched_frames_many_items_per_cta(ctis, dev):
    """8 frames of C3: every persistent CTA walks many work items, so the TMA ring's refill points
    drift across items with an odd number of windows (a back-kernel deadlock once hid here)."""
    cfg = syn.config("C3")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    plan = ctis.Plan.from_geometry(geom, taps)
    F = 8
    scenes = np.stack([syn.frame_scene(geom, i).reshape(-1) for i in range(F)])
    g = plan.forward(cuda(scenes, dev).view(F, geom.m))
    fb = torch.ones(F, geom.m, device=dev)
    plan.mlem(g, fb, 5)
    for i in (0, 5, 7):
        fi = torch.ones(geom.m, device=dev)
        plan.mlem(g[i].contiguous(), fi, 5)
        assert rel(fi.cpu().numpy(), fb[i].cpu().numpy()) <= 1e-6


def test_C5_launch_configuration_sampled(ctis, oracle_lib, dev):
    """C5 as bench.py runs it on one GPU: 256 C3 frames in ONE batched MLEM of K = 100 iterations.
    Every frame's measurement comes from the oracle; sampled outputs: frames 0, 17, 128 and 255
    against the oracle's K = 100 reconstruction, frames 0 and 255 against their single-frame runs."""
    cfg = syn.config("C5")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    plan = ctis.Plan.from_geometry(geom, taps)
    F, K = cfg.frames, cfg.K
    assert (F, K) == (256, 100)
    g_np = np.stack([oracle_lib.forward_par(geom, taps, syn.frame_scene(geom, i), os.cpu_count() or 1)
                     .astype(np.float32) for i in range(F)])
    g = torch.from_numpy(g_np).to(dev)
    fb = torch.ones(F, geom.m, device=dev)
    plan.mlem(g, fb, K)
    torch.cuda.synchronize()
    for i in (0, F - 1):
        fi = torch.ones(geom.m, device=dev)
        plan.mlem(g[i].contiguous(), fi, K)
        assert rel(fi.cpu().numpy(), fb[i].cpu().numpy()) <= 1e-5
    for i in (0, 17, 128, F - 1):
        want = oracle_lib.mlem(geom, taps, g_np[i], np.ones(geom.m), K)
        check(fb[i].cpu().numpy(), want, MLEM_TOL, f"C5 frame {i} MLEM K={K}")


# ------------------------------------------------------------------ large / dense calibration images
def _dense_order_taps(geom, R, blob, seed):
    """A dense calibration image per band: (2R+1)^2 dispersing diffraction orders, each a
    (2*blob+1)^2 block of nonzero pixels -> T = (2R+1)^2 (2 blob+1)^2 taps per band, no wrap."""
    rng = np.random.default_rng(seed)
    r0, c0 = (geom.gamma - geom.a) // 2, (geom.xi - geom.alpha) // 2
    per_band = []
    for lam in range(geom.w):
        d = geom.a * (1.0 + 0.16 * lam / max(geom.w - 1, 1))
        taps = {}
        for p in range(-R, R + 1):
            for q in range(-R, R + 1):
                for u in range(-blob, blob + 1):
                    for v in range(-blob, blob + 1):
                        dr = r0 + int(np.floor(p * d + 0.5)) + u
                        dc = c0 + int(np.floor(q * d + 0.5)) + v
                        assert 0 <= dr <= geom.gamma - geom.a and 0 <= dc <= geom.xi - geom.alpha
                        taps[dr + geom.gamma * dc] = float(rng.uniform(0.01, 0.1))
        per_band.append(taps)
    ptr, offs, wts = [0], [], []
    for d in per_band:
        for k in sorted(d):
            offs.append(k)
            wts.append(d[k])
        ptr.append(len(offs))
    return syn.Taps(np.asarray(ptr, np.int64), np.asarray(offs, np.int64), np.asarray(wts, np.float32))


@pytest.mark.parametrize("case", ["random_wrap_T2000", "dense_orders_T1225"])
def test_large_tap_counts_multi_page_plans(ctis, oracle_lib, dev, case):
    """Plans whose tap tables need several 64 KB __constant__ pages and whose back chunks must be split
    to fit one page (ctis_api.cu build_tables): T = 500..2000 random wrapping taps per band, and a dense
    calibration image of 7 x 7 dispersing orders x 5 x 5 pixels (T = 1225 per band)."""
    if case == "random_wrap_T2000":
        geom = syn.Geometry(16, 12, 6, 96, 80)
        taps = syn.random_taps(geom, (500, 2000), seed=17, region="any")
    else:
        geom = syn.Geometry(32, 32, 12, 320, 320)
        taps = _dense_order_taps(geom, R=3, blob=2, seed=4)
    plan = ctis.Plan.from_geometry(geom, taps)
    info = plan.info()
    print(f"[plan] {case}: {info}")
    assert info["fwd_pages"] >= 2 and info["back_pages"] >= 2, info
    rng = np.random.default_rng(8)
    f = rng.random(geom.m).astype(np.float32)
    u = rng.uniform(0.5, 1.5, geom.n).astype(np.float32)
    check(plan.forward(cuda(f, dev)).cpu().numpy(), oracle_lib.forward(geom, taps, f), PROJ_TOL, f"{case} forward")
    check(plan.backproject(cuda(u, dev)).cpu().numpy(), oracle_lib.backproject(geom, taps, u), PROJ_TOL,
          f"{case} back")
    _mlem_case(ctis, oracle_lib, dev, geom, taps, 20, syn.scene_random(geom, seed=2, lo=0.1),
               what=f"{case} MLEM K=20")


def test_pdl_launches_parity():
    """CTIS_PDL=1 (programmatic dependent launch between the MLEM kernels): every kernel of the chain
    must wait for its predecessor (griddepcontrol.wait) — MLEM / SMART / monitored MLEM on the TMA and
    element-loader kernel families against the oracle, in a subprocess (the switch is read once)."""
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, CTIS_PDL="1")
    r = subprocess.run([sys.executable, os.path.join(here, "poison_case.py"), "solvers"], env=env,
                       capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0


def test_error_codes_new_entry_points(ctis, dev):
    """ctis_mlem_monitored / ctis_smart / CTIS_OPT_PROJECTOR argument checking."""
    import ctypes
    from paper_2006_01573_b200 import _lib
    geom = syn.Geometry(8, 8, 2, 32, 32)
    plan = ctis.Plan.from_geometry(geom, syn.random_taps(geom, 3, seed=1))
    g = torch.ones(geom.n, device=dev)
    f = torch.ones(geom.m, device=dev)
    ws = plan.workspace(1)
    ll = torch.zeros(8, dtype=torch.float64, device=dev)
    cnt = torch.zeros(2, dtype=torch.int32, device=dev)
    P = ctypes.c_void_p
    call = lambda it, llp, cp: _lib.ctis_mlem_monitored(plan._h, P(g.data_ptr()), P(f.data_ptr()), it, 1e-3,
                                                        P(ws.data_ptr()), llp, cp, P(0))
    assert call(-1, P(ll.data_ptr()), P(cnt.data_ptr())) == ctis.ERR_INVALID_ARGUMENT
    assert call(4, P(0), P(cnt.data_ptr())) == ctis.ERR_INVALID_ARGUMENT
    assert call(4, P(ll.data_ptr() + 4), P(cnt.data_ptr())) == ctis.ERR_INVALID_ARGUMENT   # misaligned
    assert call(4, P(ll.data_ptr()), P(cnt.data_ptr() + 2)) == ctis.ERR_INVALID_ARGUMENT
    assert call(4, P(ll.data_ptr()), P(cnt.data_ptr())) == ctis.OK
    torch.cuda.synchronize()
    assert 2 <= int(cnt[0].item()) <= 4
    with pytest.raises(ctis.CtisError) as ei:
        plan.smart(g, f, -1)
    assert ei.value.status == ctis.ERR_INVALID_ARGUMENT
    with pytest.raises(ctis.CtisError) as ei:
        plan.set_option(ctis.OPT_PROJECTOR, 2)
    assert ei.value.status == ctis.ERR_INVALID_ARGUMENT
    g[3] = -1.0
    with pytest.raises(ctis.CtisError) as ei:
        plan.smart(g, f, 2)
    assert ei.value.status == ctis.ERR_DATA
