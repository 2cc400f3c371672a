"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Every check compares the oracle with something that is NOT the oracle:
  * the dense H built literally from Eqs. 3-7 (oracle/dense.py), bit for bit;
  * the paper's own Fourier algorithm, Eqs. 13/16/17 (oracle/fft_ref.py);
  * scipy convolve2d / correlate2d for non-wrapping taps (textbook 2-D shifts);
  * closed forms: column sums = per-band tap sums (P:39 with P:93-97);
  * the worked index-map examples (tests/golden/index_map_examples.json).
A dropped term, a sign/index error or a transposed operand in the oracle fails
at least one of these.
"""
import json
import os

import numpy as np
import pytest
import scipy.signal as ss

import ctis_synth as syn
from oracle import dense, fft_ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _random_geoms(count, seed, max_nw=10_000):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        a, alpha = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        gamma, xi = a + int(rng.integers(0, 6)), alpha + int(rng.integers(0, 6))
        w = int(rng.integers(1, 4))
        g = syn.Geometry(a, alpha, w, gamma, xi)
        if g.n * g.w <= max_nw:
            out.append(g)
    return out


GEOMS = _random_geoms(24, seed=11)


# --------------------------------------------------------------------------- index maps
def test_index_map_golden_examples(oracle_lib):
    gold = json.load(open(os.path.join(GOLD, "index_map_examples.json")))
    g = syn.Geometry(**gold["geometry"])
    assert (g.n, g.ell, g.m, g.n // 2 + 1) == tuple(gold["derived"][k] for k in ("n", "ell", "m", "beta"))
    for j, i in gold["embed"]:
        assert oracle_lib.embed_index(g, j) == i
    for i, j in gold["extract"]:
        assert oracle_lib.extract_index(g, i) == j
    pg = gold["paper_geometry"]
    G = syn.Geometry(pg["a"], pg["alpha"], pg["w"], pg["gamma"], pg["xi"])
    assert (G.n, G.ell, G.m) == (pg["n"], pg["ell"], pg["m"])


@pytest.mark.parametrize("g", GEOMS[:12])
def test_index_map_matches_dense_E(oracle_lib, g):
    """Eq. 11 index map == position of the 1 in each column of (I_w (x) E) from Eqs. 5-6."""
    E = dense.dense_E(g)
    IE = np.kron(np.eye(g.w), E)
    rows = IE.argmax(axis=0)
    assert np.all(IE.sum(axis=0) == 1)
    got = np.array([oracle_lib.embed_index(g, j) for j in range(g.m)])
    assert np.array_equal(got, rows)
    assert len(set(got.tolist())) == g.m                                   # injective
    assert np.array_equal(got, fft_ref.embed_indices(g))


# --------------------------------------------------------------------------- projector vs dense H
@pytest.mark.parametrize("gi", range(len(GEOMS)))
def test_forward_back_bit_exact_vs_dense_H(oracle_lib, gi):
    """Tap scatter/gather == literal dense C_i E products (wrapping taps included), bit for bit."""
    g = GEOMS[gi]
    taps = syn.random_taps(g, (1, min(6, g.n)), seed=100 + gi, region="any")
    H = dense.dense_H(g, taps)
    rng = np.random.default_rng(gi)
    f = rng.random(g.m)
    u = rng.standard_normal(g.n)
    assert np.array_equal(oracle_lib.forward(g, taps, f), dense.ordered_matvec(H, f))
    assert np.array_equal(oracle_lib.backproject(g, taps, u), dense.ordered_rmatvec(H, u))
    # sensitivity: column sums of H and the closed form sum_t w_t per band
    h = oracle_lib.sensitivity(g, taps)
    np.testing.assert_allclose(h, H.sum(axis=0), rtol=1e-14, atol=0)
    closed = np.repeat([float(np.sum(taps.band(i)[1].astype(np.float64))) for i in range(g.w)], g.ell)
    np.testing.assert_allclose(h, closed, rtol=1e-14, atol=0)


def test_dense_H_shape_and_structure():
    """H is n x m and each block H_i is built from rectangular circulant T_{i,j}."""
    g = syn.Geometry(3, 2, 2, 5, 4)
    taps = syn.random_taps(g, 3, seed=5)
    H = dense.dense_H(g, taps)
    assert H.shape == (g.n, g.m)
    # column j+1 of a field-stop column block is column j cyclically shifted by one (circulant T_{i,j})
    for i in range(g.w):
        for c in range(g.alpha):
            for r in range(g.a - 1):
                j = i * g.ell + c * g.a + r
                assert np.array_equal(np.roll(H[:, j], 1), H[:, j + 1])


# --------------------------------------------------------------------------- the paper's FFT route
@pytest.mark.parametrize("seed,geom,T,region", [
    (1, syn.Geometry(8, 8, 4, 32, 32), 9, "any"),
    (2, syn.Geometry(13, 7, 3, 40, 23), 17, "any"),
    (3, syn.Geometry(32, 24, 6, 128, 96), 25, "nowrap"),
])
def test_oracle_matches_paper_fft_algorithm(oracle_lib, seed, geom, T, region):
    """Eq. 13 (forward), Eq. 17 (Hermitian back) and Eq. 16 (full-spectrum back) vs the oracle."""
    taps = syn.random_taps(geom, T, seed=seed, region=region)
    rng = np.random.default_rng(seed)
    f = rng.random(geom.m)
    u = rng.random(geom.n)
    gf = oracle_lib.forward(geom, taps, f)
    zb = oracle_lib.backproject(geom, taps, u)
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)
    assert rel(fft_ref.forward(geom, taps, f), gf) < 1e-12
    assert rel(fft_ref.backproject(geom, taps, u), zb) < 1e-12
    assert rel(fft_ref.backproject_full_spectrum(geom, taps, u), zb) < 1e-12


def test_oracle_matches_fft_on_paper_taps_C2(oracle_lib):
    cfg = syn.config("C2")
    taps = syn.paper_taps(cfg)
    f = syn.scene_blobs(cfg.geom)
    gf = oracle_lib.forward(cfg.geom, taps, f)
    ref = fft_ref.forward(cfg.geom, taps, f)
    assert np.linalg.norm(gf - ref) / np.linalg.norm(ref) < 1e-12
    u = np.random.default_rng(0).random(cfg.geom.n)
    zb = oracle_lib.backproject(cfg.geom, taps, u)
    ref = fft_ref.backproject(cfg.geom, taps, u)
    assert np.linalg.norm(zb - ref) / np.linalg.norm(ref) < 1e-12


# --------------------------------------------------------------------------- scipy special case
def _tap_image(g, taps, band):
    K = np.zeros((g.gamma, g.xi))
    for o, w in zip(*taps.band(band)):
        K[int(o) % g.gamma, int(o) // g.gamma] += float(w)
    return K


def test_oracle_matches_scipy_2d_convolution_nowrap(oracle_lib):
    """Non-wrapping taps: the circulant equals a physical 2-D shift (reading R3):
    forward = sum_l convolve2d(f_l, K_l)[:gamma,:xi], back_l = correlate2d(u, K_l)[gamma-1:, xi-1:]."""
    g = syn.Geometry(7, 5, 3, 24, 19)
    taps = syn.random_taps(g, 8, seed=21, region="nowrap")
    rng = np.random.default_rng(4)
    f = rng.random(g.m)
    u = rng.random(g.n)
    F = f.reshape(g.w, g.alpha, g.a)
    G = np.zeros((g.gamma, g.xi))
    for lam in range(g.w):
        full = ss.convolve2d(F[lam].T, _tap_image(g, taps, lam), "full")
        assert np.all(full[g.gamma:, :] == 0) and np.all(full[:, g.xi:] == 0)
        G += full[:g.gamma, :g.xi]
    gf = oracle_lib.forward(g, taps, f).reshape(g.xi, g.gamma).T
    np.testing.assert_allclose(gf, G, rtol=1e-13, atol=1e-15)
    U = u.reshape(g.xi, g.gamma).T
    z = oracle_lib.backproject(g, taps, u).reshape(g.w, g.alpha, g.a)
    for lam in range(g.w):
        c = ss.correlate2d(U, _tap_image(g, taps, lam), "full")
        np.testing.assert_allclose(z[lam].T, c[g.gamma - 1:g.gamma - 1 + g.a, g.xi - 1:g.xi - 1 + g.alpha],
                                   rtol=1e-13, atol=1e-15)


# --------------------------------------------------------------------------- identities
def test_impulse_kernel_is_embed_and_extract(oracle_lib):
    """c = unit impulse at pixel 0 => C = I, forward = embed, back = extract."""
    g = syn.Geometry(3, 4, 2, 7, 6)
    taps = syn.Taps(np.array([0, 1, 2]), np.array([0, 0]), np.array([1.0, 1.0], np.float32))
    f = np.random.default_rng(1).random(g.m)
    v = fft_ref.embed(g, f)                             # (w, n)
    assert np.array_equal(oracle_lib.forward(g, taps, f), v.sum(axis=0))
    u = np.random.default_rng(2).random(g.n)
    z = np.tile(u, g.w)
    assert np.array_equal(oracle_lib.backproject(g, taps, u), fft_ref.extract(g, z))


def test_shift_by_one_impulse(oracle_lib):
    """c = impulse at pixel 1, f = impulse at voxel 0 => g = impulse at pixel 1."""
    g = syn.Geometry(2, 3, 1, 4, 3)
    taps = syn.Taps(np.array([0, 1]), np.array([1]), np.array([1.0], np.float32))
    f = np.zeros(g.m)
    f[0] = 1.0
    out = oracle_lib.forward(g, taps, f)
    assert out[1] == 1.0 and out.sum() == 1.0
    # wrap: last FPA pixel shifted by one lands on pixel 0 (1-D circulant, reading R3)
    g2 = syn.Geometry(2, 1, 1, 2, 1)     # n = 2, field stop fills the FPA
    f2 = np.array([0.0, 1.0])
    out2 = oracle_lib.forward(g2, taps, f2)
    assert np.array_equal(out2, [1.0, 0.0])


def test_adjointness_and_linearity(oracle_lib):
    g = syn.Geometry(24, 20, 5, 61, 47)
    taps = syn.random_taps(g, (3, 12), seed=8, region="any")
    rng = np.random.default_rng(9)
    f1, f2 = rng.standard_normal(g.m), rng.standard_normal(g.m)
    u = rng.standard_normal(g.n)
    Hf = oracle_lib.forward(g, taps, f1)
    lhs, rhs = Hf @ u, f1 @ oracle_lib.backproject(g, taps, u)
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(Hf) * np.linalg.norm(u)
    lin = oracle_lib.forward(g, taps, 2.0 * f1 - 3.0 * f2)
    np.testing.assert_allclose(lin, 2.0 * Hf - 3.0 * oracle_lib.forward(g, taps, f2), rtol=1e-12, atol=1e-12)


# --------------------------------------------------------------------------- MLEM (Eq. 2 / Alg. 1)
def _loglik(g, gh):
    m = gh > 0
    return float(np.sum(g[m] * np.log(gh[m]) - gh[m]))


def test_mlem_one_step_equals_dense_eq2(oracle_lib):
    """One oracle iteration == (f (.) H^T(g (/) Hf)) (/) h with the dense H (Alg. 1 line 12 order)."""
    g = syn.Geometry(4, 3, 3, 9, 7)
    taps = syn.random_taps(g, (2, 5), seed=31, region="any")
    H = dense.dense_H(g, taps)
    rng = np.random.default_rng(3)
    ftrue = rng.random(g.m)
    meas = dense.ordered_matvec(H, ftrue)
    f0 = rng.random(g.m) + 0.5
    gh = dense.ordered_matvec(H, f0)
    u = np.where(gh > 0, meas / np.where(gh > 0, gh, 1.0), 0.0)
    zeta = dense.ordered_rmatvec(H, u)
    h = dense.ordered_rmatvec(H, np.ones(g.n))
    want = (f0 * zeta) / h
    assert np.array_equal(oracle_lib.mlem(g, taps, meas, f0, 1), want)


def test_mlem_invariants(oracle_lib):
    """Nonnegativity, count conservation, monotone Poisson likelihood (Shepp-Vardi, cited P:34)."""
    g = syn.Geometry(6, 5, 4, 15, 12)
    taps = syn.random_taps(g, (2, 6), seed=41, region="any")
    ftrue = syn.scene_random(g, seed=5, zero_frac=0.2).astype(np.float64).reshape(-1)
    meas = oracle_lib.forward(g, taps, ftrue)
    f = np.ones(g.m)
    gh = oracle_lib.forward(g, taps, f)
    L = _loglik(meas, gh)
    for _ in range(200):
        f_next = oracle_lib.mlem(g, taps, meas, f, 1)
        assert np.all(f_next >= 0)
        gh_next = oracle_lib.forward(g, taps, f_next)
        # Sum_p (H f+)_p = Sum_{p: ghat_p > 0} g_p   (derivation in DESIGN.md)
        want = meas[gh > 0].sum()
        assert abs(gh_next.sum() - want) <= 1e-12 * want
        L_next = _loglik(meas, gh_next)
        assert L_next >= L - 1e-9 * abs(L)
        f, gh, L = f_next, gh_next, L_next


def test_mlem_fixed_point_and_zero_image(oracle_lib):
    g = syn.Geometry(5, 4, 3, 13, 11)
    taps = syn.random_taps(g, 4, seed=51, region="any")
    f = np.random.default_rng(6).random(g.m) + 0.1
    meas = oracle_lib.forward(g, taps, f)
    f1 = oracle_lib.mlem(g, taps, meas, f, 1)
    np.testing.assert_allclose(f1, f, rtol=1e-13)
    z = oracle_lib.mlem(g, taps, np.zeros(g.n), f, 1)
    assert np.all(z == 0)
    assert np.array_equal(oracle_lib.mlem(g, taps, meas, f, 0), f)


def test_mlem_w1_is_richardson_lucy(oracle_lib):
    """w = 1, non-wrapping taps: MLEM is textbook Richardson-Lucy with a 2-D PSF (scipy)."""
    g = syn.Geometry(9, 7, 1, 26, 21)
    taps = syn.random_taps(g, 7, seed=61, region="nowrap")
    K = _tap_image(g, taps, 0)
    F = syn.scene_random(g, seed=7, lo=0.2).astype(np.float64)[0].T
    conv = lambda X: ss.convolve2d(X, K, "full")[:g.gamma, :g.xi]
    corr = lambda Y: ss.correlate2d(Y, K, "full")[g.gamma - 1:g.gamma - 1 + g.a, g.xi - 1:g.xi - 1 + g.alpha]
    G = conv(F)
    X = np.ones((g.a, g.alpha))
    norm = corr(np.ones((g.gamma, g.xi)))
    for _ in range(50):
        est = conv(X)
        X = X * corr(np.where(est > 0, G / np.where(est > 0, est, 1), 0.0)) / norm
    meas = G.T.reshape(-1)
    f = oracle_lib.mlem(g, taps, meas, np.ones(g.m), 50)
    np.testing.assert_allclose(f.reshape(g.alpha, g.a).T, X, rtol=1e-11, atol=1e-13)


def test_mlem_matches_fft_em_backend(oracle_lib):
    """SPEC acceptance 5 desk geometry: tap-oracle EM vs paper-FFT EM iterate by iterate (<=1e-9)."""
    g = syn.Geometry(8, 6, 4, 32, 24)
    taps = syn.paper_taps(g, R=1, seed=3)
    ftrue = syn.scene_blobs(g, seed=4).astype(np.float64).reshape(-1)
    meas = oracle_lib.forward(g, taps, ftrue)
    d = fft_ref.spectra(g, taps)
    h = fft_ref.backproject(g, taps, np.ones(g.n), d)
    f_or = np.ones(g.m)
    f_ff = np.ones(g.m)
    for _ in range(50):
        f_or = oracle_lib.mlem(g, taps, meas, f_or, 1)
        gh = fft_ref.forward(g, taps, f_ff, d)
        u = np.where(gh > 1e-300, meas / np.maximum(gh, 1e-300), 0.0)
        f_ff = f_ff * fft_ref.backproject(g, taps, u, d) / h
        assert np.linalg.norm(f_or - f_ff) / np.linalg.norm(f_or) < 1e-9


# --------------------------------------------------------------------------- generator
def test_generator_shapes_and_determinism():
    counts = {"tiny": 9, "C2": 25, "C3": 65, "C4": 49}
    for name, T in counts.items():
        cfg = syn.config(name)
        t1 = syn.paper_taps(cfg)          # asserts the no-wrap box internally
        t2 = syn.paper_taps(cfg)
        assert np.array_equal(t1.offset, t2.offset) and np.array_equal(t1.weight, t2.weight)
        assert np.all(np.diff(t1.ptr) == T)
        assert np.all(t1.weight > 0) and t1.weight.dtype == np.float32
        assert np.all((t1.offset >= 0) & (t1.offset < cfg.geom.n))
    s = syn.scene_blobs(syn.config("C2").geom)
    assert s.shape == (25, 64, 64) and s.dtype == np.float32 and abs(float(s.max()) - 100.0) < 1e-4
    assert np.array_equal(s, syn.scene_blobs(syn.config("C2").geom))


# ------------------------------------------------------------------ §8(f) f-3: log-likelihood and early stop
def test_loglik_matches_scipy_poisson_logpmf(oracle_lib):
    """L = sum_p [g log ghat - ghat] is the Poisson log-likelihood up to the f-independent
    -sum log(g_p!) (Shepp-Vardi): check against scipy.stats.poisson.logpmf on integer counts."""
    from scipy.stats import poisson
    from scipy.special import gammaln
    cfg = syn.config("tiny")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    gbar = oracle_lib.forward(geom, taps, syn.scene_blobs(geom))
    counts = syn.poisson_counts(gbar, seed=3, photons=2.0).astype(np.float64)
    ghat = oracle_lib.forward(geom, taps, syn.scene_random(geom, seed=4, lo=0.5, hi=2.0)) * 2.0
    want = float(np.sum(poisson.logpmf(counts, ghat)) + np.sum(gammaln(counts + 1.0)))
    assert abs(oracle_lib.loglik(counts, ghat) - want) <= 1e-10 * abs(want)
    # conventions (R15): ghat = 0 with g = 0 contributes 0, with g > 0 gives -inf
    assert oracle_lib.loglik([0.0, 1.0], [0.0, 1.0]) == -1.0
    assert oracle_lib.loglik([1.0], [0.0]) == -np.inf


def test_loglik_gradient_is_backprojection_minus_sensitivity(oracle_lib):
    """dL/df_j = sum_p H_pj (g_p/ghat_p - 1) = (H^T (g/ghat))_j - h_j: central differences of the
    oracle's L against its back projection and sensitivity (two independent code paths)."""
    geom = syn.Geometry(5, 4, 2, 11, 9)
    taps = syn.random_taps(geom, (2, 4), seed=8, region="any")
    f = syn.scene_random(geom, seed=1, lo=0.5, hi=1.5).astype(np.float64).reshape(-1)
    g = oracle_lib.forward(geom, taps, syn.scene_random(geom, seed=2, lo=0.5, hi=1.5))
    ghat = oracle_lib.forward(geom, taps, f)
    u = np.divide(g, ghat, out=np.zeros_like(g), where=ghat > 0)
    grad = oracle_lib.backproject(geom, taps, u) - oracle_lib.sensitivity(geom, taps)
    eps = 1e-6
    for j in (0, 7, geom.m // 2, geom.m - 1):
        fp, fm = f.copy(), f.copy()
        fp[j] += eps
        fm[j] -= eps
        d = (oracle_lib.loglik(g, oracle_lib.forward(geom, taps, fp)) -
             oracle_lib.loglik(g, oracle_lib.forward(geom, taps, fm))) / (2 * eps)
        assert abs(d - grad[j]) <= 1e-6 * max(1.0, abs(grad[j]))


def test_mlem_monitored_trace_and_early_stop(oracle_lib):
    """Monitored MLEM: the log-likelihood rises every iteration (Shepp-Vardi); the iterate after
    k updates is the plain MLEM iterate bit for bit; the stopping rule fires where it should."""
    cfg = syn.config("tiny")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    g = syn.poisson_counts(oracle_lib.forward(geom, taps, syn.scene_blobs(geom)), seed=5, photons=1.0)
    f, ll, k = oracle_lib.mlem_monitored(geom, taps, g, np.ones(geom.m), 40, -1.0)
    assert k == 40 and np.all(np.diff(ll) > 0)
    assert np.array_equal(f, oracle_lib.mlem(geom, taps, g, np.ones(geom.m), 40))
    # L_k is the likelihood of f^(k): recompute it from the plain iterates
    f3 = oracle_lib.mlem(geom, taps, g, np.ones(geom.m), 3)
    assert ll[3] == oracle_lib.loglik(g, oracle_lib.forward(geom, taps, f3))
    # huge tolerance: stops after the second update; tol 1e-4: first k with a small relative gain
    assert oracle_lib.mlem_monitored(geom, taps, g, np.ones(geom.m), 40, 1e300)[2] == 2
    _, _, k4 = oracle_lib.mlem_monitored(geom, taps, g, np.ones(geom.m), 40, 1e-4)
    gains = (ll[1:] - ll[:-1]) / np.abs(ll[1:])
    assert k4 == 2 + int(np.argmax(gains <= 1e-4))
    # exact fixed point (g = H f, f0 = f): L is constant, the rule fires at k = 2 even with tol 0
    ft = syn.scene_random(geom, seed=9, lo=0.5, hi=1.5).astype(np.float64).reshape(-1)
    gf = oracle_lib.forward(geom, taps, ft)
    _, llf, kf = oracle_lib.mlem_monitored(geom, taps, gf, ft, 10, 0.0)
    assert kf == 2 and abs(llf[1] - llf[0]) <= 1e-12 * abs(llf[0])


# ------------------------------------------------------------------ §8(f) f-4: SMART (simultaneous MART)
def _kl(a, b):
    """Kullback-Leibler distance KL(a, b) = sum a log(a/b) + b - a (0 log 0 = 0)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    t = np.where(a > 0, a * np.log(np.where(a > 0, a, 1.0) / np.where(b > 0, b, 1.0)), 0.0)
    return float(np.sum(t + b - a))


def test_smart_decreases_kl_and_fixed_point(oracle_lib):
    """SMART minimises KL(Hf, g) and decreases it at every step for consistent positive data
    (Byrne 1993); a fixed point Hf = g is left unchanged; one step equals the dense-H update."""
    cfg = syn.config("tiny")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    ft = syn.scene_random(geom, seed=5, lo=0.5, hi=1.5)
    g = oracle_lib.forward(geom, taps, ft)
    f = np.ones(geom.m)
    kl = []
    for k in range(30):
        kl.append(_kl(oracle_lib.forward(geom, taps, f), g))
        f = oracle_lib.smart(geom, taps, g, f, 1)
    assert np.all(np.diff(kl) < 0)
    assert np.array_equal(oracle_lib.smart(geom, taps, g, np.ones(geom.m), 30), f)
    fx = oracle_lib.smart(geom, taps, g, ft, 3)
    assert np.max(np.abs(fx - ft.reshape(-1))) <= 1e-12 * np.max(ft)
    # dense H (Eqs. 3-7): f <- f * exp(H^T log(g / Hf) / h)
    geom2 = syn.Geometry(4, 3, 2, 9, 7)
    taps2 = syn.random_taps(geom2, (2, 4), seed=2, region="any")
    H = dense.dense_H(geom2, taps2)
    f0 = syn.scene_random(geom2, seed=1, lo=0.5, hi=1.5).astype(np.float64).reshape(-1)
    g2 = H @ syn.scene_random(geom2, seed=2, lo=0.5, hi=1.5).astype(np.float64).reshape(-1)
    gh = H @ f0
    u = np.where((g2 > 0) & (gh > 0), np.log(np.where(g2 > 0, g2, 1) / np.where(gh > 0, gh, 1)), 0.0)
    want = f0 * np.exp((H.T @ u) / H.sum(axis=0))
    assert np.allclose(oracle_lib.smart(geom2, taps2, g2, f0, 1), want, rtol=1e-13, atol=0)


def test_smart_single_unit_tap_is_exact_in_one_step(oracle_lib):
    """w = 1, one unit tap (H a selection): SMART reproduces the data in one step, f = E^T g."""
    geom = syn.Geometry(5, 4, 1, 9, 8)
    off = 2 + 9 * 3
    taps = syn.Taps(np.array([0, 1]), np.array([off]), np.ones(1, np.float32))
    ft = syn.scene_random(geom, seed=3, lo=0.5, hi=1.5)
    g = oracle_lib.forward(geom, taps, ft)
    f = oracle_lib.smart(geom, taps, g, np.ones(geom.m), 1)
    assert np.max(np.abs(f - ft.reshape(-1))) <= 1e-12


# --------------------------------------------------------------------------- threaded oracle
PAR_GEOMS = GEOMS + _random_geoms(12, seed=23, max_nw=40_000)


@pytest.mark.parametrize("gi", range(len(PAR_GEOMS)))
@pytest.mark.parametrize("nthreads", [1, 3, 8])
def test_parallel_oracle_is_bitwise_serial(oracle_lib, gi, nthreads):
    """oracle_forward_par / oracle_backproject_par perform, per output element, the same floating-point
    operations in the same order as the serial oracle (which the dense-H test pins bit for bit), for
    any thread count and with wrapping taps: the results must be identical, not merely close."""
    g = PAR_GEOMS[gi]
    taps = syn.random_taps(g, (1, min(9, g.n)), seed=300 + gi, region="any")
    rng = np.random.default_rng(7 + gi)
    f = rng.random(g.m)
    u = rng.standard_normal(g.n)
    assert np.array_equal(oracle_lib.forward_par(g, taps, f, nthreads), oracle_lib.forward(g, taps, f))
    assert np.array_equal(oracle_lib.backproject_par(g, taps, u, nthreads), oracle_lib.backproject(g, taps, u))


def test_parallel_oracle_paper_workload_and_iterations(oracle_lib):
    """C2 (paper-shaped taps, 25 bands on 512^2): threaded projections and 3 threaded MLEM / SMART /
    monitored-MLEM iterations equal the serial ones bit for bit."""
    cfg = syn.config("C2")
    geom, taps = cfg.geom, syn.paper_taps(cfg)
    f = syn.scene_blobs(geom).reshape(-1).astype(np.float64)
    gs = oracle_lib.forward(geom, taps, f)
    assert np.array_equal(oracle_lib.forward_par(geom, taps, f, 8), gs)
    u = np.random.default_rng(3).random(geom.n)
    assert np.array_equal(oracle_lib.backproject_par(geom, taps, u, 8), oracle_lib.backproject(geom, taps, u))
    f0 = np.ones(geom.m)
    ser = oracle_lib.mlem(geom, taps, gs, f0, 3)
    sm = oracle_lib.smart(geom, taps, gs, f0, 2)
    mon = oracle_lib.mlem_monitored(geom, taps, gs, f0, 3, 0.0)
    with oracle_lib.threads(8):
        assert oracle_lib.get_threads() in (1, 8)
        par = oracle_lib.mlem(geom, taps, gs, f0, 3)
        smp = oracle_lib.smart(geom, taps, gs, f0, 2)
        monp = oracle_lib.mlem_monitored(geom, taps, gs, f0, 3, 0.0)
    assert oracle_lib.get_threads() == 1
    assert np.array_equal(par, ser)
    assert np.array_equal(smp, sm)
    assert np.array_equal(monp[0], mon[0]) and np.array_equal(monp[1], mon[1]) and monp[2] == mon[2]


def test_parallel_forward_rejects_duplicate_offsets(oracle_lib):
    g = syn.Geometry(2, 2, 1, 4, 4)
    taps = syn.Taps(np.array([0, 2]), np.array([3, 3]), np.array([0.5, 0.25], np.float32))
    with pytest.raises(ValueError):
        oracle_lib.forward_par(g, taps, np.ones(g.m), 2)
