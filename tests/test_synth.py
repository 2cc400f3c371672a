"""-m "not gpu": the seeded workload generator (ctis_synth) — shapes of the BASELINE configs and of the
paper's own Table 1 geometry, tap validity (no wrap, sorted, positive weights), and the
reachable-FPA box the ratio pass relies on (every pixel E(q) + o of every voxel and tap lies inside it)."""
import numpy as np
import pytest

import ctis_synth as syn


@pytest.mark.parametrize("name", ["T1w75", "T1w24", "T1w3"])
def test_paper_table1_geometry(name):
    cfg = syn.config(name)
    g = cfg.geom
    assert (g.a, g.alpha, g.gamma, g.xi) == (89, 80, 2048, 2048)
    assert g.w == {"T1w75": 75, "T1w24": 24, "T1w3": 3}[name]               # Table 1
    assert cfg.K == 25 and g.a % 4 != 0                                     # K = 25 row; odd field stop
    taps = syn.paper_taps(cfg)                                              # asserts no wrap internally
    assert taps.w == g.w and int(taps.ptr[-1]) == 49 * g.w
    for lam in range(g.w):
        off, wt = taps.band(lam)
        assert np.all(np.diff(off) > 0) and np.all(wt > 0)


@pytest.mark.parametrize("name", ["tiny", "C2", "C3", "C4", "T1w3"])
def test_reachable_box_covers_every_incidence(name):
    """Brute force on a subsample of voxels: E(q) + o for every tap lies in the 2-D box spanned by the
    taps' (row, column) plus the field stop — the region outside it never receives model counts."""
    cfg = syn.config(name)
    g = cfg.geom
    taps = syn.paper_taps(cfg)
    dr, dc = taps.offset % g.gamma, taps.offset // g.gamma
    r0, r1 = dr.min(), dr.max() + g.a - 1
    c0, c1 = dc.min(), dc.max() + g.alpha - 1
    rng = np.random.default_rng(0)
    q = rng.integers(0, g.ell, size=min(g.ell, 4096))
    qr, qc = q % g.a, q // g.a
    p = (qr + g.gamma * qc)[:, None] + taps.offset[None, :]                # E(q) + o (no wrap: < n)
    assert p.max() < g.n
    pr, pc = p % g.gamma, p // g.gamma
    assert pr.min() >= r0 and pr.max() <= r1 and pc.min() >= c0 and pc.max() <= c1
