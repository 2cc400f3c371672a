"""Seeded synthetic inputs for the CTIS MLEM hot path (shared by tests, bench and smoke).

This module is the ONE place both the oracle side and the CUDA side get their
inputs from.  It holds none of the method's arithmetic: no projection, no ratio,
no back-projection, no update.  It only draws calibration taps (the sparse
first columns c_lambda of the circulant blocks C_lambda, Eq. 7)
and datacube scenes f (Eq. 9).  The measurement g = Hf is
computed by whoever needs it (the oracle in parity tests, the product forward
in the bench), never here.

Layouts (column-major everywhere, reading R1 / PAPER.md P:24):
  * scene f : float32, shape (w, alpha, a)  -> flat index j = lam*a*alpha + c*a + r
  * taps    : CSR over bands, tap_ptr int64 (w+1), tap_offset int64 in [0, n)
              (1-D column-major FPA index dr + gamma*dc), tap_weight float32 > 0.

Recipe:
  * diffraction orders (p, q) in [-R, R]^2 around the zero-order anchor
    (r0, c0) = ((gamma-a)//2, (xi-alpha)//2);
  * dispersion d(lam) = D0 * (1 + 0.16 * lam/(w-1)), D0 = a: a 16 % fractional
    bandwidth, the 421-495 nm span of the paper's system matrix;
  * order (p, q) of band lam lands at (r0 + floor(p d + 1/2), c0 + floor(q d + 1/2));
  * C3 adds dispersion streaks: ring-k orders get k+1 taps along (sgn p, sgn q);
  * weights s(lam) * eta_{p,q} * U(0.9, 1.1), rounded to float32, drawn from
    numpy default_rng(1234) in (lam, p, q, u) order.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, Tuple

import numpy as np

__all__ = [
    "Geometry", "Config", "CONFIGS", "PAPER_TABLE1", "config", "paper_taps", "random_taps",
    "scene_blobs", "scene_constant", "scene_random", "Taps",
]


@dataclasses.dataclass(frozen=True)
class Geometry:
    """Instrument geometry: a x alpha field stop, gamma x xi FPA, w bands."""
    a: int
    alpha: int
    w: int
    gamma: int
    xi: int

    @property
    def n(self) -> int:          # FPA pixels, n = gamma*xi
        return self.gamma * self.xi

    @property
    def ell(self) -> int:        # voxels per band, l = a*alpha
        return self.a * self.alpha

    @property
    def m(self) -> int:          # datacube length, m = a*alpha*w
        return self.ell * self.w


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    geom: Geometry
    R: int            # orders (p, q) in [-R, R]^2
    streak: bool      # per-order dispersion streaks (C3)
    K: int            # MLEM iterations
    frames: int = 1   # snapshot-video frames (C5)


CONFIGS: Dict[str, Config] = {
    # BASELINE.json configs[0..4]
    "tiny": Config("tiny", Geometry(8, 8, 4, 32, 32), R=1, streak=False, K=20),
    "C2": Config("C2", Geometry(64, 64, 25, 512, 512), R=2, streak=False, K=100),
    "C3": Config("C3", Geometry(128, 128, 50, 1024, 1024), R=2, streak=True, K=100),
    "C4": Config("C4", Geometry(256, 256, 100, 2048, 2048), R=3, streak=False, K=100),
    "C5": Config("C5", Geometry(128, 128, 50, 1024, 1024), R=2, streak=True, K=100, frames=256),
}


# The paper's own benchmark geometry (Table 1 at P:238-266): an 89 x 80 field stop on a
# 2048 x 2048 FPA with w in {75, 24, 3} bands of 1 nm from 421 nm.  The authors' measured system matrix
# is not available; the taps follow this module's diffraction-order recipe with 7 x 7 orders.  The
# field stop's a = 89 is not a multiple of 4 (no 16-byte row stride for TMA boxes of f).
PAPER_TABLE1: Dict[str, Config] = {
    "T1w75": Config("T1w75", Geometry(89, 80, 75, 2048, 2048), R=3, streak=False, K=25),
    "T1w24": Config("T1w24", Geometry(89, 80, 24, 2048, 2048), R=3, streak=False, K=25),
    "T1w3": Config("T1w3", Geometry(89, 80, 3, 2048, 2048), R=3, streak=False, K=25),
}


def config(name: str) -> Config:
    return CONFIGS[name] if name in CONFIGS else PAPER_TABLE1[name]


@dataclasses.dataclass
class Taps:
    """Sparse calibration images in CSR form (one row per band)."""
    ptr: np.ndarray      # int64 (w+1,)
    offset: np.ndarray   # int64 (nnz,), 1-D column-major FPA index in [0, n)
    weight: np.ndarray   # float32 (nnz,)

    @property
    def w(self) -> int:
        return len(self.ptr) - 1

    def band(self, lam: int) -> Tuple[np.ndarray, np.ndarray]:
        s, e = int(self.ptr[lam]), int(self.ptr[lam + 1])
        return self.offset[s:e], self.weight[s:e]


def _csr(per_band) -> Taps:
    ptr = [0]
    offs, wts = [], []
    for d in per_band:
        keys = sorted(d)
        offs.extend(keys)
        wts.extend(d[k] for k in keys)
        ptr.append(len(offs))
    return Taps(np.asarray(ptr, np.int64), np.asarray(offs, np.int64),
                np.asarray(wts, np.float32))


def paper_taps(cfg: Config | Geometry, R: int | None = None, streak: bool | None = None,
               seed: int = 1234, check_nowrap: bool = True) -> Taps:
    """Diffraction-order taps shaped like a CTIS calibration (recipe in module docstring).

    Returns CSR taps sorted by offset within each band; duplicate offsets within a
    band are merged (weights summed) so each band is a proper image c_lambda.
    """
    if isinstance(cfg, Config):
        geom, R, streak = cfg.geom, cfg.R if R is None else R, cfg.streak if streak is None else streak
    else:
        geom = cfg
        assert R is not None
        streak = bool(streak)
    a, alpha, w, gamma, xi = geom.a, geom.alpha, geom.w, geom.gamma, geom.xi
    rng = np.random.default_rng(seed)
    r0, c0 = (gamma - a) // 2, (xi - alpha) // 2
    D0 = float(a)
    eta0 = 0.3
    c_ring = 0.7 / sum(8.0 / k for k in range(1, R + 1)) if R > 0 else 0.0
    per_band = []
    for lam in range(w):
        frac = lam / (w - 1) if w > 1 else 0.0
        d = D0 * (1.0 + 0.16 * frac)
        s = 0.5 + 0.5 * math.sin(math.pi * (lam + 0.5) / w)
        band: Dict[int, float] = {}
        for p in range(-R, R + 1):
            for q in range(-R, R + 1):
                k = max(abs(p), abs(q))
                eta = eta0 if k == 0 else c_ring / (k * k)
                dr = r0 + math.floor(p * d + 0.5)
                dc = c0 + math.floor(q * d + 0.5)
                nu = (k + 1) if (streak and k > 0) else 1
                sp = (p > 0) - (p < 0)
                sq = (q > 0) - (q < 0)
                for u in range(nu):
                    U = rng.uniform(0.9, 1.1)
                    rr, cc = dr + u * sp, dc + u * sq
                    if check_nowrap:
                        assert 0 <= rr <= gamma - a and 0 <= cc <= xi - alpha, (lam, p, q, u, rr, cc)
                    o = rr + gamma * cc
                    wt = float(np.float32(s * eta * U / nu))
                    band[o] = float(np.float32(band.get(o, 0.0) + wt))
        per_band.append(band)
    return _csr(per_band)


def random_taps(geom: Geometry, taps_per_band: int | Tuple[int, int], seed: int,
                wmin: float = 0.05, wmax: float = 1.0, region: str = "any") -> Taps:
    """Uniformly random distinct tap offsets per band (parity cases).

    region="any" draws offsets over all of [0, n): shifted field stops then carry
    across FPA columns and wrap past the end of the flattened FPA, exercising
    the full 1-D circulant of Eq. 7 (reading R3).  region="nowrap"
    keeps every tap inside the no-wrap box 0<=dr<=gamma-a, 0<=dc<=xi-alpha.
    """
    rng = np.random.default_rng(seed)
    n = geom.n
    per_band = []
    for lam in range(geom.w):
        if isinstance(taps_per_band, tuple):
            T = int(rng.integers(taps_per_band[0], taps_per_band[1] + 1))
        else:
            T = taps_per_band
        if region == "any":
            T = min(T, n)
            offs = rng.choice(n, size=T, replace=False)
        else:
            H, W = geom.gamma - geom.a + 1, geom.xi - geom.alpha + 1
            T = min(T, H * W)
            flat = rng.choice(H * W, size=T, replace=False)
            offs = (flat % H) + geom.gamma * (flat // H)
        wts = rng.uniform(wmin, wmax, size=T).astype(np.float32)
        per_band.append({int(o): float(wt) for o, wt in zip(offs, wts)})
    return _csr(per_band)


def scene_blobs(geom: Geometry, seed: int = 99, nblobs: int = 8) -> np.ndarray:
    """Scene S1: 1 + sum of spatial x spectral Gaussian blobs, rescaled to max 100 (float32, (w, alpha, a))."""
    a, alpha, w = geom.a, geom.alpha, geom.w
    rng = np.random.default_rng(seed)
    r = np.arange(a, dtype=np.float64)[None, None, :]
    c = np.arange(alpha, dtype=np.float64)[None, :, None]
    lam = np.arange(w, dtype=np.float64)[:, None, None]
    f = np.ones((w, alpha, a), np.float64)
    for _ in range(nblobs):
        cr, cc = rng.uniform(0, a), rng.uniform(0, alpha)
        sig = rng.uniform(a / 16, a / 4)
        lc, lw = rng.uniform(0, w), rng.uniform(max(w / 8, 0.5), max(w / 2, 1.0))
        f += 100.0 * np.exp(-((lam - lc) ** 2) / (2 * lw * lw)) * \
            np.exp(-((r - cr) ** 2 + (c - cc) ** 2) / (2 * sig * sig))
    f *= 100.0 / f.max()
    return f.astype(np.float32)


def scene_constant(geom: Geometry, value: float = 100.0) -> np.ndarray:
    """Scene S0: the paper's fully illuminated field stop f(x,y,lambda) = 100."""
    return np.full((geom.w, geom.alpha, geom.a), value, np.float32)


def scene_random(geom: Geometry, seed: int, lo: float = 0.0, hi: float = 1.0,
                 zero_frac: float = 0.0) -> np.ndarray:
    """Uniform random nonnegative cube; optionally a fraction of exact zeros."""
    rng = np.random.default_rng(seed)
    f = rng.uniform(lo, hi, size=(geom.w, geom.alpha, geom.a))
    if zero_frac > 0:
        f[rng.random(f.shape) < zero_frac] = 0.0
    return f.astype(np.float32)


def frame_scene(geom: Geometry, frame: int) -> np.ndarray:
    """C5 snapshot-video frame i: scene S1 with seed 1000 + i."""
    return scene_blobs(geom, seed=1000 + frame)


def poisson_counts(g: np.ndarray, seed: int, photons: float = 1.0) -> np.ndarray:
    """Photon-limited measurement: independent Poisson counts with mean photons * g_p, returned as
    float32 (§8(f) f-3 second workload shape).  Random numbers only: the mean g comes from the caller."""
    rng = np.random.default_rng(seed)
    lam = np.asarray(g, np.float64) * float(photons)
    return rng.poisson(lam).astype(np.float32)

