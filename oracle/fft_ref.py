"""The paper's own WBH projector (Fourier route) in numpy float64 — TEST INFRASTRUCTURE ONLY.

An independent second formulation of the same operator H, used by tests to pin
the C oracle at every size:

  embed   v = (I_w (x) E) f via the index map           P:127-133 (Eq. 11), Alg. 1 line 6
  forward g = F1^-1 sum_i d_i (.) F1 v_i, d_i = F1 c_i   P:140-145 (Eq. 13), Alg. 1 line 7
  back    z_i = F1^-1 (conj(d_i) (.) F1 u)               P:180-184 (Eq. 17), Alg. 1 lines 9-10
          zeta = (I_w (x) E)^T z                         P:164-172 (Eq. 15), Alg. 1 line 11
  back'   z_i = F1 D_i F1^-1 u (full spectrum)           P:173-178 (Eq. 16)

F1 is the unnormalised DFT (numpy.fft.fft / rfft), F1^-1 its inverse (1/n).
Half spectra of length beta = floor(n/2)+1 use the Hermitian symmetry of P:180-190.
"""
from __future__ import annotations

import numpy as np


def embed_indices(geom) -> np.ndarray:
    """Eq. 11: i(j) for j = 0..m-1 (zero-based), as an int64 vector."""
    a, gamma, n, l = geom.a, geom.gamma, geom.n, geom.ell
    j = np.arange(geom.m, dtype=np.int64)
    s = j // l
    return j - s * l + (gamma - a) * ((j - s * l) // a) + s * n


def embed(geom, f) -> np.ndarray:
    """v = (I_w (x) E) f as a (w, n) array (initialise v = 0, then scatter)."""
    v = np.zeros(geom.n * geom.w)
    v[embed_indices(geom)] = np.asarray(f, np.float64).reshape(-1)
    return v.reshape(geom.w, geom.n)


def extract(geom, z) -> np.ndarray:
    """zeta = (I_w (x) E)^T z (Eq. 15): zeta_i = z_{j(i)}."""
    return np.asarray(z, np.float64).reshape(-1)[embed_indices(geom)]


def spectra(geom, taps) -> np.ndarray:
    """d_i = F1 c_i, half spectra (w, beta)."""
    c = np.zeros((geom.w, geom.n))
    for i in range(geom.w):
        off, wt = taps.band(i)
        np.add.at(c[i], off.astype(np.int64), wt.astype(np.float64))
    return np.fft.rfft(c, axis=1)


def forward(geom, taps, f, d=None) -> np.ndarray:
    """Eq. 13 / Alg. 1 line 7."""
    d = spectra(geom, taps) if d is None else d
    v = embed(geom, f)
    acc = (d * np.fft.rfft(v, axis=1)).sum(axis=0)
    return np.fft.irfft(acc, n=geom.n)


def backproject(geom, taps, u, d=None) -> np.ndarray:
    """Eq. 17 + Eq. 15 / Alg. 1 lines 9-11."""
    d = spectra(geom, taps) if d is None else d
    U = np.fft.rfft(np.asarray(u, np.float64).reshape(-1))
    z = np.fft.irfft(np.conj(d) * U[None, :], n=geom.n, axis=1)
    return extract(geom, z)


def backproject_full_spectrum(geom, taps, u) -> np.ndarray:
    """Eq. 16: C_i^T u = F1 D_i F1^-1 u with full-length complex transforms."""
    c = np.zeros((geom.w, geom.n))
    for i in range(geom.w):
        off, wt = taps.band(i)
        np.add.at(c[i], off.astype(np.int64), wt.astype(np.float64))
    D = np.fft.fft(c, axis=1)
    ui = np.fft.ifft(np.asarray(u, np.float64).reshape(-1))
    z = np.fft.fft(D * ui[None, :], axis=1).real
    return extract(geom, z)
