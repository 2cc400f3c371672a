"""Dense system matrix H built literally from the paper's Eqs. 3-7 — TEST INFRASTRUCTURE ONLY.

Used by tests to pin the C oracle (oracle/ctis_oracle.c) at tiny sizes
(n*w <= 1e4).  Nothing here is shared with, or imported by, the product.

  Q = [I_a; 0]                        (gamma x a)           P:73-81   (Eq. 5)
  E = [I_alpha (x) Q; 0]              (n x a*alpha)         P:83-91   (Eq. 6)
  C_i = circulant(c_i), n x n, first column c_i             P:93-97   (Eq. 7)
  H_i = C_i E,  H = (H_1 ... H_w)                           P:54-62, P:93-103 (Eqs. 3, 7, 8)

c_i is the band-i calibration image for a point source at field-stop pixel
(0, 0) (reading R2: "first column of T_{i,1}"), vectorised column-major
(reading R1): c_i[o_t] = w_t for each tap (o_t, w_t) of band i, zero elsewhere.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg


def dense_Q(geom) -> np.ndarray:
    """Eq. 5: the gamma x a matrix [I_a; 0]."""
    return np.vstack([np.eye(geom.a), np.zeros((geom.gamma - geom.a, geom.a))])


def dense_E(geom) -> np.ndarray:
    """Eq. 6: the n x (a*alpha) matrix [I_alpha (x) Q; 0]."""
    top = np.kron(np.eye(geom.alpha), dense_Q(geom))
    return np.vstack([top, np.zeros((geom.n - top.shape[0], top.shape[1]))])


def calibration_image(geom, taps, band: int) -> np.ndarray:
    """c_band as a dense length-n vector (first column of C_band)."""
    c = np.zeros(geom.n)
    off, wt = taps.band(band)
    for o, v in zip(off, wt):
        c[int(o)] += float(v)
    return c


def dense_C(geom, taps, band: int) -> np.ndarray:
    """Eq. 7: the n x n circulant C_band with first column c_band."""
    return scipy.linalg.circulant(calibration_image(geom, taps, band))


def dense_H(geom, taps) -> np.ndarray:
    """Eqs. 3 and 7: H = (C_1 E, ..., C_w E), n x m."""
    E = dense_E(geom)
    return np.hstack([dense_C(geom, taps, i) @ E for i in range(geom.w)])


def ordered_matvec(H: np.ndarray, f: np.ndarray) -> np.ndarray:
    """H f summed in ascending column index j (the oracle's documented order)."""
    g = np.zeros(H.shape[0])
    for j in range(H.shape[1]):
        g = g + H[:, j] * f[j]
    return g


def ordered_rmatvec(H: np.ndarray, u: np.ndarray) -> np.ndarray:
    """H^T u summed in ascending row index p (the oracle's documented order)."""
    z = np.zeros(H.shape[1])
    for p in range(H.shape[0]):
        z = z + H[p, :] * u[p]
    return z
