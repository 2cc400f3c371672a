"""CPU oracle for the CTIS MLEM hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product package
(paper_2006_01573_b200) never imports it, and it imports nothing from the
product.  See ctis_oracle.c for what is computed and which passage of
PAPER.md each step follows; dense.py builds H literally from Eqs. 3-7 and
fft_ref.py is the paper's own FFT algorithm (Eqs. 13, 17) — both are pins for
the C oracle, used only by tests.

Parity status: forward, back-projection, sensitivity and MLEM are pinned
(tests/test_oracle_*.py).  The paper's quality numbers (relative error 0.02,
average relative pixel error 0.5e-3) need the authors' measured
system matrix and RGB scene: parity unpinned for those (not reproduced).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ctis_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c99"]


def build(force: bool = False) -> str:
    """Compile ctis_oracle.c -> liboracle.so with gcc (plain C, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            i64, P = ctypes.c_int64, ctypes.c_void_p
            geo = [i64] * 5
            lib.oracle_embed_index.argtypes = geo + [i64]
            lib.oracle_embed_index.restype = i64
            lib.oracle_extract_index.argtypes = geo + [i64]
            lib.oracle_extract_index.restype = i64
            for name in ("oracle_forward", "oracle_backproject"):
                getattr(lib, name).argtypes = geo + [P, P, P, P, P]
                getattr(lib, name).restype = ctypes.c_int
            lib.oracle_sensitivity.argtypes = geo + [P, P, P, P]
            lib.oracle_sensitivity.restype = ctypes.c_int
            lib.oracle_mlem.argtypes = geo + [P, P, P, P, P, i64, P]
            lib.oracle_loglik.argtypes = [i64, P, P]
            lib.oracle_loglik.restype = ctypes.c_double
            lib.oracle_mlem_monitored.argtypes = geo + [P, P, P, P, P, i64, ctypes.c_double, P, P]
            lib.oracle_mlem_monitored.restype = ctypes.c_int
            lib.oracle_smart.argtypes = geo + [P, P, P, P, P, i64]
            lib.oracle_smart.restype = ctypes.c_int
            lib.oracle_mlem.restype = ctypes.c_int
            for name in ("oracle_forward_par", "oracle_backproject_par"):
                getattr(lib, name).argtypes = geo + [P, P, P, P, P, ctypes.c_int]
                getattr(lib, name).restype = ctypes.c_int
            lib.oracle_set_threads.argtypes = [ctypes.c_int]
            lib.oracle_set_threads.restype = ctypes.c_int
            lib.oracle_get_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(x: np.ndarray):
    return x.ctypes.data_as(ctypes.c_void_p)


def _geo(geom):
    return (geom.a, geom.alpha, geom.w, geom.gamma, geom.xi)


def _taps(taps):
    ptr = np.ascontiguousarray(taps.ptr, np.int64)
    off = np.ascontiguousarray(taps.offset, np.int64)
    wt = np.ascontiguousarray(np.asarray(taps.weight, np.float32).astype(np.float64))
    return ptr, off, wt


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what} failed with code {rc}")


def set_threads(nthreads: int) -> int:
    """Threads for mlem / mlem_monitored / smart / sensitivity (OpenMP; 1 = the serial functions).

    The parallel path performs the same floating-point operations per output element as the
    serial one (bit-identical results; tests/test_oracle_pins.py::test_parallel_oracle_*)."""
    return int(_load().oracle_set_threads(int(nthreads)))


def get_threads() -> int:
    return int(_load().oracle_get_threads())


class threads:
    """Context manager: `with oracle.threads(os.cpu_count()): oracle.mlem(...)`."""

    def __init__(self, nthreads: int):
        self.n = int(nthreads)

    def __enter__(self):
        self.prev = get_threads()
        set_threads(self.n)
        return self

    def __exit__(self, *exc):
        set_threads(self.prev)
        return False


def forward_par(geom, taps, f, nthreads: int) -> np.ndarray:
    """g = H f with oracle_forward_par (bit-identical to forward(); distinct offsets per band)."""
    lib = _load()
    ptr, off, wt = _taps(taps)
    fd = np.ascontiguousarray(np.asarray(f, np.float64).reshape(-1))
    assert fd.size == geom.m
    g = np.empty(geom.n, np.float64)
    _check(lib.oracle_forward_par(*_geo(geom), _ptr(ptr), _ptr(off), _ptr(wt), _ptr(fd), _ptr(g), int(nthreads)),
           "forward_par")
    return g


def backproject_par(geom, taps, u, nthreads: int) -> np.ndarray:
    """zeta = H^T u with oracle_backproject_par (bit-identical to backproject())."""
    lib = _load()
    ptr, off, wt = _taps(taps)
    ud = np.ascontiguousarray(np.asarray(u, np.float64).reshape(-1))
    assert ud.size == geom.n
    z = np.empty(geom.m, np.float64)
    _check(lib.oracle_backproject_par(*_geo(geom), _ptr(ptr), _ptr(off), _ptr(wt), _ptr(ud), _ptr(z), int(nthreads)),
           "backproject_par")
    return z


def embed_index(geom, j: int) -> int:
    """Eq. 11."""
    return int(_load().oracle_embed_index(*_geo(geom), int(j)))


def extract_index(geom, i: int) -> int:
    """Eq. 15."""
    return int(_load().oracle_extract_index(*_geo(geom), int(i)))


def forward(geom, taps, f) -> np.ndarray:
    """g = H f in float64 (Eq. 12).  f: any shape with m elements (flat order j)."""
    lib = _load()
    ptr, off, wt = _taps(taps)
    fd = np.ascontiguousarray(np.asarray(f, np.float64).reshape(-1))
    assert fd.size == geom.m
    g = np.empty(geom.n, np.float64)
    _check(lib.oracle_forward(*_geo(geom), _ptr(ptr), _ptr(off), _ptr(wt), _ptr(fd), _ptr(g)), "forward")
    return g


def backproject(geom, taps, u) -> np.ndarray:
    """zeta = H^T u in float64 (Eqs. 14-15)."""
    lib = _load()
    ptr, off, wt = _taps(taps)
    ud = np.ascontiguousarray(np.asarray(u, np.float64).reshape(-1))
    assert ud.size == geom.n
    z = np.empty(geom.m, np.float64)
    _check(lib.oracle_backproject(*_geo(geom), _ptr(ptr), _ptr(off), _ptr(wt), _ptr(ud), _ptr(z)), "back")
    return z


def sensitivity(geom, taps) -> np.ndarray:
    """h = H^T 1, float64, m entries."""
    lib = _load()
    ptr, off, wt = _taps(taps)
    h = np.empty(geom.m, np.float64)
    _check(lib.oracle_sensitivity(*_geo(geom), _ptr(ptr), _ptr(off), _ptr(wt), _ptr(h)), "sensitivity")
    return h


def mlem(geom, taps, g, f0, iters: int, return_ghat: bool = False):
    """Alg. 1 in float64: returns f^(iters+1) (and H f^(iters) if asked)."""
    lib = _load()
    ptr, off, wt = _taps(taps)
    gd = np.ascontiguousarray(np.asarray(g, np.float64).reshape(-1))
    f = np.array(np.asarray(f0, np.float64).reshape(-1), copy=True)
    assert gd.size == geom.n and f.size == geom.m
    gh = np.empty(geom.n, np.float64) if return_ghat else None
    _check(lib.oracle_mlem(*_geo(geom), _ptr(ptr), _ptr(off), _ptr(wt), _ptr(gd), _ptr(f), int(iters),
                           _ptr(gh) if gh is not None else None), "mlem")
    return (f, gh) if return_ghat else f


def loglik(g, ghat) -> float:
    """Poisson log-likelihood sum_p [g_p log ghat_p - ghat_p] (ctis_oracle.c: oracle_loglik)."""
    lib = _load()
    gd = np.ascontiguousarray(np.asarray(g, np.float64).reshape(-1))
    hd = np.ascontiguousarray(np.asarray(ghat, np.float64).reshape(-1))
    assert gd.size == hd.size
    return float(lib.oracle_loglik(gd.size, _ptr(gd), _ptr(hd)))


def mlem_monitored(geom, taps, g, f0, max_iters: int, rel_tol: float):
    """Alg. 1 with the per-iteration log-likelihood and the early stop (oracle_mlem_monitored):
    returns (f, ll[:iters_done], iters_done)."""
    lib = _load()
    ptr, off, wt = _taps(taps)
    gd = np.ascontiguousarray(np.asarray(g, np.float64).reshape(-1))
    f = np.array(np.asarray(f0, np.float64).reshape(-1), copy=True)
    assert gd.size == geom.n and f.size == geom.m
    ll = np.zeros(max(int(max_iters), 1), np.float64)
    done = np.zeros(1, np.int64)
    _check(lib.oracle_mlem_monitored(*_geo(geom), _ptr(ptr), _ptr(off), _ptr(wt), _ptr(gd), _ptr(f),
                                     int(max_iters), float(rel_tol), _ptr(ll), _ptr(done)), "mlem_monitored")
    k = int(done[0])
    return f, ll[:k], k


def smart(geom, taps, g, f0, iters: int) -> np.ndarray:
    """SMART (simultaneous MART) in float64 (oracle_smart): returns f after `iters` updates."""
    lib = _load()
    ptr, off, wt = _taps(taps)
    gd = np.ascontiguousarray(np.asarray(g, np.float64).reshape(-1))
    f = np.array(np.asarray(f0, np.float64).reshape(-1), copy=True)
    assert gd.size == geom.n and f.size == geom.m
    _check(lib.oracle_smart(*_geo(geom), _ptr(ptr), _ptr(off), _ptr(wt), _ptr(gd), _ptr(f), int(iters)), "smart")
    return f

