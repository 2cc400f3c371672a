"""B200-native (sm_100a) shift-invariant CTIS MLEM reconstruction — arXiv 2006.01573.

Thin ctypes binding over libctis.so (include/ctis.h).  Argument marshalling
only: every arithmetic step of the hot path (forward projection, ratio,
back-projection, multiplicative update, sensitivity) runs in the CUDA kernels
of libctis.  PyTorch provides device memory and the current stream.  There is
no CPU fallback: if libctis.so is missing this module raises at import.

Names follow the paper: a x alpha field stop, gamma x xi FPA, w bands,
n = gamma*xi, l = a*alpha, m = l*w; taps are the nonzeros
of the calibration images c_lambda.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CTIS_LIB_PATH") or os.path.join(_HERE, "libctis.so")  # override: experiment builds

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libctis.so not built at {LIB_PATH}: run `make` (or __graft_entry__.build()). "
                      "There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)
_i64, _P, _int = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int

_SIGS = {
    "ctis_plan_create": ([_i64] * 5 + [_P, _P, _P, _int, _P], _int),
    "ctis_plan_create_shard": ([_i64] * 5 + [_P, _P, _P, _i64, _i64, _int, _P], _int),
    "ctis_plan_destroy": ([_P], None),
    "ctis_plan_dims": ([_P, _P], _int),
    "ctis_plan_info": ([_P, _P], _int),
    "ctis_set_option": ([_P, _int, _i64], _int),
    "ctis_workspace_bytes": ([_P, _i64], ctypes.c_size_t),
    "ctis_forward": ([_P, _P, _P, _P], _int),
    "ctis_forward_batched": ([_P, _P, _P, _i64, _P], _int),
    "ctis_forward_accumulate": ([_P, _P, _P, _i64, _P], _int),
    "ctis_backproject": ([_P, _P, _P, _P], _int),
    "ctis_sensitivity": ([_P, _P, _P], _int),
    "ctis_mlem": ([_P, _P, _P, _int, _P, _P], _int),
    "ctis_mlem_batched": ([_P, _P, _P, _i64, _int, _P, _P], _int),
    "ctis_smart": ([_P, _P, _P, _i64, _int, _P, _P], _int),
    "ctis_mlem_monitored": ([_P, _P, _P, _int, ctypes.c_double, _P, _P, _P, _P], _int),
    "ctis_back_update_from_ghat": ([_P, _P, _P, _P, _P, _P], _int),
    "ctis_forward_ratio": ([_P, _P, _P, _P, _P], _int),
    "ctis_back_update": ([_P, _P, _P, _P], _int),
    "ctis_mlem_host": ([_P, _P, _P, _i64, _int, _P], _int),
    "ctis_comm_unique_id": ([_P], _int),
    "ctis_comm_create": ([_int, _int, _P, _int, _P], _int),
    "ctis_comm_destroy": ([_P], None),
    "ctis_band_sharded_workspace_bytes": ([_P, _P], ctypes.c_size_t),
    "ctis_mlem_band_sharded": ([_P, _P, _P, _P, _int, _P, _P], _int),
    "ctis_last_launch_count": ([_P], _i64),
    "ctis_last_error": ([], ctypes.c_char_p),
    "ctis_version": ([], ctypes.c_char_p),
}
for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res

EXPORTED = tuple(_SIGS)

# status codes (include/ctis.h)
OK, ERR_INVALID_ARGUMENT, ERR_DIMENSION, ERR_TAP, ERR_ZERO_SENSITIVITY, ERR_DATA, ERR_CUDA, \
    ERR_OUT_OF_MEMORY, ERR_UNSUPPORTED = range(9)
OPT_VALIDATE_DATA, OPT_USE_GRAPH, OPT_PROJECTOR, OPT_FUSED_RATIO, OPT_EXCHANGE = 1, 2, 3, 4, 5


def comm_unique_id() -> bytes:
    """128-byte NCCL unique id (ctis_comm_unique_id) for Comm(); create on one rank, broadcast to all."""
    buf = (ctypes.c_uint8 * 128)()
    _check(_lib.ctis_comm_unique_id(buf), "ctis_comm_unique_id")
    return bytes(buf)


class Comm:
    """NCCL communicator owned by libctis (ctis_comm_create): the latency mode's exchange."""

    def __init__(self, nranks: int, rank: int, uid: bytes, device: int = 0):
        if len(uid) != 128:
            raise ValueError("uid must be 128 bytes")
        self._h = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        _check(_lib.ctis_comm_create(int(nranks), int(rank), buf, int(device), ctypes.byref(self._h)),
               "ctis_comm_create")
        self.nranks, self.rank, self.device = int(nranks), int(rank), int(device)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.ctis_comm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CtisError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.ctis_last_error().decode(errors="replace")
        super().__init__(f"{where}: ctis status {status}: {msg}")


def _check(status: int, where: str):
    if status != OK:
        raise CtisError(status, where)


def version() -> str:
    return _lib.ctis_version().decode()


def _stream_handle(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _dev_ptr(t, numel: int, what: str):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
        raise TypeError(f"{what}: expected a float32 CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{what}: tensor must be contiguous")
    if t.numel() != numel:
        raise ValueError(f"{what}: expected {numel} elements, got {t.numel()}")
    return ctypes.c_void_p(t.data_ptr())


class Plan:
    """A calibrated CTIS operator H on one CUDA device (ctis_plan_create / _shard).

    taps: CSR arrays (tap_ptr int64 (w+1), tap_offset int64, tap_weight float32),
    or any object with .ptr/.offset/.weight.  band_range=(b0, b1) builds a
    latency-mode shard plan holding only bands [b0, b1).
    """

    def __init__(self, a: int, alpha: int, w: int, gamma: int, xi: int, taps=None, *,
                 tap_ptr=None, tap_offset=None, tap_weight=None, device: int = 0,
                 band_range: Optional[tuple] = None):
        if taps is not None:
            tap_ptr, tap_offset, tap_weight = taps.ptr, taps.offset, taps.weight
        self._ptr = np.ascontiguousarray(tap_ptr, np.int64)
        self._off = np.ascontiguousarray(tap_offset, np.int64)
        self._wt = np.ascontiguousarray(tap_weight, np.float32)
        self._h = ctypes.c_void_p()
        args = [int(a), int(alpha), int(w), int(gamma), int(xi),
                self._ptr.ctypes.data_as(_P), self._off.ctypes.data_as(_P), self._wt.ctypes.data_as(_P)]
        if band_range is None:
            _check(_lib.ctis_plan_create(*args, int(device), ctypes.byref(self._h)), "ctis_plan_create")
        else:
            b0, b1 = band_range
            _check(_lib.ctis_plan_create_shard(*args, int(b0), int(b1), int(device), ctypes.byref(self._h)),
                   "ctis_plan_create_shard")
        dims = (ctypes.c_int64 * 10)()
        _check(_lib.ctis_plan_dims(self._h, dims), "ctis_plan_dims")
        (self.a, self.alpha, self.w, self.gamma, self.xi, self.n, self.m,
         self.band_begin, self.band_end, self.total_taps) = [int(v) for v in dims]
        self.w_total = int(w)
        self.device = int(device)
        self._ws = None

    @classmethod
    def from_geometry(cls, geom, taps, device: int = 0, band_range=None) -> "Plan":
        return cls(geom.a, geom.alpha, geom.w, geom.gamma, geom.xi, taps, device=device, band_range=band_range)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.ctis_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        """Plan layout (ctis_plan_info): tap pages, chunks, kernel family choices."""
        v = (ctypes.c_int64 * 10)()
        _check(_lib.ctis_plan_info(self._h, v), "ctis_plan_info")
        keys = ("fwd_pages", "back_pages", "fwd_chunks", "back_chunks", "tma_f", "tma_b", "back_nb", "back_tc",
                "fwd_maxm", "fwd_items")
        return dict(zip(keys, (int(x) for x in v)))

    def set_option(self, option: int, value: int):
        _check(_lib.ctis_set_option(self._h, int(option), int(value)), "ctis_set_option")

    def last_launch_count(self) -> int:
        return int(_lib.ctis_last_launch_count(self._h))

    def workspace(self, frames: int = 1):
        import torch
        nbytes = int(_lib.ctis_workspace_bytes(self._h, int(frames)))
        if self._ws is None or self._ws.numel() * 4 < nbytes:
            self._ws = torch.empty(nbytes // 4, dtype=torch.float32, device=f"cuda:{self.device}")
        return self._ws

    # ---- stream-ordered operators on torch CUDA tensors -------------------------------
    def forward(self, f, out=None, stream=None):
        """g_hat = H f (Eq. 12); f: m floats -> n floats."""
        import torch
        frames = f.numel() // self.m if f.numel() > self.m else 1
        if out is None:
            out = torch.empty((frames, self.n) if frames > 1 else (self.n,), dtype=torch.float32, device=f.device)
        fp = _dev_ptr(f, self.m * frames, "f")
        gp = _dev_ptr(out, self.n * frames, "g_hat")
        _check(_lib.ctis_forward_batched(self._h, fp, gp, frames, _stream_handle(stream)), "ctis_forward")
        return out

    def forward_accumulate(self, f, out, stream=None):
        """g_hat += H f (no clearing; the forward kernels accumulate with red.add)."""
        frames = f.numel() // self.m
        _check(_lib.ctis_forward_accumulate(self._h, _dev_ptr(f, self.m * frames, "f"),
                                            _dev_ptr(out, self.n * frames, "g_hat"), frames,
                                            _stream_handle(stream)), "ctis_forward_accumulate")
        return out

    def backproject(self, r, out=None, stream=None):
        """z = H^T r (Eqs. 14-15); r: n floats -> m floats."""
        import torch
        if out is None:
            out = torch.empty(self.m, dtype=torch.float32, device=r.device)
        _check(_lib.ctis_backproject(self._h, _dev_ptr(r, self.n, "r"), _dev_ptr(out, self.m, "z"),
                                     _stream_handle(stream)), "ctis_backproject")
        return out

    def sensitivity(self, out=None, stream=None):
        """h = H^T 1, m floats."""
        import torch
        if out is None:
            out = torch.empty(self.m, dtype=torch.float32, device=f"cuda:{self.device}")
        _check(_lib.ctis_sensitivity(self._h, _dev_ptr(out, self.m, "h"), _stream_handle(stream)),
               "ctis_sensitivity")
        return out

    def mlem(self, g, f, iters: int, ws=None, stream=None):
        """In-place MLEM (Eq. 2, Alg. 1): f <- f^(iters+1).  Batched when g is [F, n]."""
        frames = g.numel() // self.n
        ws = self.workspace(frames) if ws is None else ws
        gp = _dev_ptr(g, self.n * frames, "g")
        fp = _dev_ptr(f, self.m * frames, "f")
        if frames == 1:
            _check(_lib.ctis_mlem(self._h, gp, fp, int(iters), ctypes.c_void_p(ws.data_ptr()),
                                  _stream_handle(stream)), "ctis_mlem")
        else:
            _check(_lib.ctis_mlem_batched(self._h, gp, fp, frames, int(iters), ctypes.c_void_p(ws.data_ptr()),
                                          _stream_handle(stream)), "ctis_mlem_batched")
        return f

    def smart(self, g, f, iters: int, ws=None, stream=None):
        """In-place SMART (simultaneous MART, ctis_smart): f <- f exp(H^T log(g / Hf) / h), `iters` times."""
        frames = g.numel() // self.n
        ws = self.workspace(frames) if ws is None else ws
        _check(_lib.ctis_smart(self._h, _dev_ptr(g, self.n * frames, "g"), _dev_ptr(f, self.m * frames, "f"), frames,
                               int(iters), ctypes.c_void_p(ws.data_ptr()), _stream_handle(stream)), "ctis_smart")
        return f

    def mlem_monitored(self, g, f, max_iters: int, rel_tol: float = 0.0, ws=None, stream=None):
        """In-place MLEM with the per-iteration Poisson log-likelihood and the early stop
        (ctis_mlem_monitored; R15/R16).  Returns (ll, iters_done) as device tensors:
        ll float64[max_iters] (L_k of f^(k); zero past iters_done), iters_done int32[1]."""
        import torch
        ws = self.workspace(1) if ws is None else ws
        dev = f.device
        ll = torch.empty(max(int(max_iters), 1), dtype=torch.float64, device=dev)
        done = torch.empty(1, dtype=torch.int32, device=dev)
        _check(_lib.ctis_mlem_monitored(self._h, _dev_ptr(g, self.n, "g"), _dev_ptr(f, self.m, "f"), int(max_iters),
                                        float(rel_tol), ctypes.c_void_p(ws.data_ptr()),
                                        ctypes.c_void_p(ll.data_ptr()), ctypes.c_void_p(done.data_ptr()),
                                        _stream_handle(stream)), "ctis_mlem_monitored")
        return ll, done

    def forward_ratio(self, f, g, r, stream=None):
        """r = g (/) (H f) (Alg. 1 lines 6-8, one fused kernel)."""
        _check(_lib.ctis_forward_ratio(self._h, _dev_ptr(f, self.m, "f"), _dev_ptr(g, self.n, "g"),
                                       _dev_ptr(r, self.n, "r"), _stream_handle(stream)), "ctis_forward_ratio")
        return r

    def back_update(self, r, f, stream=None):
        """f <- f (.) (H^T r) (/) h in place (Alg. 1 lines 9-12, one fused kernel)."""
        _check(_lib.ctis_back_update(self._h, _dev_ptr(r, self.n, "r"), _dev_ptr(f, self.m, "f"),
                                     _stream_handle(stream)), "ctis_back_update")
        return f

    def band_sharded_workspace(self, comm: "Comm"):
        import torch
        nbytes = int(_lib.ctis_band_sharded_workspace_bytes(self._h, comm._h))
        return torch.empty(nbytes // 4, dtype=torch.float32, device=f"cuda:{self.device}")

    def mlem_band_sharded(self, comm: "Comm", g, f_local, iters: int, ws=None, stream=None):
        """Latency mode (ctis_mlem_band_sharded): `iters` iterations of partial forward -> NCCL
        reduce-scatter -> ratio on this rank's slice -> all-gather -> back update, as one CUDA graph.
        Collective over `comm`; g: full n floats; f_local: this shard's m floats, in place."""
        ws = self.band_sharded_workspace(comm) if ws is None else ws
        _check(_lib.ctis_mlem_band_sharded(self._h, comm._h, _dev_ptr(g, self.n, "g"), _dev_ptr(f_local, self.m, "f"),
                                           int(iters), ctypes.c_void_p(ws.data_ptr()), _stream_handle(stream)),
               "ctis_mlem_band_sharded")
        return f_local

    def back_update_from_ghat(self, g, g_hat, f, ws=None, stream=None):
        """Latency mode: r = g/g_hat (all-reduced), f_shard <- f_shard (.) H_shard^T r (/) h."""
        ws = self.workspace(1) if ws is None else ws
        _check(_lib.ctis_back_update_from_ghat(self._h, _dev_ptr(g, self.n, "g"), _dev_ptr(g_hat, self.n, "g_hat"),
                                               _dev_ptr(f, self.m, "f"), ctypes.c_void_p(ws.data_ptr()),
                                               _stream_handle(stream)), "ctis_back_update_from_ghat")
        return f

    def mlem_host(self, g_host: np.ndarray, f_host: np.ndarray, iters: int, stream=None) -> np.ndarray:
        """End-to-end on HOST arrays (ctis_mlem_host): H2D, iterations, D2H, synchronise."""
        g_host = np.ascontiguousarray(g_host, np.float32)
        if not (f_host.flags.c_contiguous and f_host.dtype == np.float32):
            raise ValueError("f_host must be a contiguous float32 array (updated in place)")
        frames = g_host.size // self.n
        assert g_host.size == frames * self.n and f_host.size == frames * self.m
        _check(_lib.ctis_mlem_host(self._h, g_host.ctypes.data_as(_P), f_host.ctypes.data_as(_P), frames,
                                   int(iters), _stream_handle(stream)), "ctis_mlem_host")
        return f_host

    def mlem_host_ptr(self, g_ptr: int, f_ptr: int, frames: int, iters: int, stream=None):
        """ctis_mlem_host on raw host pointers (e.g. pinned torch CPU tensors)."""
        _check(_lib.ctis_mlem_host(self._h, ctypes.c_void_p(g_ptr), ctypes.c_void_p(f_ptr), int(frames),
                                   int(iters), _stream_handle(stream)), "ctis_mlem_host")


__all__ = ["Plan", "CtisError", "version", "LIB_PATH", "EXPORTED"]
