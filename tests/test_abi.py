"""The C-ABI library loads on CPU and exports every symbol include/ctis.h declares (no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ctis.h")
LIB = os.path.join(ROOT, "paper_2006_01573_b200", "libctis.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-C", ROOT, "-j4", "all"])
    return ctypes.CDLL(LIB)


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"CTIS_API\s+[\w\s\*]+?\b(ctis_\w+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    syms = declared_symbols()
    for need in ("ctis_plan_create", "ctis_forward", "ctis_backproject", "ctis_sensitivity", "ctis_mlem",
                 "ctis_mlem_batched", "ctis_plan_create_shard", "ctis_back_update_from_ghat"):
        assert need in syms


def test_library_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (ctis_\w+)", out))
    assert set(syms) == exported, (set(syms) ^ exported)


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    assert not re.search(r"sm_(?!100a)\d+", out.stdout)


def test_python_binding_loads_and_wraps_all_symbols():
    import paper_2006_01573_b200 as ctis
    assert set(ctis.EXPORTED) == set(declared_symbols())
    assert "sm_100a" in ctis.version()


def test_host_side_errors_without_gpu(lib):
    """Argument validation runs before any device call, so it works on a CPU-only box."""
    import numpy as np
    lib.ctis_plan_create.restype = ctypes.c_int
    lib.ctis_last_error.restype = ctypes.c_char_p
    P = ctypes.c_void_p
    ptr = np.array([0, 1], np.int64)
    off = np.array([5], np.int64)
    wt = np.array([1.0], np.float32)
    out = ctypes.c_void_p()
    args = lambda a, al, w, ga, xi, o=off, ww=wt: [ctypes.c_int64(v) for v in (a, al, w, ga, xi)] + [
        ptr.ctypes.data_as(P), o.ctypes.data_as(P), ww.ctypes.data_as(P), ctypes.c_int(0), ctypes.byref(out)]
    assert lib.ctis_plan_create(*args(4, 4, 1, 3, 4)) == 2            # gamma < a
    assert lib.ctis_plan_create(*args(0, 4, 1, 3, 4)) == 2
    assert lib.ctis_plan_create(*args(2, 2, 1, 4, 4, o=np.array([16], np.int64))) == 3   # offset >= n
    assert lib.ctis_plan_create(*args(2, 2, 1, 4, 4, ww=np.array([0.0], np.float32))) == 3
    assert b"weight" in lib.ctis_last_error()
    lib.ctis_forward.restype = ctypes.c_int
    assert lib.ctis_forward(None, None, None, None) == 1
