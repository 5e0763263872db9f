"""The C-ABI library loads on a CPU-only host and exports every entry point
declared in include/msfv.h; plan queries work without a GPU."""

import ctypes
import os
import re

import pytest

from paper_1707_07598_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "msfv.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"MSFV_API\s+[\w\s\*]+?\b(msfv_\w+)\s*\(", txt)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert len(syms) >= 20
    assert "msfv_basis_build" in syms and "msfv_coarse_factor" in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libmsfv.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding types every declared symbol
    assert set(declared_symbols()) <= set(_lib.SIGNATURES)


def test_plan_info_without_gpu():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libmsfv.so not built")
    L = _lib.load()
    assert L.msfv_abi_version() == 2
    plan = ctypes.c_void_p()
    rc = L.msfv_plan_create((ctypes.c_int32 * 3)(128, 128, 128), (ctypes.c_double * 3)(1 / 128, 1 / 128, 1 / 128),
                            (ctypes.c_int32 * 3)(8, 8, 8), ctypes.byref(plan))
    assert rc == 0
    info = (ctypes.c_int64 * _lib.INFO_COUNT)()
    assert L.msfv_plan_info(plan, info, _lib.INFO_COUNT) == 0
    assert info[_lib.INFO_N] == 129 ** 3 - 1
    assert info[_lib.INFO_NBLOCKS] == 4096
    assert info[_lib.INFO_NI] == 343
    assert info[_lib.INFO_K] == 17 ** 3
    assert info[_lib.INFO_PC] == 17 * 17 + 17 + 1
    assert info[_lib.INFO_TC] == 1
    L.msfv_plan_destroy(plan)


def test_plan_rejects_bad_geometry():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libmsfv.so not built")
    L = _lib.load()
    plan = ctypes.c_void_p()
    rc = L.msfv_plan_create((ctypes.c_int32 * 3)(10, 8, 8), (ctypes.c_double * 3)(1, 1, 1),
                            (ctypes.c_int32 * 3)(4, 4, 4), ctypes.byref(plan))
    assert rc == _lib.MSFV_SHAPE
    assert "divide" in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)
