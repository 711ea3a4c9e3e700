"""CPU checks of the C-ABI boundary: the library loads and exports exactly
what include/fcn.h declares (no compute calls; no GPU needed)."""

import ctypes
import os
import re

import pytest

from paper_1811_09953_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(REPO, "include", "fcn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fcn_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_bound_functions():
    decl = _declared()
    assert len(decl) >= 20
    assert sorted(_lib.SIGNATURES) == decl


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libfcn.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    L = _lib.load()
    assert L.fcn_version() == 1


def test_bad_arguments_fail_without_gpu():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libfcn.so not built")
    L = _lib.load()
    out = ctypes.c_void_p()
    # n not a power of two: rejected before any CUDA call
    rc = L.fcn_ring_create(0, 1000, 1, _lib.u64_array([17]), ctypes.byref(out))
    assert rc == _lib.FCN_ERR_PARAM
    assert b"power of two" in L.fcn_last_error()
    rc = L.fcn_ring_create(0, 1024, 1, _lib.u64_array([15]), ctypes.byref(out))
    assert rc == _lib.FCN_ERR_PARAM


def test_device_helpers_fail_loudly_without_cuda():
    import torch

    from paper_1811_09953_b200 import device

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(_lib.FcnUnavailable):
        device.require_cuda()
