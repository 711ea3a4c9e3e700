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


def test_ntt_f64_schedule_bounds():
    """The FP64 NTT's reduction schedule (ntt.cu f64_schedule): every third
    stage for limbs up to 2^51, once per transform for limbs just above 2^50
    (the configs' primes), never for small limbs; recomputed here from the
    bound |t| <= (1/2 + B q 2^-53) q per butterfly."""
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libfcn.so not built")
    L = _lib.load()

    def bound(logn, rs, q):
        e, B, mx = q / 2.0**53, 1.0, 1.0
        for s in range(logn):
            if (rs == 0 and s > 0 and s % 3 == 0) or (rs == 1 and s == logn // 2):
                B = 0.5
            B = B + 0.5 + B * e
            mx = max(mx, B)
        return mx * q

    for logn in range(10, 15):
        for q in ((1 << 36) + 1, (1 << 47) + 1, (1 << 50) + 2 * (1 << logn) * 7 + 1, (1 << 51) - 1,
                  int(2.0**50.2), int(2.0**50.4), int(2.0**48.2)):
            rs = L.fcn_ntt_f64_schedule(logn, q)
            assert bound(logn, rs, q) < 2.0**53, (logn, q, rs)
            if rs < 2:  # the cheaper schedule really would overflow
                assert bound(logn, rs + 1, q) >= 2.0**53 * (1 - 1e-6), (logn, q, rs)
    assert L.fcn_ntt_f64_schedule(13, (1 << 50) + 16385) == 1
    assert L.fcn_ntt_f64_schedule(14, (1 << 36) + 1) == 2
    assert L.fcn_ntt_f64_schedule(13, (1 << 51) - 1) == 0
