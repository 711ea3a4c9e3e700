"""The reference-side binding of INTEGRATION.md (Option B,
integration/hecnet_gpu.py): its ctypes declarations agree with
include/fcn.h (CPU), and bound into the reference package itself it
reproduces `hecnet.fv.mul_ct`, the engine's activation chain and
`hecnet.ring.ntt_forward/inverse` byte for byte (GPU; needs the reference
installed in baseline/_ref, which travels with the repo snapshot)."""

import ctypes as C
import os
import re
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "integration"))

import hecnet_gpu  # noqa: E402

from paper_1811_09953_b200 import _lib  # noqa: E402


def _header_params():
    """fcn.h function name -> number of parameters."""
    src = open(os.path.join(REPO, "include", "fcn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(fcn_[a-z0-9_]+)\s*\(([^)]*)\)\s*;", src):
        args = m.group(2).strip()
        out[m.group(1)] = 0 if args in ("", "void") else len(args.split(","))
    return out


def _ctype_name(t):
    return getattr(t, "__name__", repr(t))


def test_stub_bindings_match_header_and_library_signatures():
    hdr = _header_params()
    for name, (res, args) in hecnet_gpu.BINDINGS.items():
        assert name in hdr, f"{name} is not declared in include/fcn.h"
        assert len(args) == hdr[name], f"{name}: {len(args)} argtypes vs {hdr[name]} parameters in fcn.h"
        lres, largs = _lib.SIGNATURES[name]
        assert [_ctype_name(a) for a in args] == [_ctype_name(a) for a in largs], name
        assert _ctype_name(res) == _ctype_name(lres), name


def test_stub_library_symbols():
    if not os.path.exists(hecnet_gpu.LIB_PATH):
        pytest.skip("libfcn.so not built")
    L = hecnet_gpu.lib()
    for name in hecnet_gpu.BINDINGS:
        assert hasattr(L, name)
    out = C.c_void_p()
    assert L.fcn_ring_create(0, 1000, 1, hecnet_gpu._u64([17]), C.byref(out)) == _lib.FCN_ERR_PARAM


def _hecnet():
    ref = os.path.join(REPO, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        from hecnet import fv, modmath, ring
    except Exception:  # noqa: BLE001
        pytest.skip("reference package not installed in baseline/_ref")
    return fv, ring, modmath


@pytest.mark.gpu
@pytest.mark.parametrize("k,bits", [(4, 50), (2, 55)])
def test_stub_mul_ct_matches_reference(k, bits):
    """k=4 x 50-bit: the FP64 square pipeline (k=4 / K=9); k=2 x 55-bit: the
    integer kernels.  Reference keys and ciphertexts, reference result."""
    fv, ring, mm = _hecnet()
    n = 1024
    primes = tuple(mm.find_ntt_primes(n, k, bits=bits))
    params = fv.EncryptionParams(n, primes, (65537,), 1 << 32)
    sk, pk, ek = fv.keygen(params, 11)
    rng = np.random.default_rng(3)
    gp = hecnet_gpu.GpuParams(fv, params, ek)
    try:
        cts = []
        for i in range(3):
            m = fv.PlainPoly(65537, rng.integers(0, 65537, n).astype(np.uint64))
            cts.append(fv.encrypt(pk, params, m, 0, 6, rng))
        for a, b in ((cts[0], cts[0]), (cts[1], cts[2])):
            want = fv.mul_ct(a, b, ek)
            got = hecnet_gpu.mul_ct(fv, ring, a, b, gp)
            assert np.array_equal(got.c0.data, want.c0.data) and np.array_equal(got.c1.data, want.c1.data)
            assert (got.scale_exponent, got.mul_depth, got.lane) == (want.scale_exponent, want.mul_depth, want.lane)
        # the activation 2^-3 x^2 + 2^-1 x at prec 6: a2 = 8, a1 = 2^17 (engine.py:744-770)
        x, prec, a2, a1 = cts[0], 6, 8, 1 << 17
        sq = fv.mul_ct(x, x, ek)
        acc = fv.mul_pt(sq, fv.PlainPoly(65537, np.array([a2], dtype=np.uint64)), prec)
        lin = fv.mul_pt(x, fv.PlainPoly(65537, np.array([a1 % 65537], dtype=np.uint64)),
                        acc.scale_exponent - x.scale_exponent)
        want = fv.add_ct(acc, lin)
        got = hecnet_gpu.act_square(fv, ring, x, a2, a1 % 65537, prec, gp)
        assert np.array_equal(got.c0.data, want.c0.data) and np.array_equal(got.c1.data, want.c1.data)
        assert (got.scale_exponent, got.mul_depth) == (want.scale_exponent, want.mul_depth)
    finally:
        gp.close()


@pytest.mark.gpu
def test_stub_ntt_matches_reference():
    fv, ring, mm = _hecnet()
    for n, bits, k in ((1024, 50, 4), (4096, 36, 3), (16384, 50, 2)):
        ctx = ring.RingContext.create(n, tuple(mm.find_ntt_primes(n, k, bits=bits)))
        p = ring.RingPoly.random_uniform(ctx, np.random.default_rng(n))
        g = hecnet_gpu.GpuRing(ring, ctx)
        try:
            f = g.ntt_forward(p)
            want = ring.ntt_forward(p)
            assert f.domain == want.domain and np.array_equal(f.data, want.data)
            back = g.ntt_inverse(f)
            assert np.array_equal(back.data, p.data) and back.domain == ring.COEFF
        finally:
            g.close()
