"""Reference-side binding of libfcn (Option B).

This is the module a `hecnet` maintainer would add as `hecnet/_gpu.py`: a
ctypes binding of the C ABI in `include/fcn.h` that takes and returns the
reference's own objects (`fv.Ciphertext`, `ring.RingPoly`), so that
`fv.mul_ct` (reference fv.py:498-549), the engine's activation
(engine.py:744-770) and `ring.ntt_forward` / `ntt_inverse`
(ring.py:242-255) can be dispatched to the GPU without touching the rest of
the package.  It imports nothing from `paper_1811_09953_b200`: only numpy,
torch (device buffers and the stream) and the reference passed in.

`tests/test_integration_stub.py` checks every argtypes list here against
`include/fcn.h` (CPU) and runs the stub on the reference's own keys and
ciphertexts against `hecnet.fv.mul_ct` byte for byte (GPU).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FCN_LIB_PATH") or os.path.join(_HERE, "..", "paper_1811_09953_b200", "libfcn.so")

P, U64P = C.c_void_p, C.POINTER(C.c_uint64)
FCN_MUL_ACT = 1

# name -> (restype, argtypes): what the reference binds
BINDINGS = {
    "fcn_last_error": (C.c_char_p, []),
    "fcn_ring_create": (C.c_int, [C.c_int, C.c_int, C.c_int, U64P, C.POINTER(P)]),
    "fcn_ring_destroy": (C.c_int, [P]),
    "fcn_ntt_forward": (C.c_int, [P, P, C.c_int64, C.c_int, C.c_int, P]),
    "fcn_ntt_inverse": (C.c_int, [P, P, C.c_int64, C.c_int, C.c_int, P]),
    "fcn_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, U64P, C.c_int, U64P, C.c_int, C.POINTER(P)]),
    "fcn_ctx_destroy": (C.c_int, [P]),
    "fcn_keys_create": (C.c_int, [P, U64P, U64P, C.POINTER(P)]),
    "fcn_keys_destroy": (C.c_int, [P]),
    "fcn_mul_ct_workspace_bytes": (C.c_size_t, [P, C.c_int64]),
    "fcn_mul_ct": (C.c_int, [P, P, C.c_int, P, P, P, C.c_int64, P, C.c_size_t, P]),
    "fcn_mul_ct_ex": (C.c_int, [P, P, C.c_int, P, P, P, C.c_int64, C.c_int, C.c_int64, C.c_int64, P, C.c_size_t, P]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in BINDINGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _u64(v):
    v = [int(x) for x in v]
    return (C.c_uint64 * len(v))(*v)


def _check(rc, exc):
    if rc:
        raise exc(lib().fcn_last_error().decode(errors="replace"))


def _stream():
    import torch

    return torch.cuda.current_stream().cuda_stream


class GpuParams:
    """libfcn context + device eval keys for one reference EncryptionParams."""

    def __init__(self, fv, params, ek, device: int = 0):
        self.fv = fv
        L = lib()
        self.ctx = P()
        _check(L.fcn_ctx_create(device, params.n, len(params.limb_primes), _u64(params.limb_primes),
                                len(params.t_lanes), _u64(params.t_lanes), params.beta.bit_length() - 1,
                                C.byref(self.ctx)), fv.FVError)
        a = np.ascontiguousarray(np.stack([x.data for x in ek.a]))  # [ell+1][k][n], coefficient domain
        g = np.ascontiguousarray(np.stack([x.data for x in ek.g]))
        self.keys = P()
        _check(L.fcn_keys_create(self.ctx, a.ctypes.data_as(U64P), g.ctypes.data_as(U64P), C.byref(self.keys)),
               fv.FVError)

    def close(self):
        L = lib()
        if self.keys:
            L.fcn_keys_destroy(self.keys)
            self.keys = P()
        if self.ctx:
            L.fcn_ctx_destroy(self.ctx)
            self.ctx = P()


def _dev(c):
    import torch

    return torch.from_numpy(np.stack([c.c0.data, c.c1.data])[None].view(np.int64)).cuda()


def _ct_from(fv, ring, ref, body, scale, depth):
    return fv.Ciphertext(ring.RingPoly(ref.params.ctx, body[0].copy()), ring.RingPoly(ref.params.ctx, body[1].copy()),
                         ref.params, ref.lane, scale, depth)


def mul_ct(fv, ring, a, b, gp: GpuParams):
    """Drop-in for fv.mul_ct(a, b, ek) (fv.py:498-549) on the GPU."""
    import torch

    fv._check_compat(a, b, require_scale=False)
    A = _dev(a)
    B = None if b is a else _dev(b)
    out = torch.empty_like(A)
    L = lib()
    ws = torch.empty(L.fcn_mul_ct_workspace_bytes(gp.ctx, 1) // 8 + 1, dtype=torch.int64, device="cuda")
    _check(L.fcn_mul_ct(gp.ctx, gp.keys, a.lane, A.data_ptr(), None if B is None else B.data_ptr(), out.data_ptr(), 1,
                        ws.data_ptr(), ws.numel() * 8, _stream()), fv.FVError)
    o = out.cpu().numpy().view(np.uint64)[0]
    return _ct_from(fv, ring, a, o, a.scale_exponent + b.scale_exponent, max(a.mul_depth, b.mul_depth) + 1)


def act_square(fv, ring, x, c2: int, c1: int, prec: int, gp: GpuParams):
    """The activation c2 x^2 + c1 x with constant plaintexts in one call
    (engine.py:744-770 with PlainPoly(t, [c2 mod t]), PlainPoly(t, [c1 mod t]));
    metadata as the reference's chain: mul_ct -> mul_pt(prec) -> add_ct."""
    import torch

    t = int(x.params.t_lanes[x.lane])
    # the C ABI takes the centred plaintext constants (PlainPoly.centered, fv.py:162-165)
    c2, c1 = (int(c) % t for c in (c2, c1))
    c2, c1 = (c - t if c > t // 2 else c for c in (c2, c1))
    X = _dev(x)
    out = torch.empty_like(X)
    L = lib()
    ws = torch.empty(L.fcn_mul_ct_workspace_bytes(gp.ctx, 1) // 8 + 1, dtype=torch.int64, device="cuda")
    _check(L.fcn_mul_ct_ex(gp.ctx, gp.keys, x.lane, X.data_ptr(), None, out.data_ptr(), 1, FCN_MUL_ACT, c2, c1,
                           ws.data_ptr(), ws.numel() * 8, _stream()), fv.FVError)
    o = out.cpu().numpy().view(np.uint64)[0]
    return _ct_from(fv, ring, x, o, 2 * x.scale_exponent + prec, x.mul_depth + 1)


class GpuRing:
    """libfcn ring for a reference RingContext (ring.py:104-125)."""

    def __init__(self, ring, ctx, device: int = 0):
        self.ring = ring
        self.ptr = P()
        _check(lib().fcn_ring_create(device, ctx.n, len(ctx.primes), _u64(ctx.primes), C.byref(self.ptr)),
               ring.RingError)

    def _run(self, fn, p, domain):
        import torch

        d = torch.from_numpy(np.ascontiguousarray(p.data).view(np.int64)).cuda()
        _check(fn(self.ptr, d.data_ptr(), d.shape[0], d.shape[0], 0, _stream()), self.ring.RingError)
        return self.ring.RingPoly(p.ctx, d.cpu().numpy().view(np.uint64).copy(), domain)

    def ntt_forward(self, p):
        """Drop-in for ring.ntt_forward (ring.py:242-247)."""
        if p.domain != self.ring.COEFF:
            raise self.ring.RingError("ntt_forward expects a Coefficient-domain polynomial")
        return self._run(lib().fcn_ntt_forward, p, self.ring.NTT)

    def ntt_inverse(self, p):
        """Drop-in for ring.ntt_inverse (ring.py:250-255)."""
        if p.domain != self.ring.NTT:
            raise self.ring.RingError("ntt_inverse expects an NTT-domain polynomial")
        return self._run(lib().fcn_ntt_inverse, p, self.ring.COEFF)

    def close(self):
        if self.ptr:
            lib().fcn_ring_destroy(self.ptr)
            self.ptr = P()
