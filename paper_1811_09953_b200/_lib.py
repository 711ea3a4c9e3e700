"""ctypes binding of libfcn.so -- the C ABI declared in include/fcn.h.

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a).
There is no CPU fallback: if the library or a CUDA device is missing, every
compute call raises `FcnUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FCN_LIB_PATH") or os.path.join(HERE, "libfcn.so")

FCN_OK = 0
FCN_ERR_ARG = -1
FCN_ERR_PARAM = -2
FCN_ERR_CUDA = -3
FCN_ERR_STATE = -4

OP_ADD, OP_SUB, OP_NEG, OP_MUL = 0, 1, 2, 3


class FcnUnavailable(RuntimeError):
    """The native GPU library (or a CUDA device) is not available."""


class FcnError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libfcn error {code}: {msg}")
        self.code = code
        self.msg = msg


_P = C.c_void_p
_U64P = C.POINTER(C.c_uint64)
_I64 = C.c_int64
_I = C.c_int

# name -> (restype, argtypes)
SIGNATURES = {
    "fcn_last_error": (C.c_char_p, []),
    "fcn_version": (_I, []),
    "fcn_launch_count": (C.c_longlong, []),
    "fcn_stage_timing": (_I, [_I]),
    "fcn_stage_times": (_I, [C.POINTER(C.c_double), _I]),
    "fcn_ntt_f64_schedule": (_I, [_I, C.c_uint64]),
    "fcn_ring_create": (_I, [_I, _I, _I, _U64P, C.POINTER(_P)]),
    "fcn_ring_destroy": (_I, [_P]),
    "fcn_ring_roots": (_I, [_P, _U64P]),
    "fcn_ntt_forward": (_I, [_P, _P, _I64, _I, _I, _P]),
    "fcn_ntt_inverse": (_I, [_P, _P, _I64, _I, _I, _P]),
    "fcn_poly_binary": (_I, [_P, _I, _P, _P, _I64, _P, _I64, _I, _I, _P]),
    "fcn_lift_signed": (_I, [_P, _P, _I64, _P, _I, _I, _P]),
    "fcn_scalar_mul": (_I, [_P, _P, _U64P, _P, _I64, _I, _I, _P]),
    "fcn_poly_mul_monomial": (_I, [_P, _P, _I, _U64P, _P, _I64, _I, _I, _P]),
    "fcn_ctx_create": (_I, [_I, _I, _I, _U64P, _I, _U64P, _I, C.POINTER(_P)]),
    "fcn_ctx_destroy": (_I, [_P]),
    "fcn_ctx_ring": (_I, [_P, C.POINTER(_P)]),
    "fcn_ctx_query": (_I, [_P, _I, C.POINTER(_I64)]),
    "fcn_ctx_aux_primes": (_I, [_P, _U64P]),
    "fcn_ctx_fallback_count": (_I, [_P, C.POINTER(_I64)]),
    "fcn_keys_create": (_I, [_P, _U64P, _U64P, C.POINTER(_P)]),
    "fcn_keys_destroy": (_I, [_P]),
    "fcn_add_plain_terms": (_I, [_P, _I, _P, _I64, _P, _P, _P, _P]),
    "fcn_linear_mac": (_I, [_P, _P, _I64, _P, _I64, _P, _P, _P, _P, _P, _I64, _P]),
    "fcn_linear_mac_ex": (_I, [_P, _P, _I64, _P, _I64, _P, _P, _P, _P, _P, _I64, _I, C.c_uint64, _P]),
    "fcn_linear_mac_multi": (_I, [_P, _P, _I64, _P, _I64, _P, _P, _P, _P, _P, _I, _I64, _I, C.c_uint64, _P]),
    "fcn_tc_planes": (_I, [_P]),
    "fcn_tc_planes_bytes": (C.c_size_t, [_P, _I64]),
    "fcn_split_planes": (_I, [_P, _P, _I64, _P, _P]),
    "fcn_linear_mac_tc": (_I, [_P, _P, _I64, _I64, _P, _P, _P, _P, _P, _I, _I64, _I64, _P]),
    "fcn_mul_ct_workspace_bytes": (C.c_size_t, [_P, _I64]),
    "fcn_mul_ct": (_I, [_P, _P, _I, _P, _P, _P, _I64, _P, C.c_size_t, _P]),
    "fcn_mul_ct_ex": (_I, [_P, _P, _I, _P, _P, _P, _I64, _I, _I64, _I64, _P, C.c_size_t, _P]),
    "fcn_key_mac": (_I, [_P, _P, _P, _P, _I64, _P]),
    "fcn_mul_ct_multi": (_I, [_P, _P, _I, _P, _P, _P, _I, _I64, _I, _I64, _I64, _P, C.c_size_t, _P]),
    "fcn_noise_max": (_I, [_P, _I, _P, _I64, _P, _I, _I, _P]),
    "fcn_decrypt_round": (_I, [_P, _I, _P, _P, _I64, _P]),
}

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load and type the library (no CUDA context is created here)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise FcnUnavailable(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load()


def check(rc: int, exc_type=None):
    if rc == FCN_OK:
        return
    msg = lib().fcn_last_error().decode(errors="replace")
    if exc_type is not None and rc in (FCN_ERR_ARG, FCN_ERR_PARAM):
        raise exc_type(msg)
    raise FcnError(rc, msg)


def ptr_array(ptrs):
    """Host array of device pointers (uint64_t* const*) for the fan-out entry points."""
    arr = (C.c_void_p * len(ptrs))(*[int(p) for p in ptrs])
    return arr


def u64_array(values):
    vals = [int(v) for v in values]
    arr = (C.c_uint64 * max(1, len(vals)))(*vals)
    return arr
