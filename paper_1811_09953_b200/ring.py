"""RNS ring Z_q[x]/(x^n+1) with device-resident residues (mirrors reference ring.py).

Same names, argument meaning and errors as the reference module
(`RingContext.create`, `RingPoly`, `ntt_forward` / `ntt_inverse`,
`poly_add` / `poly_sub` / `poly_neg`, `scalar_mul`, `pointwise_mul`,
`poly_mul_ntt`, `poly_mul_monomial`; reference ring.py:104-361).  A
RingPoly's `data` is a (limbs, n) CUDA tensor (int64 storage of canonical
uint64 residues); every operation runs in libfcn on the current stream.
Inputs are never mutated and every op returns a fresh polynomial.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import device as dev

SUPPORTED_DEGREES = (1024, 2048, 4096, 8192, 16384, 32768)
COEFF = "coeff"
NTT = "ntt"


class RingError(ValueError):
    """Domain or parameter mismatch between ring operands (ring.py:28)."""


@dataclass(frozen=True)
class ModulusLimb:
    q: int
    n: int
    root: int

    @property
    def qv(self):
        return np.uint64(self.q)


_handles: dict = {}


class _RingHandle:
    def __init__(self, device: int, n: int, primes: tuple):
        lib = _lib.lib()
        out = C.c_void_p()
        arr = _lib.u64_array(primes)
        _lib.check(lib.fcn_ring_create(device, n, len(primes), arr, C.byref(out)), RingError)
        self.ptr = out
        self.device = device
        roots = (C.c_uint64 * len(primes))()
        _lib.check(lib.fcn_ring_roots(out, roots))
        self.roots = tuple(int(r) for r in roots)

    def __del__(self):
        try:
            if self.ptr:
                _lib.lib().fcn_ring_destroy(self.ptr)
        except Exception:
            pass


def _ring_handle(n: int, primes: tuple) -> _RingHandle:
    d = dev.current_device()
    key = (d, n, primes)
    h = _handles.get(key)
    if h is None:
        h = _RingHandle(d, n, primes)
        _handles[key] = h
    return h


@dataclass(frozen=True)
class RingContext:
    n: int
    primes: tuple

    @staticmethod
    def create(n: int, primes) -> "RingContext":
        n = int(n)
        if n < 4 or n & (n - 1):
            raise RingError(f"ring degree {n} is not a power of two")
        primes = tuple(int(q) for q in primes)
        ctx = RingContext(n, primes)
        ctx.handle()  # validates primes (prime, < 2^62, = 1 mod 2n) in libfcn
        return ctx

    def handle(self) -> _RingHandle:
        return _ring_handle(self.n, self.primes)

    @property
    def limbs(self):
        roots = self.handle().roots
        return tuple(ModulusLimb(q, self.n, r) for q, r in zip(self.primes, roots))

    @property
    def modulus(self) -> int:
        q = 1
        for p in self.primes:
            q *= p
        return q


class RingPoly:
    """Element of R_q in RNS form; data: (limbs, n) device tensor."""

    __slots__ = ("ctx", "data", "domain")

    def __init__(self, ctx: RingContext, data, domain: str = COEFF):
        if isinstance(data, np.ndarray):
            if data.dtype != np.uint64:
                raise RingError("coefficients must be uint64")
            data = dev.to_device(data)
        if tuple(data.shape) != (len(ctx.primes), ctx.n):
            raise RingError(f"coefficient block {tuple(data.shape)} does not match ({len(ctx.primes)}, {ctx.n})")
        object.__setattr__(self, "ctx", ctx)
        object.__setattr__(self, "data", data)
        object.__setattr__(self, "domain", domain)

    def __setattr__(self, k, v):
        raise AttributeError("RingPoly is immutable")

    @staticmethod
    def zero(ctx: RingContext, domain: str = COEFF) -> "RingPoly":
        return RingPoly(ctx, dev.zeros((len(ctx.primes), ctx.n)), domain)

    @staticmethod
    def from_int_coeffs(ctx: RingContext, coeffs) -> "RingPoly":
        coeffs = [int(c) for c in coeffs]
        if len(coeffs) > ctx.n:
            raise RingError(f"{len(coeffs)} coefficients exceed degree {ctx.n}")
        rows = np.zeros((len(ctx.primes), ctx.n), dtype=np.uint64)
        for i, q in enumerate(ctx.primes):
            rows[i, : len(coeffs)] = [c % q for c in coeffs]
        return RingPoly(ctx, rows, COEFF)

    @staticmethod
    def random_uniform(ctx: RingContext, rng: np.random.Generator) -> "RingPoly":
        """Same draws as the reference (ring.py:171-175): one integers() call per limb."""
        rows = np.stack([rng.integers(0, q, ctx.n, dtype=np.uint64) for q in ctx.primes])
        return RingPoly(ctx, rows, COEFF)

    def host(self) -> np.ndarray:
        return dev.to_host(self.data)

    def is_zero(self) -> bool:
        return not bool(self.data.any())

    def __eq__(self, other) -> bool:
        if not isinstance(other, RingPoly):
            return False
        return (
            self.domain == other.domain
            and self.ctx.primes == other.ctx.primes
            and self.ctx.n == other.ctx.n
            and bool((self.data == other.data).all())
        )

    def __hash__(self):
        return id(self)


def _check_pair(a: RingPoly, b: RingPoly, same_domain: bool = True) -> None:
    if a.ctx.n != b.ctx.n or a.ctx.primes != b.ctx.primes:
        raise RingError("ring parameter mismatch between operands")
    if same_domain and a.domain != b.domain:
        raise RingError(f"domain mismatch: {a.domain} vs {b.domain}")


def _rows(p: RingPoly):
    return len(p.ctx.primes)


def ntt_forward(p: RingPoly) -> RingPoly:
    """Negacyclic NTT per limb, bit-reversed output (ring.py:242-247)."""
    if p.domain != COEFF:
        raise RingError("ntt_forward expects a Coefficient-domain polynomial")
    out = p.data.clone()
    L = _rows(p)
    _lib.check(_lib.lib().fcn_ntt_forward(p.ctx.handle().ptr, out.data_ptr(), L, L, 0, dev.stream_ptr()), RingError)
    return RingPoly(p.ctx, out, NTT)


def ntt_inverse(p: RingPoly) -> RingPoly:
    """Inverse transform, exact round trip (ring.py:250-255)."""
    if p.domain != NTT:
        raise RingError("ntt_inverse expects an NTT-domain polynomial")
    out = p.data.clone()
    L = _rows(p)
    _lib.check(_lib.lib().fcn_ntt_inverse(p.ctx.handle().ptr, out.data_ptr(), L, L, 0, dev.stream_ptr()), RingError)
    return RingPoly(p.ctx, out, COEFF)


def _binary(op: int, a: RingPoly, b: RingPoly | None, domain: str) -> RingPoly:
    out = dev.empty(a.data.shape)
    L = _rows(a)
    bp = b.data.data_ptr() if b is not None else None
    _lib.check(
        _lib.lib().fcn_poly_binary(a.ctx.handle().ptr, op, a.data.data_ptr(), bp, L, out.data_ptr(), L, L, 0, dev.stream_ptr()),
        RingError,
    )
    return RingPoly(a.ctx, out, domain)


def poly_add(a: RingPoly, b: RingPoly) -> RingPoly:
    _check_pair(a, b)
    return _binary(_lib.OP_ADD, a, b, a.domain)


def poly_sub(a: RingPoly, b: RingPoly) -> RingPoly:
    _check_pair(a, b)
    return _binary(_lib.OP_SUB, a, b, a.domain)


def poly_neg(a: RingPoly) -> RingPoly:
    return _binary(_lib.OP_NEG, a, None, a.domain)


def pointwise_mul(a: RingPoly, b: RingPoly) -> RingPoly:
    """Hadamard product of NTT-domain polynomials (ring.py:291-300)."""
    _check_pair(a, b)
    if a.domain != NTT:
        raise RingError("pointwise_mul expects NTT-domain operands")
    return _binary(_lib.OP_MUL, a, b, NTT)


def poly_mul_ntt(a: RingPoly, b: RingPoly) -> RingPoly:
    """Negacyclic product via the NTT; either domain in, Coefficient out (ring.py:303-308)."""
    _check_pair(a, b, same_domain=False)
    fa = a if a.domain == NTT else ntt_forward(a)
    fb = b if b.domain == NTT else ntt_forward(b)
    return ntt_inverse(pointwise_mul(fa, fb))


def residues(c: int, primes) -> list:
    return [int(c) % int(q) for q in primes]


def scalar_mul(a: RingPoly, c: int) -> RingPoly:
    """Multiply by a python integer reduced per limb; domain-preserving (ring.py:282-288)."""
    out = dev.empty(a.data.shape)
    L = _rows(a)
    _lib.check(
        _lib.lib().fcn_scalar_mul(
            a.ctx.handle().ptr, a.data.data_ptr(), _lib.u64_array(residues(c, a.ctx.primes)), out.data_ptr(), L, L, 0, dev.stream_ptr()
        ),
        RingError,
    )
    return RingPoly(a.ctx, out, a.domain)


def poly_mul_monomial(c: RingPoly, k: int, coeff: int) -> RingPoly:
    """coeff * x^k * c in O(n) with the negacyclic wrap (ring.py:339-361)."""
    if not 0 <= k < c.ctx.n:
        raise RingError(f"monomial exponent {k} out of [0, {c.ctx.n})")
    if c.domain != COEFF:
        raise RingError("poly_mul_monomial expects a Coefficient-domain polynomial")
    out = dev.empty(c.data.shape)
    L = _rows(c)
    _lib.check(
        _lib.lib().fcn_poly_mul_monomial(
            c.ctx.handle().ptr, c.data.data_ptr(), int(k), _lib.u64_array(residues(coeff, c.ctx.primes)), out.data_ptr(), L, L, 0,
            dev.stream_ptr(),
        ),
        RingError,
    )
    return RingPoly(c.ctx, out, COEFF)
