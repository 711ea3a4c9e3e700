"""Leveled FV over the RNS ring on B200 (mirrors reference fv.py).

Same public names, argument meaning and error behaviour as the reference
(`EncryptionParams`, `PlainPoly`, keys, `Ciphertext`, `keygen`, `encrypt`,
`decrypt`, `noise_budget`, `add_ct`, `sub_ct`, `add_pt`, `mul_pt`, `mul_ct`,
serialization; reference fv.py:42-685).  Ciphertext polynomials live in HBM;
all ring arithmetic runs in libfcn.  Randomness is drawn on the host with
numpy in the reference's draw order, so keys and ciphertexts are
byte-identical to the reference for the same seeds.

Batch entry points (`encrypt_batch`, `decrypt_batch`, `mul_ct_batch`)
operate on [B][2][k][n] device buffers -- the layout of the reference's
serialized ciphertext body -- and are what the engine uses.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np

from . import _lib
from . import device as dev
from . import ring
from .ring import COEFF, NTT, RingContext, RingPoly

CT_MAGIC = 0x46434E5031000000
SERIAL_VERSION = 1
KIND_CIPHERTEXT = 0
KIND_SECRET_KEY = 1
KIND_PUBLIC_KEY = 2
KIND_EVAL_KEYS = 3

DEFAULT_SIGMA = 3.2
DEFAULT_BETA = 1 << 32


def _is_prime(v: int) -> bool:
    for w in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if v % w == 0:
            return v == w
    d, r = v - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        x = pow(a, d, v)
        if x in (1, v - 1):
            continue
        for _ in range(r - 1):
            x = x * x % v
            if x == v - 1:
                break
        else:
            return False
    return True


class FVError(ValueError):
    """Parameter, lane, or scale mismatch in scheme operations (fv.py:38)."""


# ------------------------------------------------------------------ native


class _CtxHandle:
    def __init__(self, device: int, params: "EncryptionParams"):
        lib = _lib.lib()
        out = C.c_void_p()
        _lib.check(
            lib.fcn_ctx_create(
                device,
                params.n,
                len(params.limb_primes),
                _lib.u64_array(params.limb_primes),
                len(params.t_lanes),
                _lib.u64_array(params.t_lanes),
                params.beta.bit_length() - 1,
                C.byref(out),
            ),
            FVError,
        )
        self.ptr = out
        self.device = device
        v = C.c_int64()
        _lib.check(lib.fcn_ctx_query(out, 2, C.byref(v)))
        m = v.value
        aux = (C.c_uint64 * max(1, m))()
        _lib.check(lib.fcn_ctx_aux_primes(out, aux))
        self.aux = tuple(int(aux[i]) for i in range(m))
        _lib.check(lib.fcn_ctx_query(out, 3, C.byref(v)))
        self.ell = v.value
        rp = C.c_void_p()
        _lib.check(lib.fcn_ctx_ring(out, C.byref(rp)))
        self.ring_ptr = rp

    def fallbacks(self) -> int:
        v = C.c_int64()
        _lib.check(_lib.lib().fcn_ctx_fallback_count(self.ptr, C.byref(v)))
        return v.value

    def __del__(self):
        try:
            if self.ptr:
                _lib.lib().fcn_ctx_destroy(self.ptr)
        except Exception:
            pass


_ctx_handles: dict = {}


@dataclass(frozen=True)
class EncryptionParams:
    """Everything that pins down one instantiation of the scheme (fv.py:42-130)."""

    n: int
    limb_primes: tuple
    t_lanes: tuple
    beta: int = DEFAULT_BETA
    noise_stddev: float = DEFAULT_SIGMA
    mul_depth_budget: int = 3

    def __post_init__(self):
        object.__setattr__(self, "limb_primes", tuple(int(p) for p in self.limb_primes))
        object.__setattr__(self, "t_lanes", tuple(int(t) for t in self.t_lanes))
        if self.n not in ring.SUPPORTED_DEGREES:
            raise FVError(f"ring degree {self.n} not in {ring.SUPPORTED_DEGREES}")
        if not self.t_lanes:
            raise FVError("at least one plaintext modulus lane is required")
        if self.beta & (self.beta - 1):
            raise FVError("decomposition base beta must be a power of two")
        q = math.prod(self.limb_primes)
        for t in self.t_lanes:
            if q // int(t) < (1 << 16):
                raise FVError(f"ciphertext modulus too small for lane t={t} (need q >> t)")

    @cached_property
    def ctx(self) -> RingContext:
        return RingContext(self.n, self.limb_primes)

    @cached_property
    def q(self) -> int:
        return math.prod(self.limb_primes)

    @cached_property
    def ell(self) -> int:
        e, power = 0, self.beta
        while power <= self.q:
            e += 1
            power *= self.beta
        return e

    def delta(self, lane: int) -> int:
        return self.q // int(self.t_lanes[lane])

    def native(self) -> _CtxHandle:
        d = dev.current_device()
        key = (d, self.n, self.limb_primes, self.t_lanes, self.beta)
        h = _ctx_handles.get(key)
        if h is None:
            h = _CtxHandle(d, self)
            _ctx_handles[key] = h
        return h

    @cached_property
    def aux_primes(self) -> tuple:
        """The reference's auxiliary base (fv.py:99-107), for API parity.

        libfcn's exact multiplication uses its own (possibly smaller)
        extended base, `native().aux`; results do not depend on it."""
        need = self.n.bit_length() + self.q.bit_length() + 1
        count = need // 54 + 1
        step = 2 * self.n
        p = (1 << 55) // step * step + 1
        out, skip = [], set(self.limb_primes)
        while len(out) < count:
            p += step
            if p not in skip and _is_prime(p):
                out.append(p)
        return tuple(out)

    def describe(self) -> str:
        return (
            f"n={self.n}, log2(q)={math.log2(self.q):.1f} over {len(self.limb_primes)} limbs, "
            f"lanes={list(self.t_lanes)}, beta=2^{self.beta.bit_length() - 1}, ell={self.ell}"
        )


@dataclass(frozen=True)
class PlainPoly:
    """Plaintext over R_t, canonical, trailing zeros trimmed (fv.py:133-172)."""

    t: int
    coeffs: np.ndarray

    def __post_init__(self):
        c = np.asarray(self.coeffs, dtype=np.uint64)
        nz = np.nonzero(c)[0]
        c = c[: nz[-1] + 1] if nz.size else c[:0]
        object.__setattr__(self, "coeffs", c)
        if c.size and int(c.max()) >= self.t:
            raise FVError("plaintext coefficient out of range for modulus t")

    @staticmethod
    def zero(t: int) -> "PlainPoly":
        return PlainPoly(t, np.zeros(0, dtype=np.uint64))

    def is_zero(self) -> bool:
        return self.coeffs.size == 0

    @property
    def nnz(self) -> int:
        return int(np.count_nonzero(self.coeffs))

    def is_monomial(self) -> bool:
        return self.nnz == 1

    def centered(self) -> list:
        h = self.t // 2
        return [int(c) if int(c) <= h else int(c) - self.t for c in self.coeffs]

    def __eq__(self, other) -> bool:
        return isinstance(other, PlainPoly) and self.t == other.t and np.array_equal(self.coeffs, other.coeffs)


@dataclass(frozen=True)
class SecretKey:
    s: RingPoly
    s_ntt: RingPoly = field(repr=False)


@dataclass(frozen=True)
class PublicKey:
    p0: RingPoly
    p1: RingPoly
    p0_ntt: RingPoly = field(repr=False)
    p1_ntt: RingPoly = field(repr=False)


class _KeysHandle:
    def __init__(self, params: EncryptionParams, a_host: np.ndarray, g_host: np.ndarray):
        h = params.native()
        out = C.c_void_p()
        a = np.ascontiguousarray(a_host, dtype=np.uint64)
        g = np.ascontiguousarray(g_host, dtype=np.uint64)
        _lib.check(
            _lib.lib().fcn_keys_create(
                h.ptr, a.ctypes.data_as(C.POINTER(C.c_uint64)), g.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(out)
            ),
            FVError,
        )
        self.ptr = out

    def __del__(self):
        try:
            if self.ptr:
                _lib.lib().fcn_keys_destroy(self.ptr)
        except Exception:
            pass


@dataclass(frozen=True)
class EvalKeys:
    """(a_i, g_i), g_i = [-(a_i s + e_i) + beta^i s^2]_q, i = 0..ell (fv.py:191-198)."""

    a: tuple
    g: tuple
    a_ntt: tuple = field(repr=False, default=())
    g_ntt: tuple = field(repr=False, default=())

    def native(self, params: EncryptionParams) -> _KeysHandle:
        cache = self.__dict__.setdefault("_native", {})
        key = (dev.current_device(), params.n, params.limb_primes, params.beta)
        h = cache.get(key)
        if h is None:
            a = np.stack([p.host() for p in self.a])
            g = np.stack([p.host() for p in self.g])
            h = _KeysHandle(params, a, g)
            cache[key] = h
        return h


@dataclass(frozen=True)
class Ciphertext:
    c0: RingPoly
    c1: RingPoly
    params: EncryptionParams
    lane: int = 0
    scale_exponent: int = 0
    mul_depth: int = 0

    @staticmethod
    def zero(params: EncryptionParams, lane: int = 0, scale_exponent: int = 0) -> "Ciphertext":
        z = RingPoly.zero(params.ctx)
        return Ciphertext(z, z, params, lane, scale_exponent, 0)

    def stacked(self):
        """[1][2][k][n] device buffer of this ciphertext."""
        import torch

        return torch.stack([self.c0.data, self.c1.data]).unsqueeze(0).contiguous()


def ciphertext_from_buffer(params, buf2, lane=0, scale=0, depth=0) -> Ciphertext:
    """View a [2][k][n] device slice as a Ciphertext (no copy)."""
    return Ciphertext(RingPoly(params.ctx, buf2[0]), RingPoly(params.ctx, buf2[1]), params, lane, scale, depth)


# --------------------------------------------------------------- sampling


def _signed_rows(params: EncryptionParams, values: np.ndarray) -> np.ndarray:
    v = np.asarray(values, dtype=np.int64)
    return np.stack([np.where(v < 0, q + v, v).astype(np.uint64) for q in params.limb_primes])


def _as_rng(rng) -> np.random.Generator:
    return rng if isinstance(rng, np.random.Generator) else np.random.default_rng(rng)


def _ternary(n, rng):
    return rng.integers(-1, 2, n, dtype=np.int64)


def _gaussian(n, rng, sigma):
    bound = int(math.floor(6 * sigma))
    e = np.rint(rng.normal(0.0, sigma, n)).astype(np.int64)
    return np.clip(e, -bound, bound)


def sample_ternary(ctx_params, rng) -> RingPoly:
    return RingPoly(ctx_params.ctx, _signed_rows(ctx_params, _ternary(ctx_params.n, rng)))


# ------------------------------------------------------------------- keys


def keygen(params: EncryptionParams, seed):
    """(sk, pk, ek), byte-identical to the reference for a fixed seed (fv.py:247-278)."""
    rng = _as_rng(seed)
    ctx = params.ctx
    n, sig = params.n, params.noise_stddev
    s = RingPoly(ctx, _signed_rows(params, _ternary(n, rng)))
    s_ntt = ring.ntt_forward(s)
    p0 = RingPoly.random_uniform(ctx, rng)
    e_pk = RingPoly(ctx, _signed_rows(params, _gaussian(n, rng, sig)))
    p1 = ring.poly_neg(ring.poly_add(ring.poly_mul_ntt(p0, s_ntt), e_pk))
    s_sq = ring.poly_mul_ntt(s_ntt, s_ntt)
    a_list, g_list = [], []
    for i in range(params.ell + 1):
        a_i = RingPoly.random_uniform(ctx, rng)
        e_i = RingPoly(ctx, _signed_rows(params, _gaussian(n, rng, sig)))
        term = ring.scalar_mul(s_sq, pow(params.beta, i, params.q))
        g_i = ring.poly_add(ring.poly_neg(ring.poly_add(ring.poly_mul_ntt(a_i, s_ntt), e_i)), term)
        a_list.append(a_i)
        g_list.append(g_i)
    pk = PublicKey(p0, p1, ring.ntt_forward(p0), ring.ntt_forward(p1))
    ek = EvalKeys(
        tuple(a_list), tuple(g_list), tuple(ring.ntt_forward(a) for a in a_list), tuple(ring.ntt_forward(g) for g in g_list)
    )
    return SecretKey(s, s_ntt), pk, ek


# -------------------------------------------------------------- plaintexts


def _plain_to_ring(params: EncryptionParams, m: PlainPoly) -> RingPoly:
    if m.coeffs.size > params.n:
        raise FVError("plaintext degree exceeds ring degree")
    return RingPoly.from_int_coeffs(params.ctx, m.centered())


def _delta_m(params: EncryptionParams, m: PlainPoly, lane: int) -> RingPoly:
    return ring.scalar_mul(_plain_to_ring(params, m), params.delta(lane))


# ---------------------------------------------------------------- batch core


def _k(params):
    return len(params.limb_primes)


def _ring_call(fn, *args):
    _lib.check(fn(*args), FVError)


def _ext_ring(params):
    return params.native().ring_ptr


def _lift_rows(params, vals_dev, count):
    """[count][n] signed int64 -> [count][k][n] residues mod q_i."""
    k = _k(params)
    out = dev.empty((count, k, params.n))
    _ring_call(_lib.lib().fcn_lift_signed, _ext_ring(params), vals_dev.data_ptr(), count, out.data_ptr(), k, 0, dev.stream_ptr())
    return out


def _ntt_rows(params, buf, rows, fwd=True):
    k = _k(params)
    fn = _lib.lib().fcn_ntt_forward if fwd else _lib.lib().fcn_ntt_inverse
    _ring_call(fn, _ext_ring(params), buf.data_ptr(), rows, k, 0, dev.stream_ptr())


def _binary_rows(params, op, a, b, b_rows, out, rows):
    k = _k(params)
    bp = b.data_ptr() if b is not None else None
    _ring_call(_lib.lib().fcn_poly_binary, _ext_ring(params), op, a.data_ptr(), bp, b_rows, out.data_ptr(), rows, k, 0, dev.stream_ptr())


def _scalar_rows(params, a, residues, out, rows):
    k = _k(params)
    _ring_call(
        _lib.lib().fcn_scalar_mul, _ext_ring(params), a.data_ptr(), _lib.u64_array(residues), out.data_ptr(), rows, k, 0, dev.stream_ptr()
    )


def sample_encryption_noise(params: EncryptionParams, count: int, rng):
    """Per ciphertext, in reference order: u (ternary), e1, e2 (fv.py:314-317)."""
    n, sig = params.n, params.noise_stddev
    u = np.empty((count, n), dtype=np.int64)
    e1 = np.empty((count, n), dtype=np.int64)
    e2 = np.empty((count, n), dtype=np.int64)
    for b in range(count):
        u[b] = _ternary(n, rng)
        e1[b] = _gaussian(n, rng, sig)
        e2[b] = _gaussian(n, rng, sig)
    return u, e1, e2


def encrypt_batch(pk: PublicKey, params: EncryptionParams, centered_plain: np.ndarray, lane: int = 0, rng=None, noise=None):
    """Encrypt B plaintexts given as centered coefficients (B, <=n) int64.

    Returns a [B][2][k][n] device buffer; byte-identical to B sequential
    reference `fv.encrypt` calls sharing `rng` (fv.py:298-320)."""
    import torch

    rng = _as_rng(rng)
    m = np.zeros((centered_plain.shape[0], params.n), dtype=np.int64)
    m[:, : centered_plain.shape[1]] = centered_plain
    B, n, k = m.shape[0], params.n, _k(params)
    u, e1, e2 = noise if noise is not None else sample_encryption_noise(params, B, rng)
    U = _lift_rows(params, dev.to_device(u), B)
    _ntt_rows(params, U, B * k, True)
    X1 = dev.empty((B, k, n))
    X0 = dev.empty((B, k, n))
    _binary_rows(params, _lib.OP_MUL, U, pk.p1_ntt.data, k, X1, B * k)
    _binary_rows(params, _lib.OP_MUL, U, pk.p0_ntt.data, k, X0, B * k)
    _ntt_rows(params, X1, B * k, False)
    _ntt_rows(params, X0, B * k, False)
    Mres = _lift_rows(params, dev.to_device(m), B)
    delta = params.delta(lane)
    _scalar_rows(params, Mres, [delta % q for q in params.limb_primes], Mres, B * k)
    # c0 = (Delta m + p1 u) + e1 ; c1 = p0 u + e2  (same association as fv.py:318-319)
    _binary_rows(params, _lib.OP_ADD, Mres, X1, B * k, X1, B * k)
    E1 = _lift_rows(params, dev.to_device(e1), B)
    _binary_rows(params, _lib.OP_ADD, X1, E1, B * k, X1, B * k)
    E2 = _lift_rows(params, dev.to_device(e2), B)
    _binary_rows(params, _lib.OP_ADD, X0, E2, B * k, X0, B * k)
    out = torch.stack([X1, X0], dim=1).contiguous()
    return out


def raw_decrypt_batch(sk: SecretKey, params: EncryptionParams, buf):
    """[c0 + c1 s]_q rows [B][k][n] for a [B][2][k][n] buffer."""
    B, k, n = buf.shape[0], _k(params), params.n
    C1 = buf[:, 1].contiguous()
    _ntt_rows(params, C1, B * k, True)
    _binary_rows(params, _lib.OP_MUL, C1, sk.s_ntt.data, k, C1, B * k)
    _ntt_rows(params, C1, B * k, False)
    C0 = buf[:, 0].contiguous()
    _binary_rows(params, _lib.OP_ADD, C0, C1, B * k, C1, B * k)
    return C1


def decrypt_batch(sk: SecretKey, params: EncryptionParams, buf, lane: int = 0):
    """Plaintext coefficients (B, n) uint64 (untrimmed) of B ciphertexts (fv.py:337-353)."""
    B = buf.shape[0]
    W = raw_decrypt_batch(sk, params, buf)
    M = dev.empty((B, params.n))
    _ring_call(_lib.lib().fcn_decrypt_round, params.native().ptr, lane, W.data_ptr(), M.data_ptr(), B, dev.stream_ptr())
    return dev.to_host(M)


def mul_ct_workspace(params: EncryptionParams, chunk: int):
    nbytes = _lib.lib().fcn_mul_ct_workspace_bytes(params.native().ptr, chunk)
    return dev.empty(((nbytes + 7) // 8,))


MUL_CT_WORKSPACE_CAP = 12 << 30  # default scratch cap per call (bytes)


def mul_ct_batch(params: EncryptionParams, ek: EvalKeys, lane: int, a, b=None, out=None, chunk: int | None = None,
                 workspace=None, act: tuple | None = None, fanout=()):
    """Relinearised products of [B][2][k][n] buffers (b=None: squares).

    act=(c2, c1): fused activation epilogue, out = c2*a^2 + c1*a (mod q)
    (squares only; fcn_mul_ct_ex, include/fcn.h).  fanout: device addresses
    that receive the same output rows from the final kernel
    (fcn_mul_ct_multi)."""
    B = a.shape[0]
    if out is None:
        out = dev.empty(a.shape)
    if B == 0:
        return out
    if act is not None and b is not None:
        raise FVError("the activation epilogue applies to squares only")
    h = params.native()
    kh = ek.native(params)
    if workspace is None:
        per = _lib.lib().fcn_mul_ct_workspace_bytes(h.ptr, 1)
        if chunk is None:
            chunk = max(1, min(B, MUL_CT_WORKSPACE_CAP // max(1, per)))
        workspace = mul_ct_workspace(params, chunk)
    nbytes = workspace.numel() * 8
    flags, c2, c1 = (0, 1, 0) if act is None else (1, int(act[0]), int(act[1]))
    ptrs = _lib.ptr_array([out.data_ptr()] + [int(p) for p in fanout])
    _lib.check(
        _lib.lib().fcn_mul_ct_multi(
            h.ptr, kh.ptr, lane, a.data_ptr(), b.data_ptr() if b is not None else None, C.cast(ptrs, C.c_void_p),
            1 + len(fanout), B, flags, c2, c1, workspace.data_ptr(), nbytes, dev.stream_ptr(),
        ),
        FVError,
    )
    return out


# --------------------------------------------------------- encrypt/decrypt


def encrypt(pk: PublicKey, params: EncryptionParams, m: PlainPoly, lane: int = 0, scale_exponent: int = 0, rng=None) -> Ciphertext:
    """(c0, c1) = ([Delta m + p1 u + e1]_q, [p0 u + e2]_q) (fv.py:298-320)."""
    if m.t != params.t_lanes[lane]:
        raise FVError(f"plaintext modulus {m.t} is not lane {lane}")
    if m.coeffs.size > params.n:
        raise FVError("plaintext degree exceeds ring degree")
    cen = np.array([m.centered()], dtype=np.int64) if m.coeffs.size else np.zeros((1, 1), dtype=np.int64)
    buf = encrypt_batch(pk, params, cen, lane, _as_rng(rng))
    return ciphertext_from_buffer(params, buf[0], lane, scale_exponent, 0)


def raw_decrypt_integers(sk: SecretKey, ct: Ciphertext) -> list:
    """[c0 + c1 s]_q as canonical big-int coefficients (host CRT; diagnostic)."""
    w = ring.poly_add(ct.c0, ring.poly_mul_ntt(ct.c1, sk.s_ntt))
    return _crt_coeffs(ct.params, w.host())


def _crt_coeffs(params, rows: np.ndarray) -> list:
    q = params.q
    ws = []
    for p in params.limb_primes:
        mq = q // p
        ws.append(mq * pow(mq % p, p - 2, p))
    cols = [rows[i].tolist() for i in range(len(params.limb_primes))]
    return [sum(r * w for r, w in zip(res, ws)) % q for res in zip(*cols)]


def decrypt(sk: SecretKey, ct: Ciphertext, check_budget: bool = False) -> PlainPoly:
    """m = [round(t/q [c0 + c1 s]_q)]_t with exact rounding (fv.py:337-353)."""
    params = ct.params
    t = int(params.t_lanes[ct.lane])
    m = decrypt_batch(sk, params, ct.stacked(), ct.lane)[0]
    out = PlainPoly(t, m)
    if check_budget and noise_budget(sk, ct) < 1.0:
        raise FVError("noise budget exhausted: decryption unreliable")
    return out


def noise_budget(sk: SecretKey, ct: Ciphertext) -> float:
    """Bits of headroom before noise corrupts decryption (fv.py:356-377).

    w = c0 + c1 s on the GPU; the largest |centred [t w]_q| over the
    coefficients is found by fcn_noise_max (multiword CRT per coefficient,
    block maxima) and the host takes the reference's log2 of that exact
    integer."""
    return float(noise_budget_batch(sk, ct.params, ct.stacked(), ct.lane)[0])


def noise_budget_batch(sk: SecretKey, params: EncryptionParams, buf, lane: int = 0) -> np.ndarray:
    """noise_budget of every ciphertext of a [B][2][k][n] device buffer."""
    B = buf.shape[0]
    w = raw_decrypt_batch(sk, params, buf)
    q = params.q
    words = (q.bit_length() + 63) // 64
    blocks = max(1, min(64, params.n // 256))
    out = dev.empty((B, blocks, words))
    _lib.check(_lib.lib().fcn_noise_max(params.native().ptr, lane, w.data_ptr(), B, out.data_ptr(), blocks, words,
                                        dev.stream_ptr()), FVError)
    host = dev.to_host(out)
    res = np.empty(B)
    for b in range(B):
        worst = 1
        for blk in range(blocks):
            v = sum(int(host[b, blk, i]) << (64 * i) for i in range(words))
            worst = max(worst, v)
        res[b] = math.log2(q) - 1.0 - math.log2(worst)
    return res


# --------------------------------------------------------------- evaluation


def _check_compat(a: Ciphertext, b: Ciphertext, require_scale: bool = True) -> None:
    if a.params is not b.params and a.params != b.params:
        raise FVError("ciphertext parameter mismatch")
    if a.lane != b.lane:
        raise FVError(f"lane mismatch: {a.lane} vs {b.lane}")
    if require_scale and a.scale_exponent != b.scale_exponent:
        raise FVError(f"scale mismatch: 2^{a.scale_exponent} vs 2^{b.scale_exponent}")


def add_ct(a: Ciphertext, b: Ciphertext) -> Ciphertext:
    _check_compat(a, b)
    return Ciphertext(ring.poly_add(a.c0, b.c0), ring.poly_add(a.c1, b.c1), a.params, a.lane, a.scale_exponent, max(a.mul_depth, b.mul_depth))


def sub_ct(a: Ciphertext, b: Ciphertext) -> Ciphertext:
    _check_compat(a, b)
    return Ciphertext(ring.poly_sub(a.c0, b.c0), ring.poly_sub(a.c1, b.c1), a.params, a.lane, a.scale_exponent, max(a.mul_depth, b.mul_depth))


def add_pt(ct: Ciphertext, m: PlainPoly) -> Ciphertext:
    """(c0 + Delta m, c1); a zero plaintext returns ct itself (fv.py:418-431)."""
    if m.t != ct.params.t_lanes[ct.lane]:
        raise FVError("plaintext modulus does not match ciphertext lane")
    if m.is_zero():
        return ct
    return Ciphertext(ring.poly_add(ct.c0, _delta_m(ct.params, m, ct.lane)), ct.c1, ct.params, ct.lane, ct.scale_exponent, ct.mul_depth)


def is_monomial_plain(m: PlainPoly) -> bool:
    return m.is_monomial()


def mul_pt(ct: Ciphertext, m: PlainPoly, plain_scale_exponent: int = 0) -> Ciphertext:
    """(m c0, m c1), monomial fast path when m has one term (fv.py:439-460)."""
    if m.t != ct.params.t_lanes[ct.lane]:
        raise FVError("plaintext modulus does not match ciphertext lane")
    if m.is_zero():
        raise FVError("zero plaintext multiplier: elide the operation instead")
    if is_monomial_plain(m):
        k = int(np.nonzero(m.coeffs)[0][0])
        coeff = m.centered()[k]
        c0 = ring.poly_mul_monomial(ct.c0, k, coeff)
        c1 = ring.poly_mul_monomial(ct.c1, k, coeff)
    else:
        m_ntt = ring.ntt_forward(_plain_to_ring(ct.params, m))
        c0 = ring.poly_mul_ntt(ct.c0, m_ntt)
        c1 = ring.poly_mul_ntt(ct.c1, m_ntt)
    return Ciphertext(c0, c1, ct.params, ct.lane, ct.scale_exponent + plain_scale_exponent, ct.mul_depth)


def mul_ct(a: Ciphertext, b: Ciphertext, ek: EvalKeys) -> Ciphertext:
    """Tensor, exact rescale, relinearize; scales add, depth + 1 (fv.py:498-549)."""
    _check_compat(a, b, require_scale=False)
    params = a.params
    A = a.stacked()
    Bb = None if (b is a) else b.stacked()
    out = mul_ct_batch(params, ek, a.lane, A, Bb)
    return ciphertext_from_buffer(
        params, out[0], a.lane, a.scale_exponent + b.scale_exponent, max(a.mul_depth, b.mul_depth) + 1
    )


# ------------------------------------------------------------ serialization


def _header(params, kind, lane, scale, depth) -> bytes:
    words = np.array([CT_MAGIC, SERIAL_VERSION, params.n, len(params.limb_primes), lane, scale & 0xFFFFFFFFFFFFFFFF, depth, kind], dtype=np.uint64)
    return words.astype("<u8").tobytes()


def _parse_header(data: bytes, params, expect_kind: int):
    if len(data) < 64:
        raise FVError("truncated serialization header")
    w = np.frombuffer(data[:64], dtype="<u8").astype(np.uint64)
    if int(w[0]) != CT_MAGIC:
        raise FVError("bad magic word in serialized object")
    if int(w[1]) != SERIAL_VERSION:
        raise FVError(f"unsupported serialization version {int(w[1])}")
    if int(w[2]) != params.n or int(w[3]) != len(params.limb_primes):
        raise FVError("serialized object does not match the supplied parameters")
    kind = int(w[7])
    if kind != expect_kind:
        names = {0: "ciphertext", 1: "secret key", 2: "public key", 3: "eval keys"}
        raise FVError(f"refusing to load: file holds a {names.get(kind, '?')}, expected {names.get(expect_kind, '?')}")
    scale = int(w[5])
    if scale >= 1 << 63:
        scale -= 1 << 64
    return int(w[4]), scale, int(w[6])


def _poly_from(buf: bytes, offset: int, ctx: RingContext):
    count = len(ctx.primes) * ctx.n
    end = offset + count * 8
    if end > len(buf):
        raise FVError("truncated polynomial block")
    arr = np.frombuffer(buf[offset:end], dtype="<u8").astype(np.uint64)
    return RingPoly(ctx, arr.reshape(len(ctx.primes), ctx.n), COEFF), end


def ciphertext_to_bytes(ct: Ciphertext) -> bytes:
    """8 header words then c0 then c1, limb-major u64 LE (fv.py:610-619)."""
    body = dev.to_host(ct.stacked()[0]).astype("<u8").tobytes()
    return _header(ct.params, KIND_CIPHERTEXT, ct.lane, ct.scale_exponent, ct.mul_depth) + body


def ciphertext_from_bytes(data: bytes, params: EncryptionParams) -> Ciphertext:
    lane, scale, depth = _parse_header(data, params, KIND_CIPHERTEXT)
    c0, off = _poly_from(data, 64, params.ctx)
    c1, off = _poly_from(data, off, params.ctx)
    if off != len(data):
        raise FVError("trailing bytes after ciphertext payload")
    return Ciphertext(c0, c1, params, lane, scale, depth)


def ciphertext_num_words(params: EncryptionParams) -> int:
    return 8 + 2 * len(params.limb_primes) * params.n


def eval_keys_to_bytes(ek: EvalKeys, params: EncryptionParams) -> bytes:
    blob = _header(params, KIND_EVAL_KEYS, 0, 0, params.ell)
    for a_i, g_i in zip(ek.a, ek.g):
        blob += a_i.host().astype("<u8").tobytes() + g_i.host().astype("<u8").tobytes()
    return blob


def eval_keys_from_bytes(data: bytes, params: EncryptionParams) -> EvalKeys:
    _, _, ell = _parse_header(data, params, KIND_EVAL_KEYS)
    if ell != params.ell:
        raise FVError("eval key count does not match parameters")
    a_list, g_list = [], []
    off = 64
    for _ in range(ell + 1):
        a_i, off = _poly_from(data, off, params.ctx)
        g_i, off = _poly_from(data, off, params.ctx)
        a_list.append(a_i)
        g_list.append(g_i)
    if off != len(data):
        raise FVError("trailing bytes after eval key payload")
    return EvalKeys(tuple(a_list), tuple(g_list), tuple(ring.ntt_forward(p) for p in a_list), tuple(ring.ntt_forward(p) for p in g_list))


def eval_keys_from_arrays(params: EncryptionParams, a: np.ndarray, g: np.ndarray) -> EvalKeys:
    """EvalKeys from coefficient-domain host arrays [ell+1][k][n]."""
    ctx = params.ctx
    al = tuple(RingPoly(ctx, np.ascontiguousarray(x, dtype=np.uint64)) for x in a)
    gl = tuple(RingPoly(ctx, np.ascontiguousarray(x, dtype=np.uint64)) for x in g)
    return EvalKeys(al, gl, tuple(ring.ntt_forward(p) for p in al), tuple(ring.ntt_forward(p) for p in gl))
