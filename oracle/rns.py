"""RNS polynomial arithmetic over Z_q[x]/(x^n+1) -- oracle, test infra only.

A polynomial is a numpy uint64 array of shape (limbs, n) holding canonical
residues.  This restates the reference ring layer:

  * 128-bit product emulation with 32-bit halves and Shoup multiplication
    (reference `modmath.py:31-85`),
  * per-limb tables psi^bitrev(i) / psi^-bitrev(i) (reference `ring.py:67-101`),
  * Cooley-Tukey forward NTT over psis[m:2m] with bit-reversed output
    (`ring.py:199-217`) and Gentleman-Sande inverse over ipsis[h:m] followed
    by multiplication by n^-1 (`ring.py:220-239`),
  * elementwise add/sub/neg/scalar/pointwise (`ring.py:261-300`),
  * schoolbook negacyclic product, the independent check (`ring.py:311-336`),
  * the monomial fast path with negation on wrap (`ring.py:339-361`).

Canonical residues at every boundary, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import nt

U64 = np.uint64
_LO = U64(0xFFFFFFFF)
_SH = U64(32)


def _hi64(a: np.ndarray, b) -> np.ndarray:
    """floor(a*b / 2^64) elementwise via 32-bit limbs (reference modmath.py:31-42)."""
    with np.errstate(over="ignore"):
        a0, a1 = a & _LO, a >> _SH
        b0, b1 = b & _LO, b >> _SH
        p00, p01, p10, p11 = a0 * b0, a0 * b1, a1 * b0, a1 * b1
        carry = ((p00 >> _SH) + (p01 & _LO) + (p10 & _LO)) >> _SH
        return p11 + (p01 >> _SH) + (p10 >> _SH) + carry


def shoup_pre(w: int, q: int) -> U64:
    """floor(w * 2^64 / q), the Shoup companion of constant w (modmath.py:45-47)."""
    return U64((int(w) << 64) // int(q))


def mul_const(a: np.ndarray, w, wq, q) -> np.ndarray:
    """a*w mod q for constant w with Shoup quotient wq; canonical (modmath.py:50-58)."""
    q = U64(q)
    with np.errstate(over="ignore"):
        r = a * w - _hi64(a, wq) * q
    return np.where(r >= q, r - q, r)


def add(a, b, q):
    q = U64(q)
    s = a + b
    return np.where(s >= q, s - q, s)


def sub(a, b, q):
    q = U64(q)
    d = a + (q - b)
    return np.where(d >= q, d - q, d)


def neg(a, q):
    q = U64(q)
    return np.where(a == 0, a, q - a)


def mul(a: np.ndarray, b: np.ndarray, q: int) -> np.ndarray:
    """General a*b mod q, both canonical, q < 2^62 (modmath.py:75-85).

    hi*2^64 + lo is folded as hi*(2^64 mod q) + (lo mod q).
    """
    r64 = (1 << 64) % int(q)
    with np.errstate(over="ignore"):
        hi = _hi64(a, b)
        lo = a * b
    s = mul_const(hi, U64(r64), shoup_pre(r64, q), q) + lo % U64(q)
    qq = U64(q)
    return np.where(s >= qq, s - qq, s)


# --- tables -------------------------------------------------------------------


@dataclass(frozen=True)
class Limb:
    q: int
    n: int
    root: int
    psi: np.ndarray
    psi_q: np.ndarray
    ipsi: np.ndarray
    ipsi_q: np.ndarray
    ninv: int


@lru_cache(maxsize=128)
def limb_tables(q: int, n: int) -> Limb:
    """Twiddles psi^bitrev(i), psi^-bitrev(i) with Shoup quotients (ring.py:67-101)."""
    if n < 2 or n & (n - 1):
        raise ValueError("degree must be a power of two")
    if not nt.is_prime(q) or (q - 1) % (2 * n):
        raise ValueError(f"{q} is not an NTT prime for n={n}")
    psi = nt.root_2n(q, n)
    ipsi = pow(psi, q - 2, q)
    lg = n.bit_length() - 1
    fw = [1] * n
    bw = [1] * n
    for i in range(1, n):
        fw[i] = fw[i - 1] * psi % q
        bw[i] = bw[i - 1] * ipsi % q
    order = [nt.bitrev(i, lg) for i in range(n)]
    f = [fw[j] for j in order]
    b = [bw[j] for j in order]
    return Limb(
        q=q,
        n=n,
        root=psi,
        psi=np.array(f, dtype=U64),
        psi_q=np.array([(x << 64) // q for x in f], dtype=U64),
        ipsi=np.array(b, dtype=U64),
        ipsi_q=np.array([(x << 64) // q for x in b], dtype=U64),
        ninv=pow(n, q - 2, q),
    )


# --- transforms ---------------------------------------------------------------


def ntt_row(row: np.ndarray, L: Limb) -> np.ndarray:
    """Forward negacyclic NTT of one limb row (ring.py:199-217)."""
    x = np.array(row, dtype=U64, copy=True)
    n = L.n
    half = n
    blocks = 1
    while blocks < n:
        half //= 2
        v = x.reshape(blocks, 2, half)
        w = L.psi[blocks : 2 * blocks, None]
        wq = L.psi_q[blocks : 2 * blocks, None]
        lo = v[:, 0, :].copy()
        t = mul_const(v[:, 1, :], w, wq, L.q)
        v[:, 0, :] = add(lo, t, L.q)
        v[:, 1, :] = sub(lo, t, L.q)
        blocks *= 2
    return x


def intt_row(row: np.ndarray, L: Limb) -> np.ndarray:
    """Inverse negacyclic NTT of one limb row (ring.py:220-239)."""
    x = np.array(row, dtype=U64, copy=True)
    n = L.n
    span = 1
    blocks = n // 2
    while blocks >= 1:
        v = x.reshape(blocks, 2, span)
        w = L.ipsi[blocks : 2 * blocks, None]
        wq = L.ipsi_q[blocks : 2 * blocks, None]
        a, b = v[:, 0, :].copy(), v[:, 1, :].copy()
        v[:, 0, :] = add(a, b, L.q)
        v[:, 1, :] = mul_const(sub(a, b, L.q), w, wq, L.q)
        span *= 2
        blocks //= 2
    return mul_const(x, U64(L.ninv), shoup_pre(L.ninv, L.q), L.q)


def ntt(poly: np.ndarray, primes) -> np.ndarray:
    n = poly.shape[-1]
    return np.stack([ntt_row(poly[i], limb_tables(int(q), n)) for i, q in enumerate(primes)])


def intt(poly: np.ndarray, primes) -> np.ndarray:
    n = poly.shape[-1]
    return np.stack([intt_row(poly[i], limb_tables(int(q), n)) for i, q in enumerate(primes)])


# --- elementwise over limbs -----------------------------------------------------


def padd(a, b, primes):
    return np.stack([add(a[i], b[i], q) for i, q in enumerate(primes)])


def psub(a, b, primes):
    return np.stack([sub(a[i], b[i], q) for i, q in enumerate(primes)])


def pneg(a, primes):
    return np.stack([neg(a[i], q) for i, q in enumerate(primes)])


def pscale(a, c: int, primes):
    """Multiply by a (signed) python integer reduced per limb (ring.py:282-288)."""
    rows = []
    for i, q in enumerate(primes):
        w = int(c) % int(q)
        rows.append(mul_const(a[i], U64(w), shoup_pre(w, q), q))
    return np.stack(rows)


def pmul(a, b, primes):
    """Hadamard product of NTT-domain polys (ring.py:291-300)."""
    return np.stack([mul(a[i], b[i], q) for i, q in enumerate(primes)])


def polymul(a, b, primes):
    """Negacyclic product through the NTT (ring.py:303-308)."""
    return intt(pmul(ntt(a, primes), ntt(b, primes), primes), primes)


def polymul_schoolbook(a, b, primes):
    """O(n^2) exact big-integer schoolbook product (ring.py:311-336)."""
    n = a.shape[-1]
    rows = []
    for i, q in enumerate(primes):
        av = [int(v) for v in a[i]]
        bv = [int(v) for v in b[i]]
        acc = [0] * n
        for j, x in enumerate(av):
            if not x:
                continue
            for k, y in enumerate(bv):
                if j + k < n:
                    acc[j + k] += x * y
                else:
                    acc[j + k - n] -= x * y
        rows.append(np.array([v % int(q) for v in acc], dtype=U64))
    return np.stack(rows)


def monomial(a: np.ndarray, k: int, coeff: int, primes) -> np.ndarray:
    """a * coeff * x^k: scale, rotate right by k, negate wrapped part (ring.py:339-361)."""
    n = a.shape[-1]
    if not 0 <= k < n:
        raise ValueError("monomial exponent out of range")
    rows = []
    for i, q in enumerate(primes):
        w = int(coeff) % int(q)
        s = mul_const(a[i], U64(w), shoup_pre(w, q), q)
        rows.append(np.concatenate([neg(s[n - k :], q), s[: n - k]]) if k else s)
    return np.stack(rows)


def from_ints(values, primes, n: int) -> np.ndarray:
    """Signed python ints -> residues per limb (ring.py:156-168)."""
    out = np.zeros((len(primes), n), dtype=U64)
    vals = [int(v) for v in values]
    for i, q in enumerate(primes):
        out[i, : len(vals)] = [v % int(q) for v in vals]
    return out


def random_uniform(primes, n: int, rng: np.random.Generator) -> np.ndarray:
    """Uniform residues, one rng.integers call per limb in limb order (ring.py:171-175)."""
    return np.stack([rng.integers(0, int(q), n, dtype=U64) for q in primes])
