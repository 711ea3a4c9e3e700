"""FV/BFV scheme restatement -- oracle, test infra only.

Follows reference `pkg/src/hecnet/fv.py`:
  * parameter derivations: ell (:78-85), Delta = q // t (:87-88), CRT
    weights (:90-97), auxiliary primes (:99-107), extended base (:109-124);
  * samplers and their RNG draw order (:220-241), keygen (:247-278),
    encrypt (:298-320), decrypt (:337-353), noise budget (:356-377);
  * add_ct/sub_ct/add_pt/mul_pt (:394-460);
  * exact mul_ct: centered lift to the extended base, NTT tensor,
    floor((t*T + q>>1)/q) mod q with Python big ints, base-beta digits of
    c2' folded through the eval keys (:463-549);
  * serialization: 8 LE u64 header words then limb-major bodies (:555-685).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import cached_property

import numpy as np

from . import nt, rns

U64 = np.uint64
MAGIC = 0x46434E5031000000


@dataclass(frozen=True)
class Params:
    n: int
    primes: tuple
    t_lanes: tuple
    beta: int = 1 << 32
    sigma: float = 3.2
    depth_budget: int = 3

    @cached_property
    def q(self) -> int:
        return math.prod(int(p) for p in self.primes)

    @cached_property
    def ell(self) -> int:
        """Largest e with beta^e <= q (fv.py:78-85)."""
        e, acc = 0, self.beta
        while acc <= self.q:
            e += 1
            acc *= self.beta
        return e

    @property
    def log2_beta(self) -> int:
        return self.beta.bit_length() - 1

    def delta(self, lane: int = 0) -> int:
        return self.q // int(self.t_lanes[lane])

    @cached_property
    def aux(self) -> tuple:
        """Auxiliary base for the exact tensor (fv.py:99-107)."""
        need = self.n.bit_length() + self.q.bit_length() + 1
        return tuple(nt.ntt_primes(self.n, need // 54 + 1, bits=55, exclude=self.primes))

    @cached_property
    def ext(self) -> tuple:
        return tuple(int(p) for p in self.primes) + self.aux

    @cached_property
    def ext_q(self) -> int:
        return math.prod(self.ext)


@dataclass
class Ct:
    c0: np.ndarray
    c1: np.ndarray
    lane: int = 0
    scale: int = 0
    depth: int = 0


# --- helpers ----------------------------------------------------------------


def centered_plain(coeffs, t: int) -> list[int]:
    """Plain coefficient c -> c if c <= t//2 else c - t (fv.py:162-165)."""
    h = t // 2
    return [int(c) if int(c) <= h else int(c) - t for c in coeffs]


def crt_ints(poly: np.ndarray, primes) -> list[int]:
    """Canonical integers in [0, prod) from residues (fv.py:323-328)."""
    Q = math.prod(int(p) for p in primes)
    ws = []
    for p in primes:
        m = Q // int(p)
        ws.append(m * pow(m % int(p), int(p) - 2, int(p)))
    cols = [poly[i].tolist() for i in range(len(primes))]
    return [sum(int(r) * w for r, w in zip(col, ws)) % Q for col in zip(*cols)]


def ints_to_poly(vals, primes) -> np.ndarray:
    return np.stack([np.array([int(v) % int(q) for v in vals], dtype=U64) for q in primes])


def signed_to_poly(vals: np.ndarray, primes) -> np.ndarray:
    v = np.asarray(vals, dtype=np.int64)
    return np.stack([np.where(v < 0, int(q) + v, v).astype(U64) for q in primes])


# --- sampling / keys ------------------------------------------------------------


def ternary(P: Params, rng) -> np.ndarray:
    return signed_to_poly(rng.integers(-1, 2, P.n, dtype=np.int64), P.primes)


def gaussian(P: Params, rng) -> np.ndarray:
    cap = int(math.floor(6 * P.sigma))
    e = np.rint(rng.normal(0.0, P.sigma, P.n)).astype(np.int64)
    return signed_to_poly(np.clip(e, -cap, cap), P.primes)


@dataclass
class Keys:
    s: np.ndarray
    p0: np.ndarray
    p1: np.ndarray
    a: list
    g: list


def keygen(P: Params, seed) -> Keys:
    """Draw order s, p0, e', then (a_i, e_i) for i=0..ell (fv.py:247-278)."""
    rng = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
    pr = P.primes
    s = ternary(P, rng)
    p0 = rns.random_uniform(pr, P.n, rng)
    e = gaussian(P, rng)
    p1 = rns.pneg(rns.padd(rns.polymul(p0, s, pr), e, pr), pr)
    s2 = rns.polymul(s, s, pr)
    a_l, g_l = [], []
    for i in range(P.ell + 1):
        ai = rns.random_uniform(pr, P.n, rng)
        ei = gaussian(P, rng)
        gi = rns.padd(
            rns.pneg(rns.padd(rns.polymul(ai, s, pr), ei, pr), pr),
            rns.pscale(s2, pow(P.beta, i, P.q), pr),
            pr,
        )
        a_l.append(ai)
        g_l.append(gi)
    return Keys(s, p0, p1, a_l, g_l)


def delta_m(P: Params, coeffs, lane: int) -> np.ndarray:
    """Delta * centered(m) in R_q (fv.py:284-292)."""
    t = int(P.t_lanes[lane])
    return rns.pscale(rns.from_ints(centered_plain(coeffs, t), P.primes, P.n), P.delta(lane), P.primes)


def encrypt(P: Params, keys: Keys, coeffs, lane=0, scale=0, rng=None) -> Ct:
    """c0 = Delta m + p1 u + e1, c1 = p0 u + e2; draw order u, e1, e2 (fv.py:298-320)."""
    rng = rng if isinstance(rng, np.random.Generator) else np.random.default_rng(rng)
    pr = P.primes
    u = ternary(P, rng)
    e1 = gaussian(P, rng)
    e2 = gaussian(P, rng)
    c0 = rns.padd(rns.padd(delta_m(P, coeffs, lane), rns.polymul(keys.p1, u, pr), pr), e1, pr)
    c1 = rns.padd(rns.polymul(keys.p0, u, pr), e2, pr)
    return Ct(c0, c1, lane, scale, 0)


def decrypt(P: Params, keys: Keys, ct: Ct) -> np.ndarray:
    """m = floor((w t + q>>1)/q) mod t, w = [c0 + c1 s]_q (fv.py:337-353).

    Returns the full length-n coefficient vector (untrimmed).
    """
    t = int(P.t_lanes[ct.lane])
    w = rns.padd(ct.c0, rns.polymul(ct.c1, keys.s, P.primes), P.primes)
    h = P.q >> 1
    return np.array([((v * t + h) // P.q) % t for v in crt_ints(w, P.primes)], dtype=U64)


def noise_budget(P: Params, keys: Keys, ct: Ct) -> float:
    """log2(q) - 1 - log2 ||[t (c0 + c1 s)]_q||_inf (fv.py:356-377)."""
    t = int(P.t_lanes[ct.lane])
    w = rns.padd(ct.c0, rns.polymul(ct.c1, keys.s, P.primes), P.primes)
    worst = 1
    for v in crt_ints(rns.pscale(w, t, P.primes), P.primes):
        v = P.q - v if v > (P.q >> 1) else v
        worst = max(worst, v)
    return math.log2(P.q) - 1.0 - math.log2(worst)


# --- evaluation ops ---------------------------------------------------------------


def add_ct(P: Params, a: Ct, b: Ct) -> Ct:
    if a.lane != b.lane or a.scale != b.scale:
        raise ValueError("lane/scale mismatch")
    return Ct(rns.padd(a.c0, b.c0, P.primes), rns.padd(a.c1, b.c1, P.primes), a.lane, a.scale, max(a.depth, b.depth))


def sub_ct(P: Params, a: Ct, b: Ct) -> Ct:
    if a.lane != b.lane or a.scale != b.scale:
        raise ValueError("lane/scale mismatch")
    return Ct(rns.psub(a.c0, b.c0, P.primes), rns.psub(a.c1, b.c1, P.primes), a.lane, a.scale, max(a.depth, b.depth))


def add_pt(P: Params, ct: Ct, coeffs) -> Ct:
    """(c0 + Delta m, c1); a zero plaintext returns ct itself (fv.py:418-431)."""
    if not any(int(c) for c in coeffs):
        return ct
    return Ct(rns.padd(ct.c0, delta_m(P, coeffs, ct.lane), P.primes), ct.c1, ct.lane, ct.scale, ct.depth)


def mul_pt(P: Params, ct: Ct, coeffs, plain_scale: int = 0) -> Ct:
    """Monomial fast path or NTT product (fv.py:439-460)."""
    t = int(P.t_lanes[ct.lane])
    cs = [int(c) for c in coeffs]
    nz = [i for i, c in enumerate(cs) if c]
    if not nz:
        raise ValueError("zero plaintext multiplier")
    if len(nz) == 1:
        k = nz[0]
        w = centered_plain([cs[k]], t)[0]
        c0 = rns.monomial(ct.c0, k, w, P.primes)
        c1 = rns.monomial(ct.c1, k, w, P.primes)
    else:
        m = rns.from_ints(centered_plain(cs, t), P.primes, P.n)
        c0 = rns.polymul(ct.c0, m, P.primes)
        c1 = rns.polymul(ct.c1, m, P.primes)
    return Ct(c0, c1, ct.lane, ct.scale + plain_scale, ct.depth)


def _lift_ext(P: Params, poly: np.ndarray) -> np.ndarray:
    """Centered lift (x > q>>1 -> x - q) into the extended base (fv.py:463-470)."""
    h = P.q >> 1
    cents = [v - P.q if v > h else v for v in crt_ints(poly, P.primes)]
    rows = [poly[i] for i in range(len(P.primes))]
    for p in P.aux:
        rows.append(np.array([c % p for c in cents], dtype=U64))
    return np.stack(rows)


def _rescale(P: Params, tpoly: np.ndarray, t: int) -> list[int]:
    """Centered ext-base CRT then ((c t + q>>1) // q) mod q (fv.py:473-490)."""
    B = P.ext_q
    hb = B >> 1
    h = P.q >> 1
    out = []
    for v in crt_ints(tpoly, P.ext):
        c = v - B if v > hb else v
        out.append(((c * t + h) // P.q) % P.q)
    return out


_KEY_NTT: dict = {}


def _key_ntt(P: Params, keys: Keys):
    """NTT-domain eval keys, computed once per key set like the reference's
    cached `EvalKeys.g_ntt/a_ntt` (fv.py:192-198, used at :534-535)."""
    hit = _KEY_NTT.get(id(keys))
    if hit is None or hit[0] is not keys:
        hit = (keys, [rns.ntt(g, P.primes) for g in keys.g], [rns.ntt(a, P.primes) for a in keys.a])
        _KEY_NTT.clear()
        _KEY_NTT[id(keys)] = hit
    return hit[1], hit[2]


def mul_ct(P: Params, a: Ct, b: Ct, keys: Keys) -> Ct:
    """Tensor -> exact rescale -> base-beta relinearization (fv.py:498-549)."""
    if a.lane != b.lane:
        raise ValueError("lane mismatch")
    t = int(P.t_lanes[a.lane])
    E = P.ext
    fa0, fa1 = rns.ntt(_lift_ext(P, a.c0), E), rns.ntt(_lift_ext(P, a.c1), E)
    fb0, fb1 = rns.ntt(_lift_ext(P, b.c0), E), rns.ntt(_lift_ext(P, b.c1), E)
    t0 = rns.intt(rns.pmul(fa0, fb0, E), E)
    t1 = rns.intt(rns.padd(rns.pmul(fa0, fb1, E), rns.pmul(fa1, fb0, E), E), E)
    t2 = rns.intt(rns.pmul(fa1, fb1, E), E)
    r0, r1, r2 = (_rescale(P, x, t) for x in (t0, t1, t2))
    pr = P.primes
    c0 = ints_to_poly(r0, pr)
    c1 = ints_to_poly(r1, pr)
    w = P.log2_beta
    mask = P.beta - 1
    acc0 = acc1 = None
    for i in range(P.ell + 1):
        d = [(v >> (w * i)) & mask for v in r2]
        if not any(d):
            continue
        dn = rns.ntt(ints_to_poly(d, pr), pr)
        g_ntt, a_ntt = _key_ntt(P, keys)
        g_t = rns.pmul(g_ntt[i], dn, pr)
        a_t = rns.pmul(a_ntt[i], dn, pr)
        acc0 = g_t if acc0 is None else rns.padd(acc0, g_t, pr)
        acc1 = a_t if acc1 is None else rns.padd(acc1, a_t, pr)
    if acc0 is not None:
        c0 = rns.padd(c0, rns.intt(acc0, pr), pr)
        c1 = rns.padd(c1, rns.intt(acc1, pr), pr)
    return Ct(c0, c1, a.lane, a.scale + b.scale, max(a.depth, b.depth) + 1)


# --- serialization ----------------------------------------------------------------


def ct_to_bytes(P: Params, ct: Ct) -> bytes:
    """Header [magic, 1, n, k, lane, scale mod 2^64, depth, 0] + c0 + c1 (fv.py:555-619)."""
    hdr = np.array(
        [MAGIC, 1, P.n, len(P.primes), ct.lane, ct.scale & (2**64 - 1), ct.depth, 0], dtype="<u8"
    )
    return hdr.tobytes() + ct.c0.astype("<u8").tobytes() + ct.c1.astype("<u8").tobytes()


def ct_from_bytes(P: Params, blob: bytes) -> Ct:
    w = np.frombuffer(blob[:64], dtype="<u8")
    if int(w[0]) != MAGIC or int(w[1]) != 1 or int(w[2]) != P.n or int(w[3]) != len(P.primes):
        raise ValueError("header mismatch")
    sc = int(w[5])
    sc = sc - (1 << 64) if sc >= 1 << 63 else sc
    k, n = len(P.primes), P.n
    body = np.frombuffer(blob[64:], dtype="<u8").astype(U64)
    if body.size != 2 * k * n:
        raise ValueError("body size mismatch")
    return Ct(body[: k * n].reshape(k, n).copy(), body[k * n :].reshape(k, n).copy(), int(w[4]), sc, int(w[6]))
