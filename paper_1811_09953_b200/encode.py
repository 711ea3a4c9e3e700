"""Fixed-point <-> plaintext encoders (host side; mirrors reference `encode.py`).

* `encode_integer` - base-2 integer encoder: bit i of |z| becomes
  coefficient 1 (z > 0) or t-1 (z < 0) at x^i (reference encode.py:64-78).
* `round_half_away` - nearest integer, halves away from zero (encode.py:96-98).
* `decode_integer`, `encode_fixed`, `decode_fixed`, `crt_combine` - the
  client-side decoders (encode.py:81-159); they never touch the GPU.
* `slot_encode` / `slot_decode` - the SIMD batching encoder used by the
  batched configurations: plaintext = inverse negacyclic NTT over Z_t of the
  slot vector, decode = forward NTT (the reference has no batching encoder;
  SURVEY.md sec. 0.5 pins this construction to `ring.ntt_inverse/ntt_forward`
  over RingContext(n, (t,))).  The transforms run on the GPU library.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


class EncodeError(ValueError):
    pass


class CapacityError(EncodeError):
    pass


@dataclass(frozen=True)
class FixedPointConfig:
    t_lanes: tuple
    precision_bits: int = 15

    def __post_init__(self):
        if self.precision_bits < 1:
            raise EncodeError("precision_bits must be >= 1")
        if not self.t_lanes:
            raise EncodeError("at least one plaintext lane required")
        lanes = [int(t) for t in self.t_lanes]
        for i in range(len(lanes)):
            for j in range(i + 1, len(lanes)):
                if math.gcd(lanes[i], lanes[j]) != 1:
                    raise EncodeError("plaintext lanes must be pairwise coprime")

    @property
    def lane_product(self) -> int:
        return math.prod(int(t) for t in self.t_lanes)


def round_half_away(v: float) -> int:
    """Round to nearest, ties away from zero (reference encode.py:96-98)."""
    v = float(v)
    if v >= 0:
        return int(math.floor(v + 0.5))
    return -int(math.floor(-v + 0.5))


def round_half_away_array(v: np.ndarray) -> np.ndarray:
    """Vectorised `round_half_away` (identical float64 operations, int64 out).

    Magnitudes at or above 2^62 (or non-finite values) would wrap in int64;
    they take the scalar Python-int path instead (an object array, exact like
    the reference's big-int rounding, encode.py:96-98)."""
    v = np.asarray(v, dtype=np.float64)
    if v.size and not (np.isfinite(v).all() and np.abs(v).max() < 2.0 ** 62):
        return np.array([round_half_away(x) for x in v.ravel()], dtype=object).reshape(v.shape)
    mag = np.floor(np.abs(v) + 0.5)
    return np.where(v >= 0, mag, -mag).astype(np.int64)


def integer_bits(z: int) -> list[int]:
    """Positions of the set bits of |z| (the support of encode_integer(z))."""
    mag = abs(int(z))
    out = []
    i = 0
    while mag:
        if mag & 1:
            out.append(i)
        mag >>= 1
        i += 1
    return out


def encode_integer(z: int, t: int):
    """PlainPoly of the binary expansion of z (reference encode.py:64-78)."""
    from .fv import PlainPoly

    z = int(z)
    if z == 0:
        return PlainPoly.zero(t)
    bits = integer_bits(z)
    coeffs = np.zeros(bits[-1] + 1, dtype=np.uint64)
    coeffs[bits] = 1 if z > 0 else t - 1
    return PlainPoly(t, coeffs)


def decode_integer(p) -> int:
    """Evaluate at x=2 with centered coefficients (reference encode.py:81-93)."""
    value = 0
    for i, c in enumerate(p.centered()):
        value += c << i
    if abs(value) >= 1 << 62:
        raise EncodeError(f"decoded magnitude {value} exceeds 62-bit contract")
    return value


@dataclass(frozen=True)
class EncodedValue:
    polys: tuple
    scale_exponent: int


def encode_fixed(v: float, cfg: FixedPointConfig) -> EncodedValue:
    z = round_half_away(float(v) * (1 << cfg.precision_bits))
    if abs(z) >= 1 << 62:
        raise EncodeError("value too large for fixed-point range")
    return EncodedValue(tuple(encode_integer(z, int(t)) for t in cfg.t_lanes), cfg.precision_bits)


def crt_combine(residues, moduli) -> int:
    """Centered CRT representative in (-M/2, M/2] (reference encode.py:110-118)."""
    M = math.prod(int(m) for m in moduli)
    acc = 0
    for r, m in zip(residues, moduli):
        part = M // int(m)
        acc += int(r) * part * pow(part % int(m), int(m) - 2, int(m))
    acc %= M
    return acc - M if acc > M // 2 else acc


def decode_fixed(plains, scale_exponent: int, cfg: FixedPointConfig, scale_factor: int = 1) -> float:
    """Coefficient-wise CRT, evaluate at 2, descale (reference encode.py:121-159)."""
    plains = list(plains)
    if len(plains) != len(cfg.t_lanes):
        raise EncodeError(f"expected {len(cfg.t_lanes)} lane plaintexts, got {len(plains)}")
    moduli = [int(t) for t in cfg.t_lanes]
    for p, t in zip(plains, moduli):
        if p.t != t:
            raise EncodeError("lane plaintext modulus out of order")
    length = max((p.coeffs.size for p in plains), default=0)
    trip = cfg.lane_product >> 2
    value = 0
    for i in range(length):
        if len(moduli) == 1:
            p = plains[0]
            c = p.centered()[i] if i < p.coeffs.size else 0
        else:
            res = [int(p.coeffs[i]) if i < p.coeffs.size else 0 for p in plains]
            c = crt_combine(res, moduli)
            if abs(c) > trip:
                raise EncodeError(f"coefficient {i} reconstructs near capacity ({c})")
        value += c << i if c >= 0 else -((-c) << i)
    return value / (2.0 ** scale_exponent) / scale_factor


def centered_mod(v: np.ndarray, t: int) -> np.ndarray:
    """Canonical residues mod t -> signed representatives in (-t/2, t/2]."""
    v = np.asarray(v).astype(np.int64)
    return np.where(v > t // 2, v - t, v)
