"""Number-theory helpers used to instantiate parameters (oracle; test infra only).

Restates reference `pkg/src/hecnet/modmath.py:93-157`:
  * deterministic Miller-Rabin over the first twelve prime bases (:93-115),
  * NTT-friendly prime scan upward from 2**bits in steps of 2n (:118-133),
  * the smallest-generator primitive 2n-th root rule (:136-149),
  * bit reversal (:152-157).
"""

from __future__ import annotations

WITNESSES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(v: int) -> bool:
    """Deterministic Miller-Rabin (reference modmath.py:93-115)."""
    if v < 2:
        return False
    for w in WITNESSES:
        if v % w == 0:
            return v == w
    odd, twos = v - 1, 0
    while not odd & 1:
        odd >>= 1
        twos += 1
    for w in WITNESSES:
        x = pow(w, odd, v)
        if x == 1 or x == v - 1:
            continue
        for _ in range(twos - 1):
            x = x * x % v
            if x == v - 1:
                break
        else:
            return False
    return True


def ntt_primes(n: int, count: int, bits: int = 55, exclude=()) -> list[int]:
    """Primes p = 1 mod 2n strictly above the first grid point >= 2**bits - 2n.

    Reference modmath.py:118-133: start at floor(2^bits / 2n) * 2n + 1 and
    step by 2n *before* the first test, skipping `exclude`.
    """
    stride = 2 * n
    cand = ((1 << bits) // stride) * stride + 1
    banned = set(int(e) for e in exclude)
    found: list[int] = []
    while len(found) < count:
        cand += stride
        if cand not in banned and is_prime(cand):
            found.append(cand)
    return found


def root_2n(q: int, n: int) -> int:
    """Smallest g in [2, 4096) whose g^((q-1)/2n) has order exactly 2n.

    Reference modmath.py:136-149.
    """
    if (q - 1) % (2 * n):
        raise ValueError(f"{q} is not 1 mod {2 * n}")
    e = (q - 1) // (2 * n)
    for g in range(2, 4096):
        r = pow(g, e, q)
        if pow(r, n, q) == q - 1:
            return r
    raise ValueError("no primitive root found")


def bitrev(x: int, nbits: int) -> int:
    """Reverse the low `nbits` bits of x (reference modmath.py:152-157)."""
    return int(format(x, f"0{nbits}b")[::-1], 2) if nbits else 0
