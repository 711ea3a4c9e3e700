"""The five BASELINE.json workloads as seeded synthetic inputs.

Seeds: inputs 0, weights 1, keygen 2, encryption 3.  No dataset is used;
the configurations borrow MNIST / CIFAR / feature-head *shapes* only.

Weights follow the reference's offline compression recipe, restated here
so the bench can rebuild them without the reference installed:
  * `prune_mask`: keep ceil(keep*N) largest |w|, ties by index
    (reference compress.py:68-85),
  * `quant_bounds(k=5)`: n1 = floor(log2(4s/3)), n2 = n1 - 7
    (compress.py:88-114),
  * `snap_pow2`: arithmetic-midpoint bins on the 2^e ladder
    (compress.py:117-143),
then exponents clamped into [-6, 0] (the +-[2^-6, 2^0] range of the
configs).  `tests/golden/configs.json` pins the compiled plans and HOP
counts produced from these nets against the reference's own
`compress` + `compile_network` + `project_hops`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import netplan as npn
from .encode import FixedPointConfig

T_BATCH = 65537
PREC = 6
SEED_INPUT, SEED_WEIGHTS, SEED_KEYS, SEED_ENC = 0, 1, 2, 3


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


def find_ntt_primes(n: int, count: int, bits: int = 55, exclude=()) -> list[int]:
    """Same scan as reference modmath.py:118-133 (step first, then test)."""
    step = 2 * n
    p = (1 << bits) // step * step + 1
    out, skip = [], set(exclude)
    while len(out) < count:
        p += step
        if p not in skip and _is_prime(p):
            out.append(p)
    return out


# --- offline weight compression (restated) ---------------------------------------


def prune_keep(w: np.ndarray, keep: float) -> np.ndarray:
    n = w.size
    k = math.ceil(keep * n)
    flat = np.abs(w.ravel())
    order = np.lexsort((np.arange(n), -flat))
    mask = np.zeros(n)
    mask[order[:k]] = 1.0
    return mask.reshape(w.shape)


def quantize_pow2(w: np.ndarray, mask: np.ndarray, kbits: int = 5, emin: int = -6, emax: int = 0) -> np.ndarray:
    eff = w * mask
    s = float(np.abs(eff).max())
    n1 = int(math.floor(math.log2(4.0 * s / 3.0)))
    n2 = n1 + 1 - (1 << (kbits - 1)) // 2
    out = np.zeros_like(eff).ravel()
    flat = eff.ravel()
    for i in np.nonzero(flat)[0]:
        mag = abs(flat[i])
        if mag < 0.75 * 2.0 ** n2:
            continue
        e = min(n1, math.floor(math.log2(mag * 4.0 / 3.0)))
        e = min(max(e, emin), emax)
        out[i] = math.copysign(2.0 ** e, flat[i])
    return out.reshape(w.shape)


def compressed(w: np.ndarray, keep: float) -> np.ndarray:
    return quantize_pow2(w, prune_keep(w, keep))


# --- configurations ------------------------------------------------------------------


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    limbs: int
    prime_bits: int
    t: int
    beta: int
    prec: int
    description: str

    @property
    def primes(self) -> tuple:
        return tuple(find_ntt_primes(self.n, self.limbs, bits=self.prime_bits))

    @property
    def slots(self) -> int:
        return self.n

    def fixed_point(self) -> FixedPointConfig:
        return FixedPointConfig((self.t,), self.prec)


WORKLOADS = {
    "cfg1": Workload("cfg1", 4096, 3, 36, T_BATCH, 1 << 32, PREC, "dense 784->100 (keep 0.2) + x^2"),
    "cfg2": Workload("cfg2", 8192, 4, 50, T_BATCH, 1 << 32, PREC, "MNIST-shaped conv5x5s2(5) + act + dense 845->100 + act + dense 100->10"),
    "cfg3": Workload("cfg3", 16384, 6, 50, T_BATCH, 1 << 32, PREC, "CIFAR-shaped conv3x3(16) + act + conv3x3s2(32) + act + dense 8192->128 + act + dense 128->10"),
    "cfg4": Workload("cfg4", 8192, 4, 50, T_BATCH, 1 << 32, PREC, "feature head dense 2048->256 + act + dense 256->14"),
    "cfg5": Workload("cfg5", 16384, 8, 50, T_BATCH, 1 << 134, PREC, "primitive sweep: NTT, square+relin (dnum=3), 1024-term sparse MAC"),
}


def _he(rng, *shape):
    fan_in = int(np.prod(shape[1:])) if len(shape) > 1 else shape[0]
    return rng.normal(0.0, math.sqrt(2.0 / fan_in), shape)


def act_pow2():
    """2^-3 x^2 + 2^-1 x (power-of-two quadratic, no constant)."""
    return npn.pow2_quadratic(-3, -1)


def build_network(name: str):
    """Synthetic pruned + pow2-quantized network of a workload (weights seed 1)."""
    rng = np.random.default_rng(SEED_WEIGHTS)
    L = npn
    if name == "cfg1":
        w = rng.normal(0.0, 0.05, (100, 784))
        return L.NetworkSpec((784,), [L.Dense(compressed(w, 0.20), None), L.PolyActivation(L.square_activation())])
    if name == "cfg2":
        c1 = _he(rng, 5, 1, 5, 5)
        d1 = _he(rng, 100, 845)
        d2 = _he(rng, 10, 100)
        return L.NetworkSpec(
            (1, 28, 28),
            [
                L.Conv2d(compressed(c1, 0.20), None, stride=2, padding=1),
                L.PolyActivation(act_pow2()),
                L.Dense(compressed(d1, 0.10), None),
                L.PolyActivation(act_pow2()),
                L.Dense(compressed(d2, 0.20), None),
            ],
        )
    if name == "cfg3":
        c1 = _he(rng, 16, 3, 3, 3)
        c2 = _he(rng, 32, 16, 3, 3)
        d1 = _he(rng, 128, 8192)
        d2 = _he(rng, 10, 128)
        return L.NetworkSpec(
            (3, 32, 32),
            [
                L.Conv2d(compressed(c1, 0.15), None, stride=1, padding=1),
                L.PolyActivation(act_pow2()),
                L.Conv2d(compressed(c2, 0.15), None, stride=2, padding=1),
                L.PolyActivation(act_pow2()),
                L.Dense(compressed(d1, 0.15), None),
                L.PolyActivation(act_pow2()),
                L.Dense(compressed(d2, 0.15), None),
            ],
        )
    if name == "cfg4":
        d1 = _he(rng, 256, 2048)
        d2 = _he(rng, 14, 256)
        return L.NetworkSpec(
            (2048,),
            [L.Dense(compressed(d1, 0.10), None), L.PolyActivation(act_pow2()), L.Dense(compressed(d2, 0.15), None)],
        )
    raise KeyError(name)


def build_inputs(name: str, slots: int | None = None) -> np.ndarray:
    """Integer input values (inputs, slots) for a workload (inputs seed 0).

    Returns the raw values v; the slot encoder scales them by 2^prec
    (round_half_away(v * 2^prec), engine.py:623)."""
    W = WORKLOADS[name]
    s = W.n if slots is None else slots
    rng = np.random.default_rng(SEED_INPUT)
    if name in ("cfg1", "cfg2"):
        return rng.integers(0, 256, (784, s)).astype(np.int64)
    if name == "cfg3":
        return rng.integers(0, 256, (3072, s)).astype(np.int64)
    if name == "cfg4":
        f = np.maximum(0.0, rng.normal(0.0, 1.0, (2048, s)))
        return np.rint(np.clip(f, 0.0, 4.0) * 255.0 / 4.0).astype(np.int64)
    raise KeyError(name)


def mac_sweep_plan(n_out: int = 4096, n_in: int = 4096, terms: int = 1024, seed: int = 1):
    """cfg5's sparse pow2 MAC: each output draws `terms` distinct inputs,
    exponent e in [0, 6], random sign."""
    rng = np.random.default_rng(seed)
    outs = []
    for _ in range(n_out):
        idx = np.sort(rng.choice(n_in, size=terms, replace=False))
        e = rng.integers(0, 7, terms)
        sg = rng.integers(0, 2, terms) * 2 - 1
        outs.append(npn.LinearOut(tuple(npn.TapPlan(int(i), int(s) << int(x)) for i, x, s in zip(idx, e, sg)), None))
    return npn.LinearPlan("mac-sweep", tuple(outs))
