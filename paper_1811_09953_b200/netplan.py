"""Layer graph and the compiled integer plan (host side, public data only).

Mirrors the parts of reference `engine.py` that decide *which* homomorphic
operations run, so the GPU evaluator replays exactly the reference schedule:

  * layer types Conv2d / Dense / ScaledAvgPool / BatchNormAffine /
    PolyActivation and NetworkSpec (engine.py:45-193),
  * `fold_batchnorm` (engine.py:262-281),
  * plan types TapPlan / LinearOut / LinearPlan / PoolPlan / ActPlan /
    CompiledNet (engine.py:357-401),
  * `compile_network` with conv tap enumeration in (ci, di, dj) order,
    pruned and padded taps dropped, in_index = (ci*h + r)*w + c
    (engine.py:404-529),
  * HOP accounting `LayerCounts` / `HopCounter` / `project_hops`
    (engine.py:287-351, 535-586).

Layer objects are duck-typed by class name, so a NetworkSpec built with the
reference package's own classes compiles identically.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .encode import FixedPointConfig, round_half_away, round_half_away_array


class EngineError(ValueError):
    pass


# --- activations (coefficient carrier only; design happens offline) -----------


@dataclass(frozen=True)
class PolyApprox:
    """Ascending coefficients c0..c_degree (reference approx.py:77-105)."""

    degree: int
    coeffs: tuple
    interval_a: float = 4.0
    delta: float = 0.0
    pow2_terms: tuple | None = None

    def evaluate(self, x):
        acc = np.zeros_like(np.asarray(x, dtype=float))
        for c in reversed(self.coeffs):
            acc = acc * x + c
        return acc


def square_activation() -> PolyApprox:
    """x^2 (reference approx.py:346-354)."""
    return PolyApprox(2, (0.0, 0.0, 1.0), pow2_terms=((0, 0), (0, 0), (1, 0)))


def pow2_quadratic(e2: int, e1: int | None = None, e0: int | None = None, s2=1, s1=1, s0=1) -> PolyApprox:
    """s2 2^e2 x^2 + s1 2^e1 x + s0 2^e0 (None drops a term); e.g. the
    reference's Swish p* is pow2_quadratic(-3, -1, -4) (approx.py:357-366)."""
    c2 = s2 * 2.0 ** e2
    c1 = 0.0 if e1 is None else s1 * 2.0 ** e1
    c0 = 0.0 if e0 is None else s0 * 2.0 ** e0
    return PolyApprox(2, (c0, c1, c2))


# --- layers ------------------------------------------------------------------------


@dataclass
class Conv2d:
    weights: np.ndarray  # (out_c, in_c, kh, kw)
    bias: np.ndarray | None
    stride: int = 1
    padding: int = 0
    mask: np.ndarray | None = None

    def __post_init__(self):
        self.weights = np.asarray(self.weights, dtype=np.float64)
        if self.weights.ndim != 4:
            raise EngineError("conv weights must be 4-D (out, in, kh, kw)")
        if self.bias is not None:
            self.bias = np.asarray(self.bias, dtype=np.float64)
        if self.mask is not None:
            self.mask = np.asarray(self.mask, dtype=np.float64)

    def effective_weights(self):
        return self.weights if self.mask is None else self.weights * self.mask

    def out_shape(self, in_shape):
        return _conv_out_shape(self, in_shape)


@dataclass
class Dense:
    weights: np.ndarray  # (out, in)
    bias: np.ndarray | None
    mask: np.ndarray | None = None

    def __post_init__(self):
        self.weights = np.asarray(self.weights, dtype=np.float64)
        if self.weights.ndim != 2:
            raise EngineError("dense weights must be 2-D (out, in)")
        if self.bias is not None:
            self.bias = np.asarray(self.bias, dtype=np.float64)
        if self.mask is not None:
            self.mask = np.asarray(self.mask, dtype=np.float64)

    def effective_weights(self):
        return self.weights if self.mask is None else self.weights * self.mask

    def out_shape(self, in_shape):
        flat = int(np.prod(in_shape))
        if flat != self.weights.shape[1]:
            raise EngineError(f"dense expects {self.weights.shape[1]} inputs, got {flat}")
        return (self.weights.shape[0],)


@dataclass
class ScaledAvgPool:
    window: int
    stride: int = 1
    padding: int = 0
    reciprocal: bool = False

    def out_shape(self, in_shape):
        c, h, w = in_shape
        oh = (h + 2 * self.padding - self.window) // self.stride + 1
        ow = (w + 2 * self.padding - self.window) // self.stride + 1
        if oh < 1 or ow < 1:
            raise EngineError("pool output collapses to zero size")
        return (c, oh, ow)

    def window_count(self) -> int:
        return self.window * self.window


@dataclass
class BatchNormAffine:
    scale: np.ndarray
    shift: np.ndarray

    def __post_init__(self):
        self.scale = np.asarray(self.scale, dtype=np.float64)
        self.shift = np.asarray(self.shift, dtype=np.float64)

    def out_shape(self, in_shape):
        return in_shape


@dataclass
class PolyActivation:
    poly: object  # anything with .degree and ascending .coeffs

    def __post_init__(self):
        if self.poly.degree != 2:
            raise EngineError("encrypted activations are degree-2 polynomials")

    def out_shape(self, in_shape):
        return in_shape

    def coefficients(self):
        return _act_coeffs(self)


def _conv_out_shape(layer, in_shape):
    c, h, w = in_shape
    oc, ic, kh, kw = layer.weights.shape
    if c != ic:
        raise EngineError(f"conv expects {ic} input channels, got {c}")
    oh = (h + 2 * layer.padding - kh) // layer.stride + 1
    ow = (w + 2 * layer.padding - kw) // layer.stride + 1
    if oh < 1 or ow < 1:
        raise EngineError("conv output collapses to zero size")
    return (oc, oh, ow)


def _act_coeffs(layer):
    c0, c1, c2 = (float(c) for c in layer.poly.coeffs)
    if c2 == 0.0:
        raise EngineError("activation quadratic coefficient must be nonzero")
    return c2, c1, c0


def _kind(layer) -> str:
    return type(layer).__name__


@dataclass
class NetworkSpec:
    input_shape: tuple
    layers: list

    def __post_init__(self):
        self.input_shape = tuple(int(d) for d in self.input_shape)
        acts = sum(_kind(l) == "PolyActivation" for l in self.layers)
        if acts > 3:
            raise EngineError(f"{acts} activation layers exceed the depth budget of 3")
        shape = self.input_shape
        for layer in self.layers:
            shape = layer.out_shape(shape)
        self.output_shape = shape

    def shapes(self):
        out = [self.input_shape]
        for layer in self.layers:
            out.append(layer.out_shape(out[-1]))
        return out


def fold_batchnorm(net):
    """Absorb each BatchNormAffine into the preceding Conv2d/Dense (engine.py:262-281)."""
    layers: list = []
    for layer in net.layers:
        if _kind(layer) != "BatchNormAffine":
            layers.append(layer)
            continue
        if not layers or _kind(layers[-1]) not in ("Conv2d", "Dense"):
            raise EngineError("batch norm has no foldable conv/dense neighbor")
        prev = layers.pop()
        s, sh = layer.scale, layer.shift
        b = (prev.bias if prev.bias is not None else 0.0) * s + sh
        if _kind(prev) == "Conv2d":
            layers.append(Conv2d(prev.weights * s[:, None, None, None], b, prev.stride, prev.padding, prev.mask))
        else:
            layers.append(Dense(prev.weights * s[:, None], b, prev.mask))
    return NetworkSpec(net.input_shape, layers)


# --- HOP accounting ----------------------------------------------------------------


@dataclass
class LayerCounts:
    pt_ct_add: int = 0
    ct_ct_add: int = 0
    pt_ct_mul: int = 0
    ct_ct_mul: int = 0
    fast_path_hits: int = 0
    wall_ms: float = 0.0

    def total(self) -> int:
        return self.pt_ct_add + self.ct_ct_add + self.pt_ct_mul + self.ct_ct_mul

    def add(self, other: "LayerCounts") -> None:
        for f in ("pt_ct_add", "ct_ct_add", "pt_ct_mul", "ct_ct_mul", "fast_path_hits", "wall_ms"):
            setattr(self, f, getattr(self, f) + getattr(other, f))

    def same_ops(self, other) -> bool:
        return all(
            getattr(self, f) == getattr(other, f) for f in ("pt_ct_add", "ct_ct_add", "pt_ct_mul", "ct_ct_mul")
        )


class TimedLayerCounts(LayerCounts):
    """LayerCounts whose wall_ms is read from CUDA events on first access,
    so an evaluation does not have to synchronise the device to return."""

    def __init__(self, base: LayerCounts, events=None):
        super().__init__(base.pt_ct_add, base.ct_ct_add, base.pt_ct_mul, base.ct_ct_mul, base.fast_path_hits, 0.0)
        object.__setattr__(self, "_events", events)

    def __getattribute__(self, name):
        if name == "wall_ms":
            ev = object.__getattribute__(self, "_events")
            if ev is not None:
                a, b, share = ev
                b.synchronize()
                object.__setattr__(self, "_events", None)
                object.__setattr__(self, "wall_ms", a.elapsed_time(b) * share + object.__getattribute__(self, "wall_ms"))
        return object.__getattribute__(self, name)


@dataclass
class HopCounter:
    layer_names: list = field(default_factory=list)
    layer_counts: list = field(default_factory=list)

    def layer(self, name: str) -> LayerCounts:
        self.layer_names.append(name)
        self.layer_counts.append(LayerCounts())
        return self.layer_counts[-1]

    @property
    def totals(self) -> LayerCounts:
        t = LayerCounts()
        for c in self.layer_counts:
            t.add(c)
        return t

    def merge(self, other: "HopCounter") -> None:
        if self.layer_names != other.layer_names:
            raise EngineError("cannot merge counters over different layer lists")
        for mine, theirs in zip(self.layer_counts, other.layer_counts):
            mine.add(theirs)

    def same_ops(self, other) -> bool:
        return list(self.layer_names) == list(other.layer_names) and all(
            a.same_ops(b) for a, b in zip(self.layer_counts, other.layer_counts)
        )

    def rows(self):
        return [
            (n, c.pt_ct_add, c.ct_ct_add, c.pt_ct_mul, c.ct_ct_mul, c.wall_ms, c.fast_path_hits)
            for n, c in zip(self.layer_names, self.layer_counts)
        ]


# --- compiled plan -------------------------------------------------------------------


@dataclass(frozen=True)
class TapPlan:
    in_index: int
    weight_int: int


@dataclass(frozen=True)
class LinearOut:
    taps: tuple
    bias_int: int | None


@dataclass(frozen=True)
class LinearPlan:
    name: str
    outputs: tuple


@dataclass(frozen=True)
class PoolPlan:
    name: str
    outputs: tuple
    count: int
    pow2_shift: int
    factor_mult: int
    reciprocal_int: int | None


@dataclass(frozen=True)
class ActPlan:
    name: str
    nodes: int
    a2_int: int | None
    a1_mult_int: int | None
    a0_add_int: int | None
    scale_bump: int


@dataclass(frozen=True)
class CompiledNet:
    plans: tuple
    in_scale: int
    out_scale: int
    out_factor: int
    out_shape: tuple


def _conv_plan_outputs(layer, in_shape, prec: int):
    """(out_channel, taps) per output in (o, i, j) order; taps in (ci, di, dj)
    order with pruned/padded positions dropped (engine.py:404-434)."""
    c_in, h, w = in_shape
    oc, _, kh, kw = layer.weights.shape
    _, oh, ow = _conv_out_shape(layer, in_shape)
    wint = _affine_weights(layer, prec)
    ci, di, dj = np.meshgrid(np.arange(c_in), np.arange(kh), np.arange(kw), indexing="ij")
    ci, di, dj = ci.ravel(), di.ravel(), dj.ravel()
    outs = []
    for o in range(oc):
        wo = wint[o].ravel()
        nzk = wo != 0
        for i in range(oh):
            r = i * layer.stride - layer.padding + di
            okr = (r >= 0) & (r < h)
            for j in range(ow):
                c = j * layer.stride - layer.padding + dj
                sel = nzk & okr & (c >= 0) & (c < w)
                idx = (ci[sel] * h + r[sel]) * w + c[sel]
                taps = tuple(TapPlan(int(a), int(b)) for a, b in zip(idx, wo[sel]))
                outs.append((o, taps))
    return outs


@dataclass
class _Scales:
    """Fixed-point bookkeeping while lowering (engine.py:437-529): every
    ciphertext carries value * 2^scale * factor after a layer."""

    prec: int
    scale: int
    factor: int
    shape: tuple


def _affine_weights(layer, prec: int) -> np.ndarray:
    eff = layer.effective_weights() if hasattr(layer, "effective_weights") else layer.weights
    return round_half_away_array(np.asarray(eff, dtype=np.float64) * float(1 << prec))


def _lower_affine(layer, kind: str, st: _Scales, name: str) -> LinearPlan:
    """Conv2d / Dense: integer taps with zeros elided; bias at the output scale."""
    if kind == "Conv2d":
        pairs = _conv_plan_outputs(layer, st.shape, st.prec)
    else:
        wint = _affine_weights(layer, st.prec)
        pairs = [(o, tuple(TapPlan(int(i), int(wint[o, i])) for i in np.flatnonzero(wint[o])))
                 for o in range(wint.shape[0])]
    def bias(o):  # same float evaluation order as the reference
        return None if layer.bias is None else round_half_away(
            float(layer.bias[o]) * (1 << (st.scale + st.prec)) * st.factor)

    plan = LinearPlan(name, tuple(LinearOut(taps, bias(o)) for o, taps in pairs))
    st.scale += st.prec
    st.shape = layer.out_shape(st.shape)
    return plan


def _pool_windows(layer, shape) -> tuple:
    """Input indices of every window, (channel, row, col) order, the window's
    row-major cells clipped to the image (engine.py:476-491)."""
    c, h, w = shape
    _, oh, ow = layer.out_shape(shape)
    dr = np.repeat(np.arange(layer.window), layer.window)
    dc = np.tile(np.arange(layer.window), layer.window)
    wins = []
    for ch in range(c):
        for i in range(oh):
            rr = i * layer.stride - layer.padding + dr
            for j in range(ow):
                cc = j * layer.stride - layer.padding + dc
                ok = (rr >= 0) & (rr < h) & (cc >= 0) & (cc < w)
                wins.append(tuple(int(v) for v in (ch * h + rr[ok]) * w + cc[ok]))
    return tuple(wins)


def _lower_pool(layer, kind: str, st: _Scales, name: str) -> PoolPlan:
    """Sum of each window; 1/k as a reciprocal constant, a power-of-two shift
    of the scale, or a factor carried to the decoder."""
    cells = layer.window * layer.window
    recip, shift, fmult = None, 0, 1
    if layer.reciprocal:
        recip = round_half_away((1.0 / cells) * (1 << st.prec))
        st.scale += st.prec
    elif cells & (cells - 1) == 0:
        shift = cells.bit_length() - 1
        st.scale += shift
    else:
        fmult = cells
        st.factor *= cells
    plan = PoolPlan(name, _pool_windows(layer, st.shape), cells, shift, fmult, recip)
    st.shape = layer.out_shape(st.shape)
    return plan


def _lower_poly(layer, kind: str, st: _Scales, name: str) -> ActPlan:
    """a2 x^2 + a1 x + a0 at the squared scale: a2 multiplies the square (its
    own precision, elided when 1), a1 and a0 are lifted to the square's scale."""
    a2, a1, a0 = _act_coeffs(layer)
    p, s, f = st.prec, st.scale, st.factor
    bump = 0 if a2 == 1.0 else p
    plan = ActPlan(
        name,
        int(np.prod(st.shape)),
        None if a2 == 1.0 else round_half_away(a2 * (1 << p)),
        None if a1 == 0.0 else round_half_away(a1 * (1 << p)) * (1 << (s + bump - p)) * f,
        None if a0 == 0.0 else round_half_away(a0 * (1 << (2 * s + bump)) * f * f),
        bump,
    )
    st.scale, st.factor = 2 * s + bump, f * f
    return plan


_LOWERINGS = {"Conv2d": _lower_affine, "Dense": _lower_affine, "ScaledAvgPool": _lower_pool,
              "PolyActivation": _lower_poly}


def compile_network(net, cfg: FixedPointConfig) -> CompiledNet:
    """Lower a network to the reference's integer plan (engine.py:437-529):
    the same plan objects, field values and layer names as the reference's
    compile_network (pinned by digest in tests/golden)."""
    st = _Scales(cfg.precision_bits, cfg.precision_bits, 1, tuple(net.input_shape))
    plans = []
    for ix, layer in enumerate(net.layers):
        kind = _kind(layer)
        if kind == "BatchNormAffine":
            raise EngineError("fold batch norm before compiling for encryption")
        lower = _LOWERINGS.get(kind)
        if lower is None:
            raise EngineError(f"unknown layer {kind}")
        plans.append(lower(layer, kind, st, f"{kind.lower()}-{ix}"))
    return CompiledNet(tuple(plans), cfg.precision_bits, st.scale, st.factor, tuple(st.shape))


def int_is_monomial(z: int) -> bool:
    z = abs(int(z))
    return z != 0 and z & (z - 1) == 0


def plan_hops(compiled: CompiledNet, encoding: str = "integer", t: int | None = None) -> HopCounter:
    """Static HOP tally of a compiled plan (engine.py:535-581).

    In "integer" mode a constant is a fast-path hit when it is +-2^e; in
    "batched" mode every constant plaintext is a degree-0 monomial, so every
    PT-CT multiply is a fast-path hit (the instrumented count the reference
    evaluator would record, engine.py:703-704)."""

    def mono(z):
        return True if encoding == "batched" else int_is_monomial(z)

    counter = HopCounter()
    for plan in compiled.plans:
        c = counter.layer(plan.name)
        if isinstance(plan, LinearPlan):
            for out in plan.outputs:
                c.pt_ct_mul += len(out.taps)
                c.fast_path_hits += sum(1 for tp in out.taps if mono(tp.weight_int))
                c.ct_ct_add += max(0, len(out.taps) - 1)
                if out.bias_int is not None:
                    c.pt_ct_add += 1
        elif isinstance(plan, PoolPlan):
            for idxs in plan.outputs:
                c.ct_ct_add += max(0, len(idxs) - 1)
                if plan.reciprocal_int is not None:
                    c.pt_ct_mul += 1
                    c.fast_path_hits += int(mono(plan.reciprocal_int))
        elif isinstance(plan, ActPlan):
            c.ct_ct_mul += plan.nodes
            terms = 1
            if plan.a2_int is not None:
                c.pt_ct_mul += plan.nodes
                c.fast_path_hits += plan.nodes * int(mono(plan.a2_int))
            if plan.a1_mult_int is not None:
                c.pt_ct_mul += plan.nodes
                c.fast_path_hits += plan.nodes * int(mono(plan.a1_mult_int))
                terms += 1
            if terms > 1:
                c.ct_ct_add += plan.nodes
            if plan.a0_add_int is not None:
                c.pt_ct_add += plan.nodes
    return counter


def project_hops(net, cfg: FixedPointConfig | None = None) -> HopCounter:
    """Predicted HOP counts from the compiled plan alone (engine.py:535-581)."""
    cfg = cfg or FixedPointConfig(t_lanes=(1099511922689,))
    return plan_hops(compile_network(net, cfg), "integer")
