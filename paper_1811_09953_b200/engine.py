"""Encrypted evaluation of a compiled network on B200 (mirrors reference engine.py).

`eval_encrypted(net, tensor, ek, cfg, workers=1)` keeps the reference
signature and semantics (engine.py:651-774): it compiles the same integer
plan (`netplan.compile_network`), tallies the same HOP counters, carries the
same scale / factor / depth metadata, and produces ciphertexts that are
bit-identical to the reference evaluator's.  Instead of one `fv.*` call per
HOP it issues one fused kernel per layer:

  * linear layer / pool:  `fcn_linear_mac` -- every (tap x encoded-term)
    becomes a signed monomial term c * x^r applied to an input ciphertext
    and accumulated exactly (mul_pt + add_ct chain, engine.py:698-743),
    then `fcn_add_plain_terms` for the bias (add_pt, engine.py:713-715);
  * activation: `fcn_mul_ct_ex` on all nodes (square + relinearisation)
    with a2*sq + a1*x fused into its last kernels when the multipliers are
    constant plaintexts (batched encoding), else `fcn_mul_ct` followed by
    one `fcn_linear_mac` over [sq ; x]; then add_pt(a0) (engine.py:744-770).

Sharded evaluation (`dist.py`) passes extra destinations (`fanout`): the
final kernel of a layer stores its rows into every rank's buffer.

Plaintext constants are encoded as in the reference (`encoding="integer"`:
base-2 encoder, a +-1 term per set bit at x^bit) or, for the SIMD-batched
configurations, as constant polynomials (`encoding="batched"`: one term
c = centered(z mod t) at x^0).  A CipherTensor holds one [B][2][k][n]
device buffer -- byte-identical to the serialized ciphertext bodies.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import ctypes as C

import numpy as np

from . import _lib
from . import device as dev
from . import fv
from . import mac_tc
from .encode import FixedPointConfig, decode_fixed, encode_integer, integer_bits, round_half_away
from .fv import Ciphertext, EncryptionParams, EvalKeys, FVError, PublicKey, SecretKey
from .netplan import (  # noqa: F401  (re-exported: reference engine API surface)
    ActPlan,
    BatchNormAffine,
    CompiledNet,
    Conv2d,
    Dense,
    EngineError,
    HopCounter,
    LayerCounts,
    LinearOut,
    LinearPlan,
    NetworkSpec,
    PolyActivation,
    PolyApprox,
    PoolPlan,
    ScaledAvgPool,
    TapPlan,
    compile_network,
    fold_batchnorm,
    int_is_monomial,
    plan_hops,
    project_hops,
    square_activation,
)
from .netplan import TimedLayerCounts

ENCODINGS = ("integer", "batched")


# ----------------------------------------------------------------- tensors


class CipherTensor:
    """Grid of ciphertexts sharing lane and scale (engine.py:592-607).

    `buf` is a [count][2][k][n] device buffer; `depths` the per-element
    multiplicative depth (host int array)."""

    def __init__(self, shape, cts=None, scale_exponent: int = 0, scale_factor: int = 1, *, buf=None, params=None,
                 lane: int = 0, depths=None, scales=None):
        self.shape = tuple(int(d) for d in shape)
        count = int(np.prod(self.shape))
        if cts is not None:
            cts = list(cts)
            if len(cts) != count:
                raise EngineError("ciphertext count does not match tensor shape")
            import torch

            params = cts[0].params
            lane = cts[0].lane
            buf = torch.stack([torch.stack([c.c0.data, c.c1.data]) for c in cts]).contiguous()
            depths = np.array([c.mul_depth for c in cts], dtype=np.int64)
            scales = np.array([c.scale_exponent for c in cts], dtype=np.int64)
        if buf is None or params is None:
            raise EngineError("CipherTensor needs ciphertexts or a device buffer with params")
        if buf.shape[0] != count:
            raise EngineError("ciphertext count does not match tensor shape")
        self.buf = buf
        self.params = params
        self.lane = int(lane)
        self.scale_exponent = int(scale_exponent)
        self.scale_factor = int(scale_factor)
        self.depths = np.zeros(count, dtype=np.int64) if depths is None else np.asarray(depths, dtype=np.int64)
        # per-ciphertext scale_exponent (serialized in each header, fv.py:555-571);
        # it can differ from the tensor-level exponent after pooling (engine.py:711-743)
        self.scales = (
            np.full(count, self.scale_exponent, dtype=np.int64) if scales is None else np.asarray(scales, dtype=np.int64)
        )

    @property
    def cts(self) -> list:
        return [
            fv.ciphertext_from_buffer(self.params, self.buf[i], self.lane, int(self.scales[i]), int(self.depths[i]))
            for i in range(self.buf.shape[0])
        ]

    def __len__(self):
        return self.buf.shape[0]

    def host_bodies(self) -> np.ndarray:
        """[count][2][k][n] uint64 host copy (the serialized bodies)."""
        return dev.to_host(self.buf)


def encrypt_tensor(pk: PublicKey, params: EncryptionParams, values, cfg: FixedPointConfig, lane: int = 0, rng=None) -> CipherTensor:
    """One ciphertext per scalar, base-2 integer encoding (engine.py:610-627).

    Byte-identical to the reference for the same rng (same draw order)."""
    values = np.asarray(values, dtype=np.float64)
    rng = rng if isinstance(rng, np.random.Generator) else np.random.default_rng(rng)
    t = int(params.t_lanes[lane])
    zs = [round_half_away(float(v) * (1 << cfg.precision_bits)) for v in values.ravel()]
    width = max([1] + [abs(z).bit_length() for z in zs])
    if width > params.n:
        raise FVError("plaintext degree exceeds ring degree")
    cen = np.zeros((len(zs), width), dtype=np.int64)
    for i, z in enumerate(zs):
        if z:
            cen[i, integer_bits(z)] = 1 if z > 0 else -1
    buf = fv.encrypt_batch(pk, params, cen, lane, rng)
    return CipherTensor(tuple(values.shape), scale_exponent=cfg.precision_bits, buf=buf, params=params, lane=lane)


# ------------------------------------------------------------- slot encoder


def _t_ring(params: EncryptionParams, lane: int):
    from .ring import RingContext

    return RingContext.create(params.n, (int(params.t_lanes[lane]),))


def slot_encode(params: EncryptionParams, slots: np.ndarray, lane: int = 0) -> np.ndarray:
    """(count, <=n) slot integers -> (count, n) centered plaintext coefficients.

    Plaintext = inverse negacyclic NTT over Z_t of the slot vector (SURVEY
    sec. 0.5); runs in libfcn over the t-ring."""
    t = int(params.t_lanes[lane])
    s = np.asarray(slots, dtype=np.int64)
    count = s.shape[0]
    full = np.zeros((count, params.n), dtype=np.int64)
    full[:, : s.shape[1]] = np.mod(s, t)
    tr = _t_ring(params, lane)
    d = dev.to_device(full)
    _lib.check(_lib.lib().fcn_ntt_inverse(tr.handle().ptr, d.data_ptr(), count, 1, 0, dev.stream_ptr()), FVError)
    coeffs = dev.to_host(d).astype(np.int64)
    return np.where(coeffs > t // 2, coeffs - t, coeffs)


def slot_decode(params: EncryptionParams, plain: np.ndarray, lane: int = 0) -> np.ndarray:
    """(count, n) plaintext coefficients mod t -> (count, n) slot values in [0, t)."""
    t = int(params.t_lanes[lane])
    d = dev.to_device(np.mod(np.asarray(plain, dtype=np.int64), t))
    tr = _t_ring(params, lane)
    _lib.check(_lib.lib().fcn_ntt_forward(tr.handle().ptr, d.data_ptr(), d.shape[0], 1, 0, dev.stream_ptr()), FVError)
    return dev.to_host(d).astype(np.int64)


def encrypt_tensor_batched(pk: PublicKey, params: EncryptionParams, values, cfg: FixedPointConfig, lane: int = 0, rng=None) -> CipherTensor:
    """SIMD batch: values (*shape, slots); element e's ciphertext packs
    round_half_away(v * 2^prec) mod t of every slot (engine.py:623 rule)."""
    values = np.asarray(values)
    shape = values.shape[:-1]
    flat = values.reshape(-1, values.shape[-1])
    if np.issubdtype(flat.dtype, np.integer):
        z = flat.astype(np.int64) << cfg.precision_bits
    else:
        v = flat.astype(np.float64) * float(1 << cfg.precision_bits)
        mag = np.floor(np.abs(v) + 0.5)
        z = np.where(v >= 0, mag, -mag).astype(np.int64)
    cen = slot_encode(params, z, lane)
    rng = rng if isinstance(rng, np.random.Generator) else np.random.default_rng(rng)
    buf = fv.encrypt_batch(pk, params, cen, lane, rng)
    return CipherTensor(shape, scale_exponent=cfg.precision_bits, buf=buf, params=params, lane=lane)


def decrypt_tensor(sk: SecretKey, tensor: CipherTensor) -> list:
    """Per-element PlainPoly (engine.py:630-631)."""
    t = int(tensor.params.t_lanes[tensor.lane])
    ms = fv.decrypt_batch(sk, tensor.params, tensor.buf, tensor.lane)
    return [fv.PlainPoly(t, m) for m in ms]


def decrypt_tensor_slots(sk: SecretKey, tensor: CipherTensor) -> np.ndarray:
    """Batched mode: (count, n) decrypted slot values in [0, t)."""
    ms = fv.decrypt_batch(sk, tensor.params, tensor.buf, tensor.lane)
    return slot_decode(tensor.params, ms.astype(np.int64), tensor.lane)


def decode_lane_outputs(lane_plaintexts, tensor_shape, scale_exponent, scale_factor, cfg) -> np.ndarray:
    """Per-lane decrypted grids -> real-valued tensor (engine.py:634-648)."""
    count = int(np.prod(tensor_shape))
    out = np.zeros(count)
    for i in range(count):
        out[i] = decode_fixed([lane[i] for lane in lane_plaintexts], scale_exponent, cfg, scale_factor)
    return out.reshape(tensor_shape)


# ------------------------------------------------------------ plan lowering


def const_terms(z: int, t: int, n: int, encoding: str) -> list:
    """Signed monomial terms (rot, coef) of the plaintext encoding integer z.

    integer: encode_integer(z) (encode.py:64-78) -> +-1 at each set bit;
    batched: PlainPoly(t, [z mod t]) -> centered(z mod t) at x^0."""
    z = int(z)
    if encoding == "batched":
        c = z % t
        if c == 0:
            raise FVError("zero plaintext multiplier: elide the operation instead")
        return [(0, c - t if c > t // 2 else c)]
    if z == 0:
        raise FVError("zero plaintext multiplier: elide the operation instead")
    bits = integer_bits(z)
    if bits[-1] >= n:
        raise FVError("plaintext degree exceeds ring degree")
    s = 1 if z > 0 else -1
    return [(b, s) for b in bits]


def plain_terms(z: int, t: int, n: int, encoding: str) -> list:
    """(pos, coef) of the plaintext added by add_pt(encode(z)); [] when zero."""
    z = int(z)
    if encoding == "batched":
        c = z % t
        return [] if c == 0 else [(0, c - t if c > t // 2 else c)]
    if z == 0:
        return []
    bits = integer_bits(z)
    if bits[-1] >= n:
        raise FVError("plaintext degree exceeds ring degree")
    s = 1 if z > 0 else -1
    return [(b, s) for b in bits]


@dataclass
class _Mac:
    rowptr: object
    col: object
    rot: object
    coef: object
    n_out: int
    n_terms: int
    no_rot: bool = False
    max_abs_coef: int = 0
    host: tuple | None = None  # (rowptr, col, coef) numpy: the tensor-core lowering's input
    tc: dict = field(default_factory=dict)  # (planes, cols, n_in) -> _TcPlan | None


@dataclass
class _Bias:
    ct_index: object
    pos: object
    coef: object
    n_terms: int


def _upload_mac(rowptr, col, rot, coef) -> _Mac:
    import torch

    d = "cuda"
    rot_a = np.asarray(rot, dtype=np.int64)
    coef_a = np.asarray(coef, dtype=np.int64)
    no_rot = bool(len(rot) == 0 or not np.any(rot_a))
    return _Mac(
        torch.as_tensor(np.asarray(rowptr, dtype=np.int32), device=d),
        torch.as_tensor(np.asarray(col, dtype=np.int32) if len(col) else np.zeros(1, np.int32), device=d),
        torch.as_tensor(rot_a.astype(np.int32) if len(rot) else np.zeros(1, np.int32), device=d),
        torch.as_tensor(coef_a if len(coef) else np.zeros(1, np.int64), device=d),
        len(rowptr) - 1,
        len(col),
        no_rot,
        int(np.abs(coef_a).max()) if len(coef) else 0,
        (np.asarray(rowptr, dtype=np.int64), np.asarray(col, dtype=np.int64), coef_a) if no_rot else None,
    )


def _upload_bias(idx, pos, coef) -> _Bias | None:
    import torch

    if not idx:
        return None
    d = "cuda"
    return _Bias(
        torch.as_tensor(np.asarray(idx, dtype=np.int32), device=d),
        torch.as_tensor(np.asarray(pos, dtype=np.int32), device=d),
        torch.as_tensor(np.asarray(coef, dtype=np.int64), device=d),
        len(idx),
    )


def _lower_linear(plan: LinearPlan, t: int, n: int, encoding: str):
    """CSR of monomial terms for a LinearPlan (vectorised for big layers)."""
    outs = plan.outputs
    counts = np.array([len(o.taps) for o in outs], dtype=np.int64)
    cols = np.fromiter((tp.in_index for o in outs for tp in o.taps), dtype=np.int64, count=int(counts.sum()))
    wts = [tp.weight_int for o in outs for tp in o.taps]
    small = all(abs(w) < (1 << 62) for w in wts)
    if encoding == "batched" and small:
        w = np.asarray(wts, dtype=np.int64)
        c = np.mod(w, t)
        if np.any(c == 0):
            raise FVError("zero plaintext multiplier: elide the operation instead")
        coef = np.where(c > t // 2, c - t, c)
        rowptr = np.concatenate([[0], np.cumsum(counts)])
        mac = (rowptr, cols, np.zeros_like(cols), coef)
    else:
        rowptr = [0]
        col, rot, coef = [], [], []
        k = 0
        for o in outs:
            for tp in o.taps:
                for r, c in const_terms(tp.weight_int, t, n, encoding):
                    col.append(tp.in_index)
                    rot.append(r)
                    coef.append(c)
                k += 0
            rowptr.append(len(col))
        mac = (rowptr, col, rot, coef)
    bidx, bpos, bcoef = [], [], []
    for o_i, o in enumerate(outs):
        if o.bias_int is not None:
            for p, c in plain_terms(o.bias_int, t, n, encoding):
                bidx.append(o_i)
                bpos.append(p)
                bcoef.append(c)
    taps = (np.concatenate([[0], np.cumsum(counts)]), cols)
    return _upload_mac(*mac), _upload_bias(bidx, bpos, bcoef), taps


def _lower_pool(plan: PoolPlan, t: int, n: int, encoding: str):
    rterms = [(0, 1)] if plan.reciprocal_int is None else const_terms(plan.reciprocal_int, t, n, encoding)
    rowptr, col, rot, coef = [0], [], [], []
    for idxs in plan.outputs:
        for i in idxs:
            for r, c in rterms:
                col.append(i)
                rot.append(r)
                coef.append(c)
        rowptr.append(len(col))
    counts = np.array([len(w) for w in plan.outputs], dtype=np.int64)
    taps = (np.concatenate([[0], np.cumsum(counts)]), np.fromiter((i for w in plan.outputs for i in w), dtype=np.int64))
    return _upload_mac(rowptr, col, rot, coef), None, taps


def _lower_act(plan: ActPlan, t: int, n: int, encoding: str, nodes: int | None = None):
    """MAC over [sq ; x]: a2 * sq[o] + a1 * x[o]; bias terms for a0."""
    a2 = [(0, 1)] if plan.a2_int is None else const_terms(plan.a2_int, t, n, encoding)
    a1 = [] if plan.a1_mult_int is None else const_terms(plan.a1_mult_int, t, n, encoding)
    N = plan.nodes if nodes is None else nodes
    per = len(a2) + len(a1)
    o = np.arange(N, dtype=np.int64)
    col = np.concatenate([np.repeat(o[:, None], len(a2), 1), np.repeat(o[:, None] + N, len(a1), 1)], axis=1).ravel()
    rot = np.tile(np.array([r for r, _ in a2] + [r for r, _ in a1], dtype=np.int64), N)
    coef = np.tile(np.array([c for _, c in a2] + [c for _, c in a1], dtype=np.int64), N)
    rowptr = np.arange(N + 1, dtype=np.int64) * per
    bidx, bpos, bcoef = [], [], []
    if plan.a0_add_int is not None:
        pt = plain_terms(plan.a0_add_int, t, n, encoding)
        for i in range(N):
            for p, c in pt:
                bidx.append(i)
                bpos.append(p)
                bcoef.append(c)
    identity = plan.a2_int is None and plan.a1_mult_int is None
    return _upload_mac(rowptr, col, rot, coef), _upload_bias(bidx, bpos, bcoef), identity


_lower_cache: dict = {}
_compile_cache: dict = {}


def _net_fingerprint(net) -> bytes:
    """Content hash of everything compile_network reads (weights, masks,
    biases, geometry, activation coefficients)."""
    import hashlib

    h = hashlib.blake2b(digest_size=16)
    h.update(repr(tuple(net.input_shape)).encode())
    for layer in net.layers:
        h.update(type(layer).__name__.encode())
        for attr in ("weights", "mask", "bias", "scale", "shift"):
            v = getattr(layer, attr, None)
            if v is not None:
                a = np.ascontiguousarray(v, dtype=np.float64)
                h.update(repr(a.shape).encode())
                h.update(a.tobytes())
        for attr in ("stride", "padding", "window", "reciprocal"):
            if hasattr(layer, attr):
                h.update(repr(getattr(layer, attr)).encode())
        poly = getattr(layer, "poly", None)
        if poly is not None:
            h.update(repr(tuple(float(c) for c in poly.coeffs)).encode())
    return h.digest()


_hops_cache: dict = {}


def _hops(compiled: CompiledNet, encoding: str, t: int) -> HopCounter:
    """Fresh HopCounter with the plan's static tally (cached per plan)."""
    key = (id(compiled), encoding, t)
    hit = _hops_cache.get(key)
    if hit is None or hit[0] is not compiled:
        hit = (compiled, plan_hops(compiled, encoding, t))
        _hops_cache[key] = hit
    tmpl = hit[1]
    out = HopCounter()
    for name, c in zip(tmpl.layer_names, tmpl.layer_counts):
        lc = out.layer(name)
        lc.add(c)
        lc.wall_ms = 0.0
    return out


def _compiled(net, cfg) -> CompiledNet:
    """compile_network with a content-addressed cache (the plan is public,
    deterministic host data; recompiling per call would dominate a step)."""
    if isinstance(net, CompiledNet):
        return net
    key = (_net_fingerprint(net), tuple(int(t) for t in cfg.t_lanes), cfg.precision_bits)
    hit = _compile_cache.get(key)
    if hit is None:
        hit = compile_network(net, cfg)
        if len(_compile_cache) > 64:
            _compile_cache.clear()
        _compile_cache[key] = hit
    return hit


def _lowered(compiled: CompiledNet, t: int, n: int, encoding: str):
    key = (id(compiled), t, n, encoding, dev.current_device())
    hit = _lower_cache.get(key)
    if hit is not None and hit[0] is compiled:
        return hit[1]
    low = []
    for plan in compiled.plans:
        if isinstance(plan, LinearPlan):
            low.append(("linear",) + _lower_linear(plan, t, n, encoding))
        elif isinstance(plan, PoolPlan):
            low.append(("pool",) + _lower_pool(plan, t, n, encoding))
        elif isinstance(plan, ActPlan):
            low.append(("act",) + _lower_act(plan, t, n, encoding))
        else:
            raise EngineError(f"unknown plan {type(plan).__name__}")
    _lower_cache[key] = (compiled, low)
    return low


# ------------------------------------------------------------------ kernels


def _row_bytes(params) -> int:
    return 2 * len(params.limb_primes) * params.n * 8


def _run_mac(params, in0, in1, mac: _Mac, out, fanout=()):
    """out rows (and the same rows at every fan-out pointer) = the MAC."""
    h = params.native()
    n_in0 = in0.shape[0]
    n_in1 = in1.shape[0] if in1 is not None else 0
    ptrs = _lib.ptr_array([out.data_ptr()] + [int(p) for p in fanout])
    _lib.check(
        _lib.lib().fcn_linear_mac_multi(
            h.ptr, in0.data_ptr(), n_in0, in1.data_ptr() if in1 is not None else None, n_in1, mac.rowptr.data_ptr(),
            mac.col.data_ptr(), mac.rot.data_ptr(), mac.coef.data_ptr(), C.cast(ptrs, C.c_void_p), 1 + len(fanout),
            mac.n_out, int(mac.no_rot), min(mac.max_abs_coef, (1 << 64) - 1), dev.stream_ptr(),
        ),
        FVError,
    )


def _run_bias(params, lane, buf, bias: _Bias | None, fanout=()):
    if bias is None:
        return
    for ptr in [buf.data_ptr()] + [int(p) for p in fanout]:
        _lib.check(
            _lib.lib().fcn_add_plain_terms(
                params.native().ptr, lane, ptr, bias.n_terms, bias.ct_index.data_ptr(), bias.pos.data_ptr(),
                bias.coef.data_ptr(), dev.stream_ptr(),
            ),
            FVError,
        )


def _mac_out(params, mac: _Mac, in0, in1, out=None, fanout=()):
    if out is None:
        out = dev.empty((mac.n_out, 2, len(params.limb_primes), params.n))
    rb = _row_bytes(params)
    for lo in range(0, mac.n_out, 65535):
        hi = min(mac.n_out, lo + 65535)
        if lo == 0 and hi == mac.n_out:
            _run_mac(params, in0, in1, mac, out, fanout)
        else:  # split launches over output rows (grid.y limit)
            sub = _Mac(mac.rowptr[lo : hi + 1], mac.col, mac.rot, mac.coef, hi - lo, mac.n_terms, mac.no_rot, mac.max_abs_coef)
            _run_mac(params, in0, in1, sub, out[lo:hi], [int(p) + lo * rb for p in fanout])
    return out


# ------------------------------------------------------- range execution

_range_cache: dict = {}


def _bias_range(bias: _Bias | None, lo: int, hi: int):
    """Bias terms of outputs [lo, hi), re-indexed from 0 (cached per range).

    Keyed by the lowered bias object itself (one per plan, encoding, t, n and
    device), which the cache entry keeps alive so its id cannot be reused."""
    import torch

    if bias is None:
        return None
    ck = ("bias", id(bias), lo, hi)
    hit = _range_cache.get(ck)
    if hit is None or hit[0] is not bias:
        idx = bias.ct_index.cpu().numpy()
        sel = (idx >= lo) & (idx < hi)
        if not sel.any():
            hit = (bias, None)
        else:
            d = bias.ct_index.device
            hit = (
                bias,
                _Bias(
                    torch.as_tensor(idx[sel] - lo, dtype=torch.int32, device=d),
                    bias.pos[torch.as_tensor(sel, device=d)].contiguous(),
                    bias.coef[torch.as_tensor(sel, device=d)].contiguous(),
                    int(sel.sum()),
                ),
            )
        _range_cache[ck] = hit
    return hit[1]


def _act_lowered(plan, t, n, encoding, m):
    ck = ("act", id(plan), t, n, encoding, m, dev.current_device())
    hit = _range_cache.get(ck)
    if hit is None or hit[0] is not plan:
        hit = (plan, _lower_act(plan, t, n, encoding, nodes=m))
        _range_cache[ck] = hit
    return hit[1]


def _layer_range(params, lane, ek, plan, lw, cur, lo: int, hi: int, encoding: str, mul_chunk=None, out=None,
                 fanout=()):
    """Outputs [lo, hi) of one compiled layer as a [hi-lo][2][k][n] buffer.

    `cur` holds every input of the layer (for an activation, its inputs
    are the same rows as its outputs, so cur may also be just [lo, hi)).
    `out` (optional) receives the rows; every pointer in `fanout` (device
    addresses of row lo of other buffers, e.g. peers' buffers over NVLink)
    receives the same rows from the layer's final kernel."""
    t = int(params.t_lanes[lane])
    kind = lw[0]
    if kind in ("linear", "pool"):
        mac, bias = lw[1], lw[2]
        tcp = mac_tc.plan_for(params, mac, cur.shape[0]) if mac.host is not None else None
        if tcp is not None:  # tensor-core MAC (csrc/mac_tc.cu)
            if out is None:
                out = dev.empty((hi - lo, 2, len(params.limb_primes), params.n))
            mac_tc.run(params, tcp, cur, out, fanout, lo, hi)
            _run_bias(params, lane, out, bias if (lo == 0 and hi == mac.n_out) else _bias_range(bias, lo, hi), fanout)
            return out
        if lo == 0 and hi == mac.n_out:
            out = _mac_out(params, mac, cur, None, out, fanout)
            _run_bias(params, lane, out, bias, fanout)
            return out
        sub = _Mac(mac.rowptr[lo : hi + 1], mac.col, mac.rot, mac.coef, hi - lo, mac.n_terms, mac.no_rot, mac.max_abs_coef)
        out = _mac_out(params, sub, cur, None, out, fanout)
        _run_bias(params, lane, out, _bias_range(bias, lo, hi), fanout)
        return out
    x = cur if cur.shape[0] == hi - lo else cur[lo:hi]
    mac, bias, identity = _act_lowered(plan, t, params.n, encoding, hi - lo)
    fused = _act_scalars(plan, t, params.n, encoding)
    if identity or fused is not None:
        # a2 x^2 + a1 x with constant plaintexts (or x^2): one fused product epilogue
        out = fv.mul_ct_batch(params, ek, lane, x, None, out=out, chunk=mul_chunk, act=None if identity else fused,
                              fanout=fanout)
    else:
        sq = fv.mul_ct_batch(params, ek, lane, x, None, chunk=mul_chunk)
        out = _mac_out(params, mac, sq, x, out, fanout)
    _run_bias(params, lane, out, bias, fanout)
    return out


def _act_scalars(plan, t: int, n: int, encoding: str):
    """(c2, c1) when the activation's MAC is c2*sq[o] + c1*x[o] with constant
    (rotation-0) multipliers -- the batched encoding -- else None."""
    if encoding != "batched":
        return None
    a2 = [(0, 1)] if plan.a2_int is None else const_terms(plan.a2_int, t, n, encoding)
    a1 = [(0, 0)] if plan.a1_mult_int is None else const_terms(plan.a1_mult_int, t, n, encoding)
    if len(a2) != 1 or len(a1) != 1 or a2[0][0] != 0 or a1[0][0] != 0:
        return None
    return a2[0][1], a1[0][1]


def _meta_step(plan, lw, depths, scales, scale, factor, prec):
    """Per-ciphertext (depth, scale) and tensor-level (scale, factor) after a layer."""
    kind = lw[0]
    if kind == "linear":
        depths, scales, nonempty = _gather_meta(lw[3], depths, scales, scale + prec)
        scales = np.where(nonempty, scales + prec, scales)
        return depths, scales, scale + prec, factor
    if kind == "pool":
        depths, scales, _ = _gather_meta(lw[3], depths, scales, scale)
        if plan.reciprocal_int is not None:
            return depths, scales + prec, scale + prec, factor
        return depths, scales, scale + plan.pow2_shift, factor * plan.factor_mult
    return depths + 1, 2 * scales + (prec if plan.a2_int is not None else 0), 2 * scale + plan.scale_bump, factor * factor


# --------------------------------------------------------------- evaluator


def _gather_meta(taps, depths, scales, empty_scale):
    """Per-output (depth, scale) of an add_ct chain over the taps' inputs.

    depth = max over inputs (add_ct, fv.py:394-403), 0 for an empty row
    (Ciphertext.zero); every input of a chain must share its scale
    exponent, exactly as the reference's add_ct demands (fv.py:383-391)."""
    rowptr, cols = taps
    n_out = len(rowptr) - 1
    d = np.zeros(n_out, dtype=np.int64)
    sc = np.full(n_out, empty_scale, dtype=np.int64)
    nonempty = np.diff(rowptr) > 0
    if cols.size:
        starts = rowptr[:-1][nonempty]
        d[nonempty] = np.maximum.reduceat(depths[cols], starts)
        smin = np.minimum.reduceat(scales[cols], starts)
        smax = np.maximum.reduceat(scales[cols], starts)
        if np.any(smin != smax):
            bad = int(np.nonzero(smin != smax)[0][0])
            raise FVError(f"scale mismatch: 2^{int(smin[bad])} vs 2^{int(smax[bad])}")
        sc[nonempty] = smin
    return d, sc, nonempty


def eval_encrypted(net, tensor: CipherTensor, ek: EvalKeys, cfg: FixedPointConfig, workers: int = 1,
                   encoding: str = "integer", mul_chunk: int | None = None, timing: bool = True):
    """Execute the compiled plan over a ciphertext tensor, tallying every HOP.

    Same contract as reference engine.eval_encrypted (engine.py:651-774);
    `workers` is accepted for API compatibility (the GPU parallelises
    every layer's outputs).  `net` may also be the CompiledNet that
    `compile_network(net, cfg)` returned, which skips the per-call content
    hash of the weights that keys the plan cache (~0.7 ms for cfg2; a server
    evaluating one network repeatedly compiles it once).  `encoding` selects the plaintext encoding of
    the integer constants ("integer" = the reference's base-2 encoder;
    "batched" = constant polynomials for SIMD-packed slots).  `timing=False`
    records no per-layer CUDA events (layer wall_ms then reads 0), e.g. for
    CUDA-graph capture (`EvalGraph`)."""
    if encoding not in ENCODINGS:
        raise EngineError(f"encoding must be one of {ENCODINGS}")
    if not isinstance(tensor, CipherTensor):
        raise EngineError("tensor must be a CipherTensor")
    import torch

    params = tensor.params
    lane = tensor.lane
    t = int(params.t_lanes[lane])
    if int(cfg.t_lanes[lane]) != t:
        raise EngineError("fixed-point lane configuration disagrees with ciphertexts")
    if isinstance(net, CompiledNet):  # a plan from compile_network: no per-call content hash
        acts = sum(isinstance(p, ActPlan) for p in net.plans)
    else:
        acts = sum(type(l).__name__ == "PolyActivation" for l in net.layers)
    if acts > params.mul_depth_budget:
        raise EngineError(f"{acts} activations exceed the parameter depth budget {params.mul_depth_budget}")
    compiled = _compiled(net, cfg)
    counter = _hops(compiled, encoding, t)
    low = _lowered(compiled, t, params.n, encoding)
    prec = cfg.precision_bits
    cur = tensor.buf
    depths = tensor.depths.copy()
    scales = tensor.scales.copy()
    scale = tensor.scale_exponent
    factor = tensor.scale_factor
    events = []
    for plan, lw in zip(compiled.plans, low):
        if timing:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record()
        n_out = lw[1].n_out if lw[0] in ("linear", "pool") else plan.nodes
        depths, scales, scale, factor = _meta_step(plan, lw, depths, scales, scale, factor, prec)
        cur = _layer_range(params, lane, ek, plan, lw, cur, 0, n_out, encoding, mul_chunk)
        if timing:
            ev1.record()
            events.append((ev0, ev1))
    # wall_ms resolves from the events on first access (no device sync here)
    if timing:
        counter.layer_counts = [TimedLayerCounts(c, (a, b, 1.0)) for c, (a, b) in zip(counter.layer_counts, events)]
    out = CipherTensor(compiled.out_shape, scale_exponent=scale, scale_factor=factor, buf=cur, params=params, lane=lane,
                       depths=depths, scales=scales)
    return out, counter


# ---------------------------------------------------------------- CUDA graphs


class EvalGraph:
    """One `eval_encrypted` over a fixed input buffer, captured as a CUDA graph.

    The plan's ~17 kernel launches per cfg2 step (and the host-side layer
    walk that issues them) become one graph launch: `replay()` re-runs the
    whole network on whatever ciphertexts are in `tensor.buf` at that moment
    and returns the output CipherTensor, whose buffer is the graph's own
    (overwritten by the next replay).  Intermediates live in the graph's
    private memory pool.  Same bytes as `eval_encrypted` (tested)."""

    def __init__(self, net, tensor: CipherTensor, ek: EvalKeys, cfg: FixedPointConfig, encoding: str = "batched",
                 mul_chunk: int | None = None):
        import torch

        # lowering, kernel attributes and workspace sizes settle outside the capture
        eval_encrypted(net, tensor, ek, cfg, encoding=encoding, mul_chunk=mul_chunk, timing=False)
        torch.cuda.synchronize()
        self.tensor = tensor
        self.graph = torch.cuda.CUDAGraph()
        lib = _lib.lib()
        n0 = lib.fcn_launch_count()
        with torch.cuda.graph(self.graph):
            self.out, self.counter = eval_encrypted(net, tensor, ek, cfg, encoding=encoding, mul_chunk=mul_chunk,
                                                    timing=False)
        self.kernels = int(lib.fcn_launch_count() - n0)  # libfcn kernels each replay runs

    def replay(self) -> CipherTensor:
        self.graph.replay()
        return self.out


# ---------------------------------------------------------------- streaming


def evaluate_stream(net, host_batches, ek: EvalKeys, cfg: FixedPointConfig, params: EncryptionParams, shape,
                    scale_exponent: int, lane: int = 0, encoding: str = "batched", host_out=None):
    """Serve a sequence of encrypted batches held in (pinned) host memory.

    host_batches: iterable of [count][2][k][n] int64 CPU tensors (the
    serialized ciphertext bodies).  For each batch this uploads it, runs
    `eval_encrypted`, and yields the output bodies as a CPU tensor.  Uploads
    run on a separate copy stream into two preallocated device buffers, so
    batch i+1 crosses PCIe while batch i is evaluated (what a server loop
    does); every batch's H2D copy and its result's D2H read stay in the loop.

    Results land in a ring of three pinned host buffers (pinned allocation
    costs ~0.14 ms/MB, more than the transfer): a yielded tensor stays valid
    until two further batches have been yielded -- copy it to keep it longer.
    `host_out` (optional): a list of >= 3 pinned CPU tensors to use as that
    ring, so a long-running server allocates them once."""
    import torch

    compute = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    it = iter(host_batches)
    bufs = [None, None]
    done = [None, None]  # compute-stream event: eval reading bufs[s] finished

    def upload(i, hb):
        s = i % 2
        with torch.cuda.stream(copy):
            if bufs[s] is None or tuple(bufs[s].shape) != tuple(hb.shape):
                bufs[s] = torch.empty(hb.shape, dtype=hb.dtype, device="cuda")
            if done[s] is not None:
                copy.wait_event(done[s])
            bufs[s].copy_(hb, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
        return ev

    i = 0
    ring_out = list(host_out) if host_out is not None else [None, None, None]
    if len(ring_out) < 3:
        raise EngineError("host_out needs at least three buffers")
    hb = next(it, None)
    ready = upload(0, hb) if hb is not None else None
    pending = None  # (pinned host result, event) of the previous batch
    while ready is not None:
        s = i % 2
        compute.wait_event(ready)
        nxt = next(it, None)
        ready = upload(i + 1, nxt) if nxt is not None else None
        t_in = CipherTensor(shape, scale_exponent=scale_exponent, buf=bufs[s], params=params, lane=lane)
        out, _ = eval_encrypted(net, t_in, ek, cfg, encoding=encoding)
        ev = torch.cuda.Event()
        ev.record(compute)
        done[s] = ev
        slot = i % len(ring_out)
        if ring_out[slot] is None or tuple(ring_out[slot].shape) != tuple(out.buf.shape):
            ring_out[slot] = torch.empty(out.buf.shape, dtype=out.buf.dtype, pin_memory=True)
        res = ring_out[slot]
        res.copy_(out.buf, non_blocking=True)
        rev = torch.cuda.Event()
        rev.record(compute)
        if pending is not None:  # hand back batch i-1 while batch i runs
            pending[1].synchronize()
            yield pending[0]
        pending = (res, rev)
        i += 1
    if pending is not None:
        pending[1].synchronize()
        yield pending[0]
