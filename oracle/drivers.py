"""Plan evaluators over oracle ciphertexts -- test infra only.

`run_plan` mirrors the reference evaluation loop `engine.eval_encrypted`
(engine.py:692-774) op for op: per linear output a chain of mul_pt + add_ct
seeded by the first term (empty rows -> transparent zero at scale+prec),
then add_pt of the bias; pool windows as add_ct chains (+ reciprocal
mul_pt); activations as mul_ct(x, x) -> mul_pt(a2) -> + mul_pt(x, a1) ->
add_pt(a0).  It consumes a compiled plan with the reference field names
(engine.py:357-401), so it runs equally on plans from the reference or from
`paper_1811_09953_b200.netplan`.

Two plaintext encodings of the integer constants:
  * "integer": the reference's base-2 encoder (encode.py:64-78), i.e. the
    reference evaluator itself;
  * "batched": the constant polynomial PlainPoly(t, [z mod t]) -- the SIMD
    slot encoding of SURVEY.md sec. 0.5 / 8(c), evaluated with the very same
    reference `fv` operations.
"""

from __future__ import annotations

import numpy as np

from . import bfv, rns


def encode_const(z: int, t: int, encoding: str, n: int) -> list[int]:
    """Plaintext coefficients of integer constant z under the chosen encoding."""
    z = int(z)
    if encoding == "batched":
        return [z % t]
    if z == 0:
        return []
    mag = abs(z)
    bit = 1 if z > 0 else t - 1
    out = []
    while mag:
        out.append(bit if mag & 1 else 0)
        mag >>= 1
    return out


def slot_encode(values: np.ndarray, t: int, n: int) -> list[int]:
    """Slots -> plaintext coefficients: inverse NTT over Z_t."""
    v = np.zeros(n, dtype=np.uint64)
    vals = np.asarray(values, dtype=np.int64) % t
    v[: vals.size] = vals.astype(np.uint64)
    return [int(x) for x in rns.intt_row(v, rns.limb_tables(int(t), n))]


def slot_decode(coeffs, t: int, n: int) -> np.ndarray:
    v = np.zeros(n, dtype=np.uint64)
    c = np.asarray([int(x) for x in coeffs], dtype=np.uint64)
    v[: c.size] = c
    return rns.ntt_row(v, rns.limb_tables(int(t), n))


def run_plan(P: bfv.Params, compiled, cts: list, keys: bfv.Keys, prec: int, encoding: str = "integer"):
    """Execute a compiled plan over oracle ciphertexts; returns (cts, scale, factor)."""
    lane = cts[0].lane
    t = int(P.t_lanes[lane])
    cur = list(cts)
    scale = cts[0].scale
    factor = 1
    for plan in compiled.plans:
        kind = type(plan).__name__
        if kind == "LinearPlan":
            nxt = []
            for out in plan.outputs:
                acc = None
                for tap in out.taps:
                    term = bfv.mul_pt(P, cur[tap.in_index], encode_const(tap.weight_int, t, encoding, P.n), prec)
                    acc = term if acc is None else bfv.add_ct(P, acc, term)
                if acc is None:
                    z = np.zeros((len(P.primes), P.n), dtype=np.uint64)
                    acc = bfv.Ct(z, z.copy(), lane, scale + prec, 0)
                if out.bias_int is not None:
                    acc = bfv.add_pt(P, acc, encode_const(out.bias_int, t, encoding, P.n))
                nxt.append(acc)
            cur = nxt
            scale += prec
        elif kind == "PoolPlan":
            nxt = []
            for idxs in plan.outputs:
                acc = None
                for i in idxs:
                    acc = cur[i] if acc is None else bfv.add_ct(P, acc, cur[i])
                if plan.reciprocal_int is not None:
                    acc = bfv.mul_pt(P, acc, encode_const(plan.reciprocal_int, t, encoding, P.n), prec)
                nxt.append(acc)
            cur = nxt
            if plan.reciprocal_int is not None:
                scale += prec
            else:
                scale += plan.pow2_shift
                factor *= plan.factor_mult
        elif kind == "ActPlan":
            nxt = []
            for x in cur:
                sq = bfv.mul_ct(P, x, x, keys)
                if plan.a2_int is not None:
                    acc = bfv.mul_pt(P, sq, encode_const(plan.a2_int, t, encoding, P.n), prec)
                else:
                    acc = sq
                if plan.a1_mult_int is not None:
                    lin = bfv.mul_pt(P, x, encode_const(plan.a1_mult_int, t, encoding, P.n), acc.scale - x.scale)
                    acc = bfv.add_ct(P, acc, lin)
                if plan.a0_add_int is not None:
                    acc = bfv.add_pt(P, acc, encode_const(plan.a0_add_int, t, encoding, P.n))
                nxt.append(acc)
            cur = nxt
            scale = 2 * scale + plan.scale_bump
            factor = factor * factor
        else:
            raise ValueError(f"unknown plan {kind}")
    return cur, scale, factor


def plain_model_batched(compiled, x_int: np.ndarray, t: int) -> np.ndarray:
    """Slot-wise integer model mod t of a compiled plan.

    x_int: (inputs, slots) integers already scaled by 2^prec.  Returns the
    expected decrypted slot values (outputs, slots) in [0, t).  Every value
    stays below t < 2^31, so int64 products cannot overflow.
    """
    cur = [np.mod(np.asarray(v, dtype=np.int64), t) for v in x_int]
    for plan in compiled.plans:
        kind = type(plan).__name__
        if kind == "LinearPlan":
            nxt = []
            for out in plan.outputs:
                acc = np.zeros_like(cur[0])
                for tap in out.taps:
                    acc = (acc + (int(tap.weight_int) % t) * cur[tap.in_index]) % t
                if out.bias_int is not None:
                    acc = (acc + int(out.bias_int) % t) % t
                nxt.append(acc)
            cur = nxt
        elif kind == "PoolPlan":
            nxt = []
            for idxs in plan.outputs:
                acc = cur[idxs[0]].copy()
                for i in idxs[1:]:
                    acc = (acc + cur[i]) % t
                if plan.reciprocal_int is not None:
                    acc = acc * (int(plan.reciprocal_int) % t) % t
                nxt.append(acc)
            cur = nxt
        elif kind == "ActPlan":
            nxt = []
            for x in cur:
                acc = x * x % t
                if plan.a2_int is not None:
                    acc = acc * (int(plan.a2_int) % t) % t
                if plan.a1_mult_int is not None:
                    acc = (acc + x * (int(plan.a1_mult_int) % t)) % t
                if plan.a0_add_int is not None:
                    acc = (acc + int(plan.a0_add_int) % t) % t
                nxt.append(acc)
            cur = nxt
    return np.stack(cur).astype(np.int64)
