"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports `hecnet` read-only from /root/reference/pkg/src and writes small
fixtures next to this file.  The oracle (oracle/) and the host plan code
(paper_1811_09953_b200.netplan/configs) are pinned against these files by
tests/test_oracle_golden.py; the GPU path is then pinned against the oracle
and, where small enough, against these files directly.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from hecnet import compress, encode, engine, fv, modmath as mm, ring  # noqa: E402
from hecnet.approx import PolyApprox, square_activation  # noqa: E402
from hecnet.params_io import load_bundled  # noqa: E402
from hecnet.ring import RingContext, RingPoly  # noqa: E402

from paper_1811_09953_b200 import configs as mycfg  # noqa: E402


def u64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def ct_arr(ct):
    return np.stack([ct.c0.data, ct.c1.data])


def ct_meta(ct):
    return [ct.lane, ct.scale_exponent, ct.mul_depth]


# ----------------------------------------------------------------------------- NTT


def gen_ntt():
    rng = np.random.default_rng(7)
    cases = {
        "n4": (4, (17,)),
        "n16": (16, tuple(mm.find_ntt_primes(16, 1, bits=30))),
        "n1024": (1024, tuple(mm.find_ntt_primes(1024, 2, bits=55))),
        "n4096": (4096, tuple(mm.find_ntt_primes(4096, 3, bits=36))),
        "n8192": (8192, tuple(mm.find_ntt_primes(8192, 1, bits=50))),
        "n16384": (16384, tuple(mm.find_ntt_primes(16384, 1, bits=55))),
        "t65537_n1024": (1024, (65537,)),
    }
    out = {}
    meta = {}
    for name, (n, primes) in cases.items():
        ctx = RingContext.create(n, primes)
        p = RingPoly.random_uniform(ctx, rng)
        f = ring.ntt_forward(p)
        g = ring.ntt_inverse(RingPoly(ctx, p.data.copy(), ring.NTT))
        out[f"{name}_in"] = u64(p.data)
        out[f"{name}_fwd"] = u64(f.data)
        out[f"{name}_inv"] = u64(g.data)
        meta[name] = {"n": n, "primes": [int(q) for q in primes], "roots": [int(l.root) for l in ctx.limbs]}
    np.savez_compressed(os.path.join(HERE, "ntt.npz"), **out)
    return meta


# ---------------------------------------------------------------------------- ring ops


def gen_ringops():
    rng = np.random.default_rng(11)
    n = 1024
    primes = tuple(mm.find_ntt_primes(n, 2, bits=55))
    ctx = RingContext.create(n, primes)
    a = RingPoly.random_uniform(ctx, rng)
    b = RingPoly.random_uniform(ctx, rng)
    out = {"a": u64(a.data), "b": u64(b.data)}
    out["add"] = u64(ring.poly_add(a, b).data)
    out["sub"] = u64(ring.poly_sub(a, b).data)
    out["neg"] = u64(ring.poly_neg(a).data)
    out["scalar_m12345"] = u64(ring.scalar_mul(a, -12345).data)
    fa, fb = ring.ntt_forward(a), ring.ntt_forward(b)
    out["pointwise"] = u64(ring.pointwise_mul(fa, fb).data)
    out["polymul"] = u64(ring.poly_mul_ntt(a, b).data)
    monos = []
    t = 1099511922689
    for i in range(6):
        k = int(rng.integers(0, n))
        c = int(rng.integers(-(t // 2), t // 2 + 1))
        monos.append((k, c))
        out[f"mono{i}"] = u64(ring.poly_mul_monomial(a, k, c).data)
    # small schoolbook check at n=64
    ctx64 = RingContext.create(64, tuple(mm.find_ntt_primes(64, 2, bits=55)))
    x, y = RingPoly.random_uniform(ctx64, rng), RingPoly.random_uniform(ctx64, rng)
    out["sb_x"], out["sb_y"] = u64(x.data), u64(y.data)
    out["sb_xy"] = u64(ring.poly_mul_naive(x, y).data)
    np.savez_compressed(os.path.join(HERE, "ringops.npz"), **out)
    return {"n": n, "primes": [int(q) for q in primes], "monomials": monos, "sb_primes": [int(q) for q in ctx64.primes]}


# ------------------------------------------------------------------------------- FV


def params_meta(P):
    return {
        "n": P.n,
        "primes": [int(q) for q in P.limb_primes],
        "t_lanes": [int(t) for t in P.t_lanes],
        "beta": int(P.beta),
        "ell": int(P.ell),
        "aux": [int(q) for q in P.aux_primes],
        "delta0": str(P.delta(0)),
    }


def keys_arrays(prefix, sk, pk, ek, out):
    out[f"{prefix}_s"] = u64(sk.s.data)
    out[f"{prefix}_p0"] = u64(pk.p0.data)
    out[f"{prefix}_p1"] = u64(pk.p1.data)
    out[f"{prefix}_a"] = u64(np.stack([x.data for x in ek.a]))
    out[f"{prefix}_g"] = u64(np.stack([x.data for x in ek.g]))


def gen_fv():
    out, meta = {}, {}
    # tiny bundled params, integer encoder
    pf = load_bundled("tiny")
    P = pf.params
    sk, pk, ek = fv.keygen(P, seed=42)
    keys_arrays("tiny", sk, pk, ek, out)
    t = int(P.t_lanes[0])
    rng = np.random.default_rng(99)
    vals = [5, -3, 1234, -777]
    cts = [fv.encrypt(pk, P, encode.encode_integer(v, t), 0, 12, rng) for v in vals]
    out["tiny_cts"] = u64(np.stack([ct_arr(c) for c in cts]))
    a, b = cts[0], cts[1]
    out["tiny_add"] = u64(ct_arr(fv.add_ct(a, b)))
    out["tiny_sub"] = u64(ct_arr(fv.sub_ct(a, b)))
    out["tiny_addpt"] = u64(ct_arr(fv.add_pt(a, encode.encode_integer(-13, t))))
    out["tiny_mulpt_mono"] = u64(ct_arr(fv.mul_pt(a, encode.encode_integer(-8, t), 3)))
    out["tiny_mulpt_gen"] = u64(ct_arr(fv.mul_pt(a, encode.encode_integer(11, t), 3)))
    sq = fv.mul_ct(a, a, ek)
    ab = fv.mul_ct(cts[2], cts[3], ek)
    out["tiny_sq"] = u64(ct_arr(sq))
    out["tiny_ab"] = u64(ct_arr(ab))
    meta["tiny"] = params_meta(P)
    meta["tiny"]["vals"] = vals
    meta["tiny"]["sq_meta"] = ct_meta(sq)
    meta["tiny"]["dec"] = {
        "sq": encode.decode_integer(fv.decrypt(sk, sq)),
        "ab": encode.decode_integer(fv.decrypt(sk, ab)),
        "a": encode.decode_integer(fv.decrypt(sk, a)),
    }
    meta["tiny"]["budget_fresh"] = fv.noise_budget(sk, a)
    meta["tiny"]["budget_sq"] = fv.noise_budget(sk, sq)
    out["tiny_ser"] = np.frombuffer(fv.ciphertext_to_bytes(sq), dtype=np.uint8).copy()

    # batched: t = 65537 slot encoder at n=1024, three 36-bit limbs
    n = 1024
    primes = tuple(mm.find_ntt_primes(n, 3, bits=36))
    Pb = fv.EncryptionParams(n, primes, (65537,))
    skb, pkb, ekb = fv.keygen(Pb, seed=2)
    keys_arrays("bat", skb, pkb, ekb, out)
    tctx = RingContext.create(n, (65537,))
    rng = np.random.default_rng(5)
    slots = rng.integers(0, 65537, (2, n), dtype=np.uint64)
    pts = []
    for s in slots:
        m = ring.ntt_inverse(RingPoly(tctx, s[None, :].copy(), ring.NTT))
        pts.append(fv.PlainPoly(65537, m.data[0]))
    bcts = [fv.encrypt(pkb, Pb, p, 0, 6, rng) for p in pts]
    out["bat_slots"] = u64(slots)
    out["bat_cts"] = u64(np.stack([ct_arr(c) for c in bcts]))
    prod = fv.mul_ct(bcts[0], bcts[1], ekb)
    out["bat_prod"] = u64(ct_arr(prod))
    dec = fv.decrypt(skb, prod)
    dpoly = np.zeros(n, dtype=np.uint64)
    dpoly[: dec.coeffs.size] = dec.coeffs
    out["bat_prod_slots"] = u64(ring.ntt_forward(RingPoly(tctx, dpoly[None, :], ring.COEFF)).data[0])
    out["bat_mulconst"] = u64(ct_arr(fv.mul_pt(bcts[0], fv.PlainPoly(65537, np.array([65537 - 2], dtype=np.uint64)), 0)))
    meta["bat"] = params_meta(Pb)

    # multiword digits: beta = 2^70 over four 50-bit limbs (ell = 2)
    primes = tuple(mm.find_ntt_primes(n, 4, bits=50))
    Pw = fv.EncryptionParams(n, primes, (65537,), beta=1 << 70)
    skw, pkw, ekw = fv.keygen(Pw, seed=3)
    keys_arrays("b70", skw, pkw, ekw, out)
    rng = np.random.default_rng(6)
    x = RingPoly.random_uniform(Pw.ctx, rng)
    y = RingPoly.random_uniform(Pw.ctx, rng)
    ct = fv.Ciphertext(x, y, Pw, 0, 0, 0)
    out["b70_in"] = u64(ct_arr(ct))
    out["b70_sq"] = u64(ct_arr(fv.mul_ct(ct, ct, ekw)))
    meta["b70"] = params_meta(Pw)

    # uniform random ciphertexts (no keys needed for the bytes) at cfg1 shape
    W = mycfg.WORKLOADS["cfg1"]
    P1 = fv.EncryptionParams(W.n, W.primes, (W.t,))
    sk1, pk1, ek1 = fv.keygen(P1, seed=2)
    keys_arrays("cfg1", sk1, pk1, ek1, out)
    rng = np.random.default_rng(0)
    u = fv.Ciphertext(RingPoly.random_uniform(P1.ctx, rng), RingPoly.random_uniform(P1.ctx, rng), P1, 0, 0, 0)
    out["cfg1_u"] = u64(ct_arr(u))
    out["cfg1_usq"] = u64(ct_arr(fv.mul_ct(u, u, ek1)))
    meta["cfg1"] = params_meta(P1)

    np.savez_compressed(os.path.join(HERE, "fv.npz"), **out)
    return meta


# --------------------------------------------------------------------------- engine


def _ref_layer(L):
    """Translate one of my layers into the reference's classes."""
    k = type(L).__name__
    if k == "Conv2d":
        return engine.Conv2d(L.weights, L.bias, L.stride, L.padding, L.mask)
    if k == "Dense":
        return engine.Dense(L.weights, L.bias, L.mask)
    if k == "ScaledAvgPool":
        return engine.ScaledAvgPool(L.window, L.stride, L.padding, L.reciprocal)
    if k == "PolyActivation":
        c = tuple(float(v) for v in L.poly.coeffs)
        return engine.PolyActivation(PolyApprox(2, c, 4.0, 0.0))
    raise KeyError(k)


def plan_digest(compiled) -> str:
    h = hashlib.sha256()
    for plan in compiled.plans:
        h.update(type(plan).__name__.encode())
        if isinstance(plan, engine.LinearPlan):
            for o in plan.outputs:
                h.update(repr([(t.in_index, t.weight_int) for t in o.taps]).encode())
                h.update(repr(o.bias_int).encode())
        elif isinstance(plan, engine.PoolPlan):
            h.update(repr((plan.outputs, plan.count, plan.pow2_shift, plan.factor_mult, plan.reciprocal_int)).encode())
        else:
            h.update(repr((plan.nodes, plan.a2_int, plan.a1_mult_int, plan.a0_add_int, plan.scale_bump)).encode())
    h.update(repr((compiled.in_scale, compiled.out_scale, compiled.out_factor, tuple(compiled.out_shape))).encode())
    return h.hexdigest()


def ref_compressed(w, keep):
    """The configs' weight recipe through the reference's own compress module."""
    wt = compress.WeightTensor(w)
    pr = compress.prune_mask(wt, keep)
    spec = compress.quant_bounds(pr)
    qt = compress.quantize_to_pow2(pr, spec, 1.0)
    eff = qt.effective()
    out = np.zeros_like(eff)
    nz = eff != 0
    e = np.clip(np.round(np.log2(np.abs(eff[nz]))), -6, 0)
    out[nz] = np.sign(eff[nz]) * 2.0 ** e
    return out


def gen_configs():
    meta = {}
    for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
        net = mycfg.build_network(name)
        # rebuild the raw weights with the same draws, compress via the reference
        rng = np.random.default_rng(mycfg.SEED_WEIGHTS)
        ref_layers = []
        for L in net.layers:
            k = type(L).__name__
            if k in ("Conv2d", "Dense"):
                shape = L.weights.shape
                raw = rng.normal(0.0, 0.05, shape) if name == "cfg1" else mycfg._he(rng, *shape)
                keep = {"cfg1": [0.2], "cfg2": [0.2, 0.1, 0.2], "cfg3": [0.15] * 4, "cfg4": [0.1, 0.15]}[name]
                idx = sum(1 for x in ref_layers if type(x).__name__ in ("Conv2d", "Dense"))
                w = ref_compressed(raw, keep[idx])
                if k == "Conv2d":
                    ref_layers.append(engine.Conv2d(w, None, L.stride, L.padding))
                else:
                    ref_layers.append(engine.Dense(w, None))
            else:
                ref_layers.append(_ref_layer(L))
        rnet = engine.NetworkSpec(net.input_shape, ref_layers)
        cfg = encode.FixedPointConfig((65537,), 6)
        comp = engine.compile_network(rnet, cfg)
        hops = engine.project_hops(rnet, cfg)
        tot = hops.totals
        meta[name] = {
            "digest": plan_digest(comp),
            "layers": [list(r[:5]) + [r[6]] for r in hops.rows()],
            "totals": [tot.pt_ct_add, tot.ct_ct_add, tot.pt_ct_mul, tot.ct_ct_mul, tot.fast_path_hits],
            "out_scale": comp.out_scale,
            "acts": [
                [p.a2_int, p.a1_mult_int, p.a0_add_int, p.scale_bump] for p in comp.plans if isinstance(p, engine.ActPlan)
            ],
        }
        print(name, meta[name]["totals"])
    return meta


def gen_engine():
    """Tiny integer-mode network through the reference evaluator itself."""
    pf = load_bundled("tiny")
    P = pf.params
    cfg = encode.FixedPointConfig(P.t_lanes, 4)
    sk, pk, ek = fv.keygen(P, seed=42)
    rng = np.random.default_rng(21)
    conv_w = np.zeros((2, 1, 3, 3))
    conv_w[0, 0] = [[0.5, 0, -0.25], [0, 1.0, 0], [0.125, 0, 0]]
    conv_w[1, 0] = [[0, -0.5, 0], [0.75, 0, 0], [0, 0, 0.25]]  # 0.75 -> non-monomial path
    dense_w = np.zeros((2, 18))
    dense_w[0, [0, 4, 8, 9, 13, 17]] = [0.5, -1.0, 0.25, 0.5, -0.5, 1.0]  # row 1 stays empty
    layers = [
        engine.Conv2d(conv_w, np.array([0.25, -0.5]), stride=1, padding=0),
        engine.PolyActivation(PolyApprox(2, (0.0625, 0.5, 0.125), 4.0, 0.0)),
        engine.ScaledAvgPool(2, stride=1, padding=1),
        engine.Dense(dense_w, np.array([0.5, -0.25])),
    ]
    net = engine.NetworkSpec((1, 4, 4), layers)
    x = rng.uniform(-1, 1, (1, 4, 4)).round(3)
    tensor = engine.encrypt_tensor(pk, P, x, cfg, 0, np.random.default_rng(22))
    out_t, counter = engine.eval_encrypted(net, tensor, ek, cfg)
    out = {
        "x": x,
        "in_cts": u64(np.stack([ct_arr(c) for c in tensor.cts])),
        "out_cts": u64(np.stack([ct_arr(c) for c in out_t.cts])),
        "out_meta": np.array([ct_meta(c) for c in out_t.cts], dtype=np.int64),
    }
    plains = engine.decrypt_tensor(sk, out_t)
    dec = engine.decode_lane_outputs([plains], out_t.shape, out_t.scale_exponent, out_t.scale_factor, cfg)
    out["decoded"] = dec
    out["plain"] = engine.eval_plain(net, x)
    np.savez_compressed(os.path.join(HERE, "engine_tiny.npz"), **out)
    return {
        "conv_w": conv_w.tolist(),
        "dense_w": dense_w.tolist(),
        "conv_b": [0.25, -0.5],
        "dense_b": [0.5, -0.25],
        "act": [0.0625, 0.5, 0.125],
        "prec": 4,
        "out_scale": out_t.scale_exponent,
        "out_factor": out_t.scale_factor,
        "hops": [list(r[:5]) + [r[6]] for r in counter.rows()],
    }


def main():
    meta = {"ntt": gen_ntt(), "ringops": gen_ringops()}
    meta["fv"] = gen_fv()
    meta["engine_tiny"] = gen_engine()
    meta["configs"] = gen_configs()
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    for fn in sorted(os.listdir(HERE)):
        print(fn, os.path.getsize(os.path.join(HERE, fn)))


if __name__ == "__main__":
    main()
