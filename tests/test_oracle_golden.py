"""Pin the CPU oracle (oracle/) and the host plan code against golden vectors
produced by the reference itself (tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import bfv, drivers, nt, rns
from paper_1811_09953_b200 import configs, netplan
from paper_1811_09953_b200.encode import FixedPointConfig


def test_primes_and_roots(golden_meta):
    for name, case in golden_meta["ntt"].items():
        n = case["n"]
        for q, r in zip(case["primes"], case["roots"]):
            assert nt.root_2n(q, n) == r
    for key in ("tiny", "bat", "b70", "cfg1"):
        m = golden_meta["fv"][key]
        P = bfv.Params(m["n"], tuple(m["primes"]), tuple(m["t_lanes"]), m["beta"])
        assert list(P.aux) == m["aux"]
        assert P.ell == m["ell"]
        assert str(P.delta(0)) == m["delta0"]
    assert configs.WORKLOADS["cfg1"].primes == tuple(golden_meta["fv"]["cfg1"]["primes"])


@pytest.mark.parametrize("name", ["n4", "n16", "n1024", "n4096", "n8192", "n16384", "t65537_n1024"])
def test_ntt_matches_reference(name, golden_meta, golden_npz):
    d = golden_npz("ntt")
    primes = golden_meta["ntt"][name]["primes"]
    assert np.array_equal(rns.ntt(d[f"{name}_in"], primes), d[f"{name}_fwd"])
    assert np.array_equal(rns.intt(d[f"{name}_in"], primes), d[f"{name}_inv"])
    assert np.array_equal(rns.intt(d[f"{name}_fwd"], primes), d[f"{name}_in"])


def test_ring_ops_match_reference(golden_meta, golden_npz):
    d = golden_npz("ringops")
    m = golden_meta["ringops"]
    pr = m["primes"]
    a, b = d["a"], d["b"]
    assert np.array_equal(rns.padd(a, b, pr), d["add"])
    assert np.array_equal(rns.psub(a, b, pr), d["sub"])
    assert np.array_equal(rns.pneg(a, pr), d["neg"])
    assert np.array_equal(rns.pscale(a, -12345, pr), d["scalar_m12345"])
    assert np.array_equal(rns.pmul(rns.ntt(a, pr), rns.ntt(b, pr), pr), d["pointwise"])
    assert np.array_equal(rns.polymul(a, b, pr), d["polymul"])
    for i, (k, c) in enumerate(m["monomials"]):
        assert np.array_equal(rns.monomial(a, k, c, pr), d[f"mono{i}"])
    assert np.array_equal(rns.polymul_schoolbook(d["sb_x"], d["sb_y"], m["sb_primes"]), d["sb_xy"])
    assert np.array_equal(rns.polymul(d["sb_x"], d["sb_y"], m["sb_primes"]), d["sb_xy"])


def test_hand_known_answers():
    # (1+x)^2 and x^3*x = -1 in Z_17[x]/(x^4+1) (reference tests/test_ring.py:48-66)
    p = rns.from_ints([1, 1], [17], 4)
    assert rns.polymul(p, p, [17])[0].tolist() == [1, 2, 1, 0]
    x3 = rns.from_ints([0, 0, 0, 1], [17], 4)
    x1 = rns.from_ints([0, 1], [17], 4)
    assert rns.polymul(x3, x1, [17])[0].tolist() == [16, 0, 0, 0]
    assert rns.monomial(x3, 1, 1, [17])[0].tolist() == [16, 0, 0, 0]


def _params(m):
    return bfv.Params(m["n"], tuple(m["primes"]), tuple(m["t_lanes"]), m["beta"])


def _keys_match(P, prefix, d, seed):
    K = bfv.keygen(P, seed)
    assert np.array_equal(K.s, d[f"{prefix}_s"])
    assert np.array_equal(K.p0, d[f"{prefix}_p0"])
    assert np.array_equal(K.p1, d[f"{prefix}_p1"])
    assert np.array_equal(np.stack(K.a), d[f"{prefix}_a"])
    assert np.array_equal(np.stack(K.g), d[f"{prefix}_g"])
    return K


def _arr(ct):
    return np.stack([ct.c0, ct.c1])


def test_fv_tiny_matches_reference(golden_meta, golden_npz):
    d = golden_npz("fv")
    m = golden_meta["fv"]["tiny"]
    P = _params(m)
    K = _keys_match(P, "tiny", d, 42)
    t = P.t_lanes[0]
    rng = np.random.default_rng(99)
    cts = [bfv.encrypt(P, K, drivers.encode_const(v, t, "integer", P.n), 0, 12, rng) for v in m["vals"]]
    assert np.array_equal(np.stack([_arr(c) for c in cts]), d["tiny_cts"])
    a, b = cts[0], cts[1]
    assert np.array_equal(_arr(bfv.add_ct(P, a, b)), d["tiny_add"])
    assert np.array_equal(_arr(bfv.sub_ct(P, a, b)), d["tiny_sub"])
    assert np.array_equal(_arr(bfv.add_pt(P, a, drivers.encode_const(-13, t, "integer", P.n))), d["tiny_addpt"])
    assert np.array_equal(_arr(bfv.mul_pt(P, a, drivers.encode_const(-8, t, "integer", P.n), 3)), d["tiny_mulpt_mono"])
    assert np.array_equal(_arr(bfv.mul_pt(P, a, drivers.encode_const(11, t, "integer", P.n), 3)), d["tiny_mulpt_gen"])
    sq = bfv.mul_ct(P, a, a, K)
    assert np.array_equal(_arr(sq), d["tiny_sq"])
    assert [sq.lane, sq.scale, sq.depth] == m["sq_meta"]
    assert np.array_equal(_arr(bfv.mul_ct(P, cts[2], cts[3], K)), d["tiny_ab"])
    assert bfv.ct_to_bytes(P, sq) == d["tiny_ser"].tobytes()
    dec = bfv.decrypt(P, K, sq)
    val = sum(c << i for i, c in enumerate(bfv.centered_plain(dec, t)))
    assert val == m["dec"]["sq"]
    assert abs(bfv.noise_budget(P, K, a) - m["budget_fresh"]) < 1e-9
    assert abs(bfv.noise_budget(P, K, sq) - m["budget_sq"]) < 1e-9


def test_fv_batched_matches_reference(golden_meta, golden_npz):
    d = golden_npz("fv")
    P = _params(golden_meta["fv"]["bat"])
    K = _keys_match(P, "bat", d, 2)
    rng = np.random.default_rng(5)
    slots = rng.integers(0, 65537, (2, P.n), dtype=np.uint64)
    assert np.array_equal(slots, d["bat_slots"])
    cts = [bfv.encrypt(P, K, drivers.slot_encode(s, 65537, P.n), 0, 6, rng) for s in slots]
    assert np.array_equal(np.stack([_arr(c) for c in cts]), d["bat_cts"])
    prod = bfv.mul_ct(P, cts[0], cts[1], K)
    assert np.array_equal(_arr(prod), d["bat_prod"])
    got = drivers.slot_decode(bfv.decrypt(P, K, prod), 65537, P.n)
    assert np.array_equal(got, d["bat_prod_slots"])
    want = (slots[0].astype(object) * slots[1].astype(object)) % 65537
    assert np.array_equal(got.astype(object), want)
    assert np.array_equal(_arr(bfv.mul_pt(P, cts[0], [65535], 0)), d["bat_mulconst"])


def test_fv_multiword_digits(golden_meta, golden_npz):
    d = golden_npz("fv")
    P = _params(golden_meta["fv"]["b70"])
    K = _keys_match(P, "b70", d, 3)
    ct = bfv.Ct(d["b70_in"][0], d["b70_in"][1])
    assert np.array_equal(_arr(bfv.mul_ct(P, ct, ct, K)), d["b70_sq"])


def test_fv_cfg1_uniform(golden_meta, golden_npz):
    d = golden_npz("fv")
    P = _params(golden_meta["fv"]["cfg1"])
    K = _keys_match(P, "cfg1", d, 2)
    ct = bfv.Ct(d["cfg1_u"][0], d["cfg1_u"][1])
    assert np.array_equal(_arr(bfv.mul_ct(P, ct, ct, K)), d["cfg1_usq"])


def _tiny_net(meta):
    L = netplan
    conv = L.Conv2d(np.array(meta["conv_w"]), np.array(meta["conv_b"]), 1, 0)
    c0, c1, c2 = meta["act"]
    act = L.PolyActivation(L.PolyApprox(2, (c0, c1, c2)))
    pool = L.ScaledAvgPool(2, stride=1, padding=1)
    dense = L.Dense(np.array(meta["dense_w"]), np.array(meta["dense_b"]))
    return L.NetworkSpec((1, 4, 4), [conv, act, pool, dense])


def test_engine_tiny_integer_mode(golden_meta, golden_npz):
    d = golden_npz("engine_tiny")
    em = golden_meta["engine_tiny"]
    m = golden_meta["fv"]["tiny"]
    P = _params(m)
    K = _keys_match(P, "tiny", golden_npz("fv"), 42)
    net = _tiny_net(em)
    cfg = FixedPointConfig(tuple(m["t_lanes"]), em["prec"])
    comp = netplan.compile_network(net, cfg)
    cts = [bfv.Ct(x[0], x[1], 0, em["prec"], 0) for x in d["in_cts"]]
    out, scale, factor = drivers.run_plan(P, comp, cts, K, em["prec"], "integer")
    assert scale == em["out_scale"] and factor == em["out_factor"]
    assert np.array_equal(np.stack([_arr(c) for c in out]), d["out_cts"])
    assert np.array_equal(np.array([[c.lane, c.scale, c.depth] for c in out]), d["out_meta"])
    hops = netplan.plan_hops(comp, "integer")
    assert [list(r[:5]) + [r[6]] for r in hops.rows()] == em["hops"]


def _digest(comp):
    h = hashlib.sha256()
    for plan in comp.plans:
        kind = type(plan).__name__
        h.update(kind.encode())
        if kind == "LinearPlan":
            for o in plan.outputs:
                h.update(repr([(t.in_index, t.weight_int) for t in o.taps]).encode())
                h.update(repr(o.bias_int).encode())
        elif kind == "PoolPlan":
            h.update(repr((plan.outputs, plan.count, plan.pow2_shift, plan.factor_mult, plan.reciprocal_int)).encode())
        else:
            h.update(repr((plan.nodes, plan.a2_int, plan.a1_mult_int, plan.a0_add_int, plan.scale_bump)).encode())
    h.update(repr((comp.in_scale, comp.out_scale, comp.out_factor, tuple(comp.out_shape))).encode())
    return h.hexdigest()


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_config_plans_match_reference(name, golden_meta):
    g = golden_meta["configs"][name]
    net = configs.build_network(name)
    comp = netplan.compile_network(net, configs.WORKLOADS[name].fixed_point())
    assert _digest(comp) == g["digest"]
    hops = netplan.plan_hops(comp, "integer")
    assert [list(r[:5]) + [r[6]] for r in hops.rows()] == g["layers"]
    assert comp.out_scale == g["out_scale"]


def test_integer_encoder_known_answers():
    """Reference test_encode.py:19-35 known answers of the base-2 encoder the
    integer encoding uses (host code, no GPU): 5 -> [1, 0, 1], -3 -> [t-1,
    t-1], 0 -> zero polynomial; decode inverts them."""
    from paper_1811_09953_b200 import encode

    t = 65537
    assert encode.encode_integer(5, t).coeffs.tolist() == [1, 0, 1]
    assert encode.encode_integer(-3, t).coeffs.tolist() == [t - 1, t - 1]
    for z in (0, 1, -1, 5, -3, 1 << 40, -(1 << 40) + 7):
        assert encode.decode_integer(encode.encode_integer(z, t)) == z
