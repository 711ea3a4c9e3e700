"""GPU parity of the FV layer: keys, encryption, evaluation ops and the exact
mul_ct against reference golden vectors and the CPU oracle.  Bit-exact."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import bfv as ob  # noqa: E402
from oracle import drivers as od  # noqa: E402


@pytest.fixture(scope="module")
def F():
    import torch

    from paper_1811_09953_b200 import fv

    assert torch.cuda.is_available()
    return fv


def _params(F, m):
    return F.EncryptionParams(m["n"], tuple(m["primes"]), tuple(m["t_lanes"]), m["beta"])


def _arr(ct):
    return np.stack([ct.c0.host(), ct.c1.host()])


def _keys_equal(F, P, prefix, d, seed):
    sk, pk, ek = F.keygen(P, seed)
    assert np.array_equal(sk.s.host(), d[f"{prefix}_s"])
    assert np.array_equal(pk.p0.host(), d[f"{prefix}_p0"])
    assert np.array_equal(pk.p1.host(), d[f"{prefix}_p1"])
    assert np.array_equal(np.stack([x.host() for x in ek.a]), d[f"{prefix}_a"])
    assert np.array_equal(np.stack([x.host() for x in ek.g]), d[f"{prefix}_g"])
    return sk, pk, ek


def test_params_derivations(F, golden_meta):
    for key in ("tiny", "bat", "b70", "cfg1"):
        m = golden_meta["fv"][key]
        P = _params(F, m)
        assert list(P.aux_primes) == m["aux"]
        assert P.ell == m["ell"]
        assert str(P.delta(0)) == m["delta0"]


def test_tiny_scheme_matches_reference(F, golden_meta, golden_npz):
    from paper_1811_09953_b200 import encode

    d = golden_npz("fv")
    m = golden_meta["fv"]["tiny"]
    P = _params(F, m)
    sk, pk, ek = _keys_equal(F, P, "tiny", d, 42)
    t = P.t_lanes[0]
    rng = np.random.default_rng(99)
    cts = [F.encrypt(pk, P, encode.encode_integer(v, t), 0, 12, rng) for v in m["vals"]]
    assert np.array_equal(np.stack([_arr(c) for c in cts]), d["tiny_cts"])
    a, b = cts[0], cts[1]
    assert np.array_equal(_arr(F.add_ct(a, b)), d["tiny_add"])
    assert np.array_equal(_arr(F.sub_ct(a, b)), d["tiny_sub"])
    assert np.array_equal(_arr(F.add_pt(a, encode.encode_integer(-13, t))), d["tiny_addpt"])
    assert np.array_equal(_arr(F.mul_pt(a, encode.encode_integer(-8, t), 3)), d["tiny_mulpt_mono"])
    assert np.array_equal(_arr(F.mul_pt(a, encode.encode_integer(11, t), 3)), d["tiny_mulpt_gen"])
    sq = F.mul_ct(a, a, ek)
    assert np.array_equal(_arr(sq), d["tiny_sq"])
    assert [sq.lane, sq.scale_exponent, sq.mul_depth] == m["sq_meta"]
    ab = F.mul_ct(cts[2], cts[3], ek)
    assert np.array_equal(_arr(ab), d["tiny_ab"])
    assert F.ciphertext_to_bytes(sq) == d["tiny_ser"].tobytes()
    back = F.ciphertext_from_bytes(d["tiny_ser"].tobytes(), P)
    assert np.array_equal(_arr(back), d["tiny_sq"])
    assert encode.decode_integer(F.decrypt(sk, sq)) == m["dec"]["sq"]
    assert encode.decode_integer(F.decrypt(sk, ab)) == m["dec"]["ab"]
    assert encode.decode_integer(F.decrypt(sk, a)) == m["dec"]["a"]
    assert abs(F.noise_budget(sk, a) - m["budget_fresh"]) < 1e-9
    assert abs(F.noise_budget(sk, sq) - m["budget_sq"]) < 1e-9


def test_batched_product_matches_reference(F, golden_meta, golden_npz):
    from paper_1811_09953_b200 import engine

    d = golden_npz("fv")
    P = _params(F, golden_meta["fv"]["bat"])
    sk, pk, ek = _keys_equal(F, P, "bat", d, 2)
    slots = d["bat_slots"]
    cen = engine.slot_encode(P, slots.astype(np.int64))
    want_cen = [od.slot_encode(s, 65537, P.n) for s in slots]
    want_cen = np.array([[c - 65537 if c > 32768 else c for c in row] for row in want_cen])
    assert np.array_equal(cen, want_cen)
    # rng state: the golden draws slots first, then encrypts
    rng = np.random.default_rng(5)
    rng.integers(0, 65537, (2, P.n), dtype=np.uint64)
    buf = F.encrypt_batch(pk, P, cen, 0, rng)
    from paper_1811_09953_b200 import device as dev

    assert np.array_equal(dev.to_host(buf), d["bat_cts"])
    prod = F.mul_ct_batch(P, ek, 0, buf[0:1], buf[1:2])
    assert np.array_equal(dev.to_host(prod)[0], d["bat_prod"])
    slots_out = engine.slot_decode(P, F.decrypt_batch(sk, P, prod).astype(np.int64))
    assert np.array_equal(slots_out[0].astype(np.uint64), d["bat_prod_slots"])


def test_multiword_digits_beta70(F, golden_meta, golden_npz):
    from paper_1811_09953_b200 import device as dev

    d = golden_npz("fv")
    P = _params(F, golden_meta["fv"]["b70"])
    sk, pk, ek = _keys_equal(F, P, "b70", d, 3)
    out = F.mul_ct_batch(P, ek, 0, dev.to_device(d["b70_in"][None]))
    assert np.array_equal(dev.to_host(out)[0], d["b70_sq"])


def test_cfg1_uniform_square(F, golden_meta, golden_npz):
    from paper_1811_09953_b200 import device as dev

    d = golden_npz("fv")
    P = _params(F, golden_meta["fv"]["cfg1"])
    sk, pk, ek = _keys_equal(F, P, "cfg1", d, 2)
    out = F.mul_ct_batch(P, ek, 0, dev.to_device(d["cfg1_u"][None]))
    assert np.array_equal(dev.to_host(out)[0], d["cfg1_usq"])


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg5"])
def test_config_shape_square_vs_oracle(F, cfg):
    """mul_ct on random uniform ciphertexts at the full config ring shapes."""
    from paper_1811_09953_b200 import configs
    from paper_1811_09953_b200 import device as dev

    W = configs.WORKLOADS[cfg]
    P = F.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    OP = ob.Params(W.n, W.primes, (W.t,), W.beta)
    sk, pk, ek = F.keygen(P, 2)
    K = ob.Keys(sk.s.host(), pk.p0.host(), pk.p1.host(), [x.host() for x in ek.a], [x.host() for x in ek.g])
    rng = np.random.default_rng(0)
    from oracle import rns as orn

    B = 3
    x = np.stack([np.stack([orn.random_uniform(W.primes, W.n, rng) for _ in range(2)]) for _ in range(B)])
    out = dev.to_host(F.mul_ct_batch(P, ek, 0, dev.to_device(x)))
    for b in (0, B - 1):
        c = ob.Ct(x[b, 0], x[b, 1])
        want = ob.mul_ct(OP, c, c, K)
        assert np.array_equal(out[b], np.stack([want.c0, want.c1]))


def test_square_extreme_ciphertexts_cfg2(F):
    """mul_ct (FP64 lift / tensor / rescale / key MAC over the cfg2 base with
    auxiliary primes just below 2^51) on ciphertexts whose coefficients sit
    at the extremes of the centred lift: q-1, (q-1)/2, (q+1)/2, 0."""
    from paper_1811_09953_b200 import configs
    from paper_1811_09953_b200 import device as dev

    W = configs.WORKLOADS["cfg2"]
    P = F.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    OP = ob.Params(W.n, W.primes, (W.t,), W.beta)
    sk, pk, ek = F.keygen(P, 2)
    K = ob.Keys(sk.s.host(), pk.p0.host(), pk.p1.host(), [x.host() for x in ek.a], [x.host() for x in ek.g])
    q = math.prod(W.primes)
    n = W.n

    def rows(v):
        return np.stack([np.full(n, v % p, dtype=np.uint64) for p in W.primes])

    mix = np.stack([np.array([(q - 1, (q - 1) // 2, (q + 1) // 2, 0)[j % 4] % p for j in range(n)], dtype=np.uint64)
                    for p in W.primes])
    cts = [(rows(q - 1), rows(q - 1)), (rows((q - 1) // 2), rows((q + 1) // 2)), (mix, mix[:, ::-1].copy())]
    x = np.stack([np.stack([a, b]) for a, b in cts])
    out = dev.to_host(F.mul_ct_batch(P, ek, 0, dev.to_device(x)))
    for i, (a, b) in enumerate(cts):
        want = ob.mul_ct(OP, ob.Ct(a, b), ob.Ct(a, b), K)
        assert np.array_equal(out[i], np.stack([want.c0, want.c1])), i


@pytest.mark.parametrize("primes", [(36028797018972161, 36028797018990593), (1125899906826241, 1125899906820097)],
                         ids=["int64-55bit", "fp64-50bit"])
@pytest.mark.parametrize("c2,c1", [(1, 0), (-3, 5), (64, -1), (12345, -32768)])
def test_fused_activation_epilogue(F, primes, c2, c1):
    """mul_ct_batch(act=(c2, c1)) == c2 * mul_ct(x, x) + c1 * x (mod q_i),
    bit-exact, on the FP64 and the integer kernel families."""
    from oracle import rns as orn
    from paper_1811_09953_b200 import device as dev

    n = 1024
    P = F.EncryptionParams(n, primes, (65537,))
    OP = ob.Params(n, primes, P.t_lanes, P.beta)
    sk, pk, ek = F.keygen(P, 5)
    K = ob.keygen(OP, 5)
    rng = np.random.default_rng(3)
    B = 4
    x = np.stack([np.stack([orn.random_uniform(primes, n, rng) for _ in range(2)]) for _ in range(B)])
    got = dev.to_host(F.mul_ct_batch(P, ek, 0, dev.to_device(x), act=(c2, c1), chunk=3))
    for b in range(B):
        c = ob.Ct(x[b, 0], x[b, 1])
        sq = ob.mul_ct(OP, c, c, K)
        for p_i, (pa, xa) in enumerate(zip((sq.c0, sq.c1), (x[b, 0], x[b, 1]))):
            for l, q in enumerate(primes):
                want = (pa[l].astype(object) * (c2 % q) + xa[l].astype(object) * (c1 % q)) % q
                assert np.array_equal(got[b, p_i, l].astype(object), want), (b, p_i, l)


def test_general_product_and_batch_chunking(F, golden_meta, golden_npz):
    """a*b with distinct operands, across several workspace chunks."""
    from oracle import rns as orn
    from paper_1811_09953_b200 import device as dev

    d = golden_npz("fv")
    m = golden_meta["fv"]["tiny"]
    P = _params(F, m)
    OP = ob.Params(P.n, P.limb_primes, P.t_lanes, P.beta)
    sk, pk, ek = F.keygen(P, 42)
    K = ob.keygen(OP, 42)
    rng = np.random.default_rng(17)
    B = 5
    xa = np.stack([np.stack([orn.random_uniform(P.limb_primes, P.n, rng) for _ in range(2)]) for _ in range(B)])
    xb = np.stack([np.stack([orn.random_uniform(P.limb_primes, P.n, rng) for _ in range(2)]) for _ in range(B)])
    ws = F.mul_ct_workspace(P, 2)  # forces 3 chunks
    out = dev.to_host(F.mul_ct_batch(P, ek, 0, dev.to_device(xa), dev.to_device(xb), workspace=ws))
    for b in range(B):
        want = ob.mul_ct(OP, ob.Ct(xa[b, 0], xa[b, 1]), ob.Ct(xb[b, 0], xb[b, 1]), K)
        assert np.array_equal(out[b], np.stack([want.c0, want.c1]))


def _sqrt_mod_p(a, p):
    """Tonelli-Shanks; None if a is a non-residue."""
    a %= p
    if a == 0:
        return 0
    if pow(a, (p - 1) // 2, p) != 1:
        return None
    q, s = p - 1, 0
    while q % 2 == 0:
        q //= 2
        s += 1
    z = 2
    while pow(z, (p - 1) // 2, p) != p - 1:
        z += 1
    m, c, t, r = s, pow(z, q, p), pow(a, q, p), pow(a, (q + 1) // 2, p)
    while t != 1:
        i, tt = 0, t
        while tt != 1:
            tt = tt * tt % p
            i += 1
        b = pow(c, 1 << (m - i - 1), p)
        m, c, t, r = i, b * b % p, t * b * b % p, r * b % p
    return r


@pytest.mark.parametrize("primes", [(36028797018972161, 36028797018990593), (1125899906826241, 1125899906820097)],
                         ids=["int64-55bit", "fp64-50bit"])
def test_exact_fallback_paths(F, primes):
    """Inputs placed on the float64 ambiguity bands must take the exact
    multiword path and still match the oracle bit-for-bit (55-bit limbs run
    the integer kernels, 50-bit limbs the FP64-pipe kernels)."""
    from paper_1811_09953_b200 import device as dev

    n = 1024
    P = F.EncryptionParams(n, primes, (1099511922689,))
    OP = ob.Params(n, primes, P.t_lanes, P.beta)
    sk, pk, ek = F.keygen(P, 42)
    K = ob.keygen(OP, 42)
    q, t = P.q, P.t_lanes[0]
    h = q >> 1
    cases = []
    # (1) lift: coefficient exactly at the centered-lift boundary (q-1)/2 and (q+1)/2
    for v in (h, h + 1):
        c0 = np.zeros((2, n), dtype=np.uint64)
        c0[:, 0] = [v % p for p in primes]
        c0[:, 5] = [(q - 3) % p for p in primes]
        cases.append((c0, np.zeros((2, n), dtype=np.uint64)))
    # (2) rescale: c0 = x (constant), c1 = 0 with t*x^2 = -h (mod q) -> (t x^2 + h)/q is an integer
    for delta in range(0, 200):
        target = (delta - h) * pow(t, -1, q) % q
        roots = [_sqrt_mod_p(target % p, p) for p in primes]
        if all(r is not None for r in roots):
            break
    assert all(r is not None for r in roots)
    if True:
        x = 0
        for r, p in zip(roots, primes):
            mp = q // p
            x += r * mp * pow(mp, -1, p)
        x %= q
        c0 = np.zeros((2, n), dtype=np.uint64)
        c0[:, 0] = [x % p for p in primes]
        cases.append((c0, np.zeros((2, n), dtype=np.uint64)))
    before = P.native().fallbacks()
    bufs = np.stack([np.stack([a, b]) for a, b in cases])
    out = dev.to_host(F.mul_ct_batch(P, ek, 0, dev.to_device(bufs)))
    for i, (a, b) in enumerate(cases):
        want = ob.mul_ct(OP, ob.Ct(a, b), ob.Ct(a, b), K)
        assert np.array_equal(out[i], np.stack([want.c0, want.c1])), i
    assert P.native().fallbacks() > before
    # (3) decrypt rounding: w on the exact rounding boundary of floor((w t + h)/q)
    from paper_1811_09953_b200 import _lib

    ws = []
    for j in (1, 7, 123456789):
        # smallest w with w t + h >= j q, and its predecessor
        w = (j * q - h + t - 1) // t
        ws += [w, w - 1]
    W = np.zeros((1, 2, n), dtype=np.uint64)
    for i, w in enumerate(ws):
        W[0, :, i] = [w % p for p in primes]
    Wd = dev.to_device(W)
    M = dev.empty((1, n))
    _lib.check(_lib.lib().fcn_decrypt_round(P.native().ptr, 0, Wd.data_ptr(), M.data_ptr(), 1, dev.stream_ptr()))
    got = dev.to_host(M)[0]
    for i, w in enumerate(ws):
        assert int(got[i]) == ((w * t + h) // q) % t


def test_errors(F):
    from paper_1811_09953_b200 import encode

    P = F.EncryptionParams(1024, (36028797018972161, 36028797018990593), (1099511922689,))
    sk, pk, ek = F.keygen(P, 1)
    ct = F.encrypt(pk, P, encode.encode_integer(3, P.t_lanes[0]), 0, 4, 1)
    with pytest.raises(F.FVError):
        F.mul_pt(ct, F.PlainPoly.zero(P.t_lanes[0]))
    with pytest.raises(F.FVError):
        F.add_ct(ct, F.Ciphertext(ct.c0, ct.c1, P, 0, 5, 0))
    with pytest.raises(F.FVError):
        F.EncryptionParams(1000, (17,), (2,))
    assert F.add_pt(ct, F.PlainPoly.zero(P.t_lanes[0])) is ct


@pytest.mark.parametrize("env", [{"FCN_NTT_INT": "1"}, {"FCN_SQ_FUSE": "0"}, {"FCN_NTT_RS": "0"},
                                 {"FCN_DBL_ROWS": "0", "FCN_PRESCALE": "0"}, {"FCN_TWIST_C2": "0"},
                                 {"FCN_PRESCALE": "0"}, {"FCN_PAIR_RELIN": "0"}],
                         ids=["integer-kernels", "unfused-square", "ntt-rs0", "u64-rows", "scaling-epilogue",
                              "no-prescale", "per-limb-relin"])
def test_kernel_family_subprocess(env):
    """Kernel families the default dispatch does not pick for these shapes,
    each forced in a fresh process (the switches are read once per process):
    FCN_NTT_INT=1 the integer kernels (used for limbs >= 2^51), FCN_SQ_FUSE=0
    the separate forward NTT + tensor kernels for squares, FCN_NTT_RS=0 the
    FP64 NTT's every-third-stage reduction schedule (limbs near 2^51),
    FCN_DBL_ROWS=0 / FCN_PRESCALE=0 the square pipeline with canonical u64
    workspace rows and the rescale's first factor in the rescale kernel,
    FCN_TWIST_C2=0 the activation's c2 in the final INTT's epilogue instead
    of its twist, FCN_PAIR_RELIN=0 the per-limb relinearisation (digits
    transformed under every limb) where the default is the shared prime
    pair.  Squares (plain and with the fused a2 x^2 + a1 x
    activation) and NTTs on the cfg1/cfg2 shapes must match the oracle.
    Squares and NTTs on the cfg1/cfg2 shapes must match the oracle."""
    import os
    import subprocess
    import sys

    code = r"""
import numpy as np
from oracle import bfv as ob, rns as orn
from paper_1811_09953_b200 import configs, fv, ring
from paper_1811_09953_b200 import device as dev
for name in ("cfg1", "cfg2"):
    W = configs.WORKLOADS[name]
    P = fv.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    OP = ob.Params(W.n, W.primes, (W.t,), W.beta)
    sk, pk, ek = fv.keygen(P, 2)
    K = ob.Keys(sk.s.host(), pk.p0.host(), pk.p1.host(), [x.host() for x in ek.a], [x.host() for x in ek.g])
    rng = np.random.default_rng(1)
    x = np.stack([np.stack([orn.random_uniform(W.primes, W.n, rng) for _ in range(2)]) for _ in range(2)])
    out = dev.to_host(fv.mul_ct_batch(P, ek, 0, dev.to_device(x)))
    act = dev.to_host(fv.mul_ct_batch(P, ek, 0, dev.to_device(x), act=(-3, 5)))
    for b in range(2):
        c = ob.Ct(x[b, 0], x[b, 1])
        w = ob.mul_ct(OP, c, c, K)
        assert np.array_equal(out[b], np.stack([w.c0, w.c1])), (name, b)
        for p_i, (pa, xa) in enumerate(((w.c0, x[b, 0]), (w.c1, x[b, 1]))):
            for l, q in enumerate(W.primes):
                want = (pa[l].astype(object) * (-3 % q) + xa[l].astype(object) * 5) % q
                assert np.array_equal(act[b, p_i, l].astype(object), want), (name, b, p_i, l)
    ctx = ring.RingContext.create(W.n, W.primes)
    r = x[0, 0]
    assert np.array_equal(ring.ntt_forward(ring.RingPoly(ctx, r)).host(), orn.ntt(r, W.primes))
print("ok")
"""
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=repo, **env)
    res = subprocess.run([sys.executable, "-c", code], cwd=repo, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and res.stdout.strip().endswith("ok"), res.stdout[-2000:] + res.stderr[-2000:]


def _ctx_query(P, what):
    import ctypes as C

    from paper_1811_09953_b200 import _lib

    v = C.c_int64()
    _lib.check(_lib.lib().fcn_ctx_query(P.native().ptr, what, C.byref(v)))
    return v.value


def test_shared_pair_relin_selection(F):
    """Which parameter sets relinearise squares through the shared prime pair
    (fcn_ctx_query 7): beta = 2^32 with 50-bit limbs and k >= 3 (cfg2, cfg3,
    cfg4) do; cfg1 (37-bit limbs: q_0 q_1 is too small for the two-residue
    CRT), cfg5 (beta = 2^134: the digits are not below the limbs) and a
    two-limb set keep the per-limb form."""
    from paper_1811_09953_b200 import configs

    want = {"cfg1": 0, "cfg2": 1, "cfg3": 1, "cfg4": 1, "cfg5": 0}
    for name, on in want.items():
        W = configs.WORKLOADS[name]
        P = F.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
        assert _ctx_query(P, 7) == on, name
    P2 = F.EncryptionParams(1024, (1125899906826241, 1125899906820097), (65537,))
    assert _ctx_query(P2, 7) == 0
    # every k in 3..7 of 50-bit limbs has an exact-size FP64 lift / rescale and so the shared pair
    from oracle import nt as ont

    for k in (3, 5, 7):
        Pk = F.EncryptionParams(1024, tuple(ont.ntt_primes(1024, k, 50)), (65537,))
        assert _ctx_query(Pk, 6) == 1 and _ctx_query(Pk, 7) == 1, k
    P1 = F.EncryptionParams(1024, tuple(ont.ntt_primes(1024, 1, 50)), (65537,))
    assert _ctx_query(P1, 6) == 0 and _ctx_query(P1, 7) == 0


@pytest.mark.parametrize("n,k", [(1024, 3), (1024, 4), (1024, 5), (2048, 6), (1024, 7)])
def test_shared_pair_relin_extreme_keys(F, n, k):
    """Squares relinearised through the shared prime pair with evaluation-key
    words at the extremes of the centred lift of every limb ((q_j-1)/2,
    (q_j+1)/2, q_j-1, 0, 1, mixed per coefficient and per limb) and
    ciphertexts at the extremes too, so the rebuilt integer sums reach both
    signs at full magnitude: bit-exact against the oracle's per-limb
    relinearisation (fv.py:524-537), plain and with the fused activation."""
    from oracle import nt as ont
    from oracle import rns as orn
    from paper_1811_09953_b200 import device as dev
    from paper_1811_09953_b200 import ring

    primes = tuple(ont.ntt_primes(n, k, 50))
    P = F.EncryptionParams(n, primes, (65537,))
    assert _ctx_query(P, 7) == 1
    OP = ob.Params(n, primes, P.t_lanes, P.beta)
    rng = np.random.default_rng(11)
    D = P.ell + 1

    def extreme_poly(shift):
        rows = []
        for l, q in enumerate(primes):
            vals = [(q - 1) // 2, (q + 1) // 2, q - 1, 0, 1, (q - 1) // 2, (q + 1) // 2]
            idx = (np.arange(n) + shift + 3 * l) % len(vals)
            rows.append(np.array([vals[i] for i in idx], dtype=np.uint64))
        return np.stack(rows)

    a_h = [extreme_poly(i) if i % 2 == 0 else orn.random_uniform(primes, n, rng) for i in range(D)]
    g_h = [extreme_poly(2 * i + 1) for i in range(D)]
    # every key word at +q_j/2 and every digit large: the sums at full magnitude
    g_h[0] = np.stack([np.full(n, (q - 1) // 2, dtype=np.uint64) for q in primes])
    a_h[0] = np.stack([np.full(n, (q + 1) // 2, dtype=np.uint64) for q in primes])
    ek = F.EvalKeys(tuple(ring.RingPoly(P.ctx, x) for x in a_h), tuple(ring.RingPoly(P.ctx, x) for x in g_h))
    K = ob.Keys(None, None, None, a_h, g_h)
    q = math.prod(primes)
    full = lambda v: np.stack([np.full(n, v % p, dtype=np.uint64) for p in primes])
    cts = [np.stack([orn.random_uniform(primes, n, rng) for _ in range(2)]) for _ in range(3)]
    cts.append(np.stack([full(q - 1), full((q - 1) // 2)]))
    cts.append(np.stack([extreme_poly(0), extreme_poly(5)]))
    x = np.stack(cts)
    for act in (None, (-3, 5), (12345, -32768)):
        # a second destination exercises the fan-out stores of both final inverses (the sharded evaluator's form)
        peer = dev.empty(x.shape)
        got = dev.to_host(F.mul_ct_batch(P, ek, 0, dev.to_device(x), act=act, chunk=2, fanout=(peer.data_ptr(),)))
        assert np.array_equal(dev.to_host(peer), got), act
        for b in range(len(cts)):
            c = ob.Ct(x[b, 0], x[b, 1])
            sq = ob.mul_ct(OP, c, c, K)
            for p_i, (pa, xa) in enumerate(((sq.c0, x[b, 0]), (sq.c1, x[b, 1]))):
                for l, ql in enumerate(primes):
                    if act is None:
                        want = pa[l].astype(object)
                    else:
                        want = (pa[l].astype(object) * (act[0] % ql) + xa[l].astype(object) * (act[1] % ql)) % ql
                    assert np.array_equal(got[b, p_i, l].astype(object), want), (act, b, p_i, l)


def test_single_limb_square_vs_oracle(F):
    """k = 1 (one 50-bit limb, two digits; integer lift / rescale kernels):
    squares against the oracle."""
    from oracle import nt as ont
    from oracle import rns as orn
    from paper_1811_09953_b200 import device as dev

    n = 1024
    primes = tuple(ont.ntt_primes(n, 1, 50))
    P = F.EncryptionParams(n, primes, (65537,))
    OP = ob.Params(n, primes, P.t_lanes, P.beta)
    sk, pk, ek = F.keygen(P, 4)
    K = ob.Keys(sk.s.host(), pk.p0.host(), pk.p1.host(), [x.host() for x in ek.a], [x.host() for x in ek.g])
    rng = np.random.default_rng(8)
    q = primes[0]
    cts = [np.stack([orn.random_uniform(primes, n, rng) for _ in range(2)]) for _ in range(2)]
    cts.append(np.stack([np.full((1, n), q - 1, dtype=np.uint64), np.full((1, n), (q - 1) // 2, dtype=np.uint64)]))
    x = np.stack(cts)
    got = dev.to_host(F.mul_ct_batch(P, ek, 0, dev.to_device(x)))
    for b in range(len(cts)):
        c = ob.Ct(x[b, 0], x[b, 1])
        w = ob.mul_ct(OP, c, c, K)
        assert np.array_equal(got[b], np.stack([w.c0, w.c1])), b


def test_empty_and_single_unit_batches(F):
    """Edge cases of the C ABI on the cfg2 ring: zero-count calls return OK and
    leave the output untouched; squares of batches of 1, 2 and 5 ciphertexts
    (fewer fused (ciphertext, limb) units than resident CTAs, an odd count)
    match the oracle."""
    import torch

    from oracle import rns as orn
    from paper_1811_09953_b200 import _lib, configs
    from paper_1811_09953_b200 import device as dev

    W = configs.WORKLOADS["cfg2"]
    P = F.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    OP = ob.Params(W.n, W.primes, (W.t,), W.beta)
    sk, pk, ek = F.keygen(P, 2)
    L, h, st = _lib.lib(), P.native(), dev.stream_ptr()
    k, n = len(W.primes), W.n
    sentinel = dev.zeros((1, 2, k, n)) + 7
    ws = F.mul_ct_workspace(P, 1)
    kh = ek.native(P)
    assert L.fcn_ntt_forward(h.ring_ptr, sentinel.data_ptr(), 0, k, 0, st) == 0
    assert L.fcn_ntt_inverse(h.ring_ptr, sentinel.data_ptr(), 0, k, 0, st) == 0
    assert L.fcn_mul_ct_ex(h.ptr, kh.ptr, 0, sentinel.data_ptr(), None, sentinel.data_ptr(), 0, 0, 1, 0,
                           ws.data_ptr(), ws.numel() * 8, st) == 0
    assert L.fcn_key_mac(h.ptr, kh.ptr, sentinel.data_ptr(), sentinel.data_ptr(), 0, st) == 0
    torch.cuda.synchronize()
    assert bool((sentinel == 7).all())
    K = ob.Keys(sk.s.host(), pk.p0.host(), pk.p1.host(), [x.host() for x in ek.a], [x.host() for x in ek.g])
    rng = np.random.default_rng(3)
    for B in (1, 2, 5):
        x = np.stack([np.stack([orn.random_uniform(W.primes, n, rng) for _ in range(2)]) for _ in range(B)])
        out = dev.to_host(F.mul_ct_batch(P, ek, 0, dev.to_device(x)))
        for b in {0, B - 1}:
            want = ob.mul_ct(OP, ob.Ct(x[b, 0], x[b, 1]), ob.Ct(x[b, 0], x[b, 1]), K)
            assert np.array_equal(out[b], np.stack([want.c0, want.c1])), (B, b)


def test_wire_format_round_trip_cfg2(F):
    """Reference A6 / test_fv.py serialization: at the cfg2 shape a
    ciphertext is 65,544 u64 words (64-byte header + [2][4][8192] body), so
    784 of them are 411,091,968 bytes; bytes -> ciphertext -> bytes is the
    identity (data and lane / scale / depth metadata), truncation, trailing
    bytes and evaluation-key bytes are rejected."""
    from paper_1811_09953_b200 import configs

    W = configs.WORKLOADS["cfg2"]
    P = F.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    sk, pk, ek = F.keygen(P, 2)
    assert F.ciphertext_num_words(P) == 65544
    assert 784 * F.ciphertext_num_words(P) * 8 == 411091968
    ct = F.encrypt(pk, P, F.PlainPoly(W.t, [7, 0, 3]), 0, 5, np.random.default_rng(1))
    sq = F.mul_ct(ct, ct, ek)
    for c in (ct, sq):
        data = F.ciphertext_to_bytes(c)
        assert len(data) == 65544 * 8
        back = F.ciphertext_from_bytes(data, P)
        assert F.ciphertext_to_bytes(back) == data
        assert (back.lane, back.scale_exponent, back.mul_depth) == (c.lane, c.scale_exponent, c.mul_depth)
        with pytest.raises(F.FVError):
            F.ciphertext_from_bytes(data[:-8], P)
        with pytest.raises(F.FVError):
            F.ciphertext_from_bytes(data + bytes(8), P)
    with pytest.raises(F.FVError):
        F.ciphertext_from_bytes(F.eval_keys_to_bytes(ek, P), P)


def test_homomorphic_round_trips_random(F):
    """Reference A2-style homomorphism on the FP64 hot path (n = 1024, three
    primes just above 2^50, t = 65537): for random plaintext polynomials a, b
    and constants c, decrypt(add_ct) = a + b, decrypt(mul_pt) = c a and
    decrypt(mul_ct) = a b in Z_t[x]/(x^n + 1)."""
    from paper_1811_09953_b200 import configs

    n, t = 1024, 65537
    primes = tuple(configs.find_ntt_primes(n, 3, bits=50))
    P = F.EncryptionParams(n, primes, (t,), 1 << 32)
    sk, pk, ek = F.keygen(P, 11)
    rng = np.random.default_rng(12)

    def negacyclic(a, b):
        full = np.zeros(2 * n, dtype=object)
        for i in np.nonzero(a)[0]:
            full[i : i + n] += int(a[i]) * b.astype(object)
        return np.array([(full[j] - full[j + n]) % t for j in range(n)], dtype=object)

    def dense(p):
        out = np.zeros(n, dtype=object)
        out[: p.coeffs.size] = p.coeffs.astype(object)
        return out

    for trial in range(12):
        a = np.zeros(n, dtype=np.uint64)
        b = np.zeros(n, dtype=np.uint64)
        ia = rng.choice(n, 6, replace=False)
        ib = rng.choice(n, 6, replace=False)
        a[ia] = rng.integers(0, t, 6)
        b[ib] = rng.integers(0, t, 6)
        c = int(rng.integers(1, t))
        ca = F.encrypt(pk, P, F.PlainPoly(t, a), 0, 0, rng)
        cb = F.encrypt(pk, P, F.PlainPoly(t, b), 0, 0, rng)
        A, B = a.astype(object), b.astype(object)
        assert np.array_equal(dense(F.decrypt(sk, F.add_ct(ca, cb))), (A + B) % t), trial
        assert np.array_equal(dense(F.decrypt(sk, F.mul_pt(ca, F.PlainPoly(t, [c])))), (A * c) % t), trial
        assert np.array_equal(dense(F.decrypt(sk, F.mul_ct(ca, cb, ek))), negacyclic(a, b)), trial


def test_cfg5_full_batch_square_decrypts():
    """BASELINE configs[4] at full size: 4,096 ciphertexts of n = 16384 over
    8 limbs, squared and relinearised with the dnum = 3 key (beta = 2^134) in
    one batched call (the sweep's operation); every result decrypts to the
    square of its plaintext m = c + d x^j in Z_t[x]/(x^n + 1)."""
    from paper_1811_09953_b200 import configs
    from paper_1811_09953_b200 import device as dev
    from paper_1811_09953_b200 import fv as F

    W = configs.WORKLOADS["cfg5"]
    P = F.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    assert P.ell + 1 == 3
    sk, pk, ek = F.keygen(P, configs.SEED_KEYS)
    B, n, t = 4096, W.n, W.t
    rng = np.random.default_rng(21)
    c = rng.integers(-(t // 2), t // 2 + 1, B)
    d = rng.integers(-(t // 2), t // 2 + 1, B)
    j = rng.integers(1, n, B)
    plain = np.zeros((B, n), dtype=np.int64)
    plain[:, 0] = c
    plain[np.arange(B), j] = d
    cts = F.encrypt_batch(pk, P, plain, 0, np.random.default_rng(22))
    sq = F.mul_ct_batch(P, ek, 0, cts)
    got = F.decrypt_batch(sk, P, sq).astype(np.int64)
    want = np.zeros((B, n), dtype=object)
    want[:, 0] = c.astype(object) ** 2
    want[np.arange(B), j] += 2 * c.astype(object) * d.astype(object)
    for b in range(B):  # d^2 x^(2j): negacyclic wrap
        e = 2 * int(j[b])
        if e < n:
            want[b, e] += int(d[b]) ** 2
        else:
            want[b, e - n] -= int(d[b]) ** 2
    assert np.array_equal(got, (want % t).astype(np.int64))
    # bit-exact against the oracle on ciphertexts from inside the batch
    # (first, middle, last): the batched call equals the reference's mul_ct
    from oracle import bfv as ob

    OP = ob.Params(n, tuple(W.primes), (t,), W.beta)
    K = ob.Keys(sk.s.host(), pk.p0.host(), pk.p1.host(), [a.host() for a in ek.a], [g.host() for g in ek.g])
    xs, ys = dev.to_host(cts), dev.to_host(sq)
    for b in (0, 2049, B - 1):
        x = ob.Ct(xs[b, 0], xs[b, 1])
        w = ob.mul_ct(OP, x, x, K)
        assert np.array_equal(ys[b], np.stack([w.c0, w.c1])), b


@pytest.mark.parametrize("k,bits,n", [(4, 50, 1024), (3, 36, 4096), (2, 55, 1024), (6, 50, 2048)])
def test_noise_budget_on_gpu_matches_oracle(k, bits, n):
    """fv.noise_budget (fcn_noise_max: multiword CRT + block maxima on the
    GPU, the reference's log2 on the host; fv.py:356-377) equals the
    oracle's big-int computation exactly, fresh and after a square."""
    from oracle import bfv as ob
    from paper_1811_09953_b200 import configs
    from paper_1811_09953_b200 import device as dev
    from paper_1811_09953_b200 import fv as F

    primes = tuple(configs.find_ntt_primes(n, k, bits=bits))
    P = F.EncryptionParams(n, primes, (65537,), 1 << 32)
    OP = ob.Params(n, primes, (65537,), 1 << 32)
    sk, pk, ek = F.keygen(P, 8)
    K = ob.Keys(sk.s.host(), pk.p0.host(), pk.p1.host(), [a.host() for a in ek.a], [g.host() for g in ek.g])
    rng = np.random.default_rng(n + k)
    plain = rng.integers(-300, 300, (5, n))
    cts = F.encrypt_batch(pk, P, plain, 0, np.random.default_rng(9))
    sq = F.mul_ct_batch(P, ek, 0, cts)
    for buf in (cts, sq):
        got = F.noise_budget_batch(sk, P, buf)
        host = dev.to_host(buf)
        for b in range(buf.shape[0]):
            want = ob.noise_budget(OP, K, ob.Ct(host[b, 0], host[b, 1]))
            assert got[b] == want, (b, got[b], want)
    one = F.ciphertext_from_buffer(P, cts[0])
    assert F.noise_budget(sk, one) == ob.noise_budget(OP, K, ob.Ct(dev.to_host(cts)[0, 0], dev.to_host(cts)[0, 1]))
