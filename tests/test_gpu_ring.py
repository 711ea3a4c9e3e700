"""GPU parity of the ring layer (libfcn NTT / elementwise / monomial) against
the reference golden vectors and the CPU oracle.  Bit-exact."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import rns as orn  # noqa: E402


@pytest.fixture(scope="module")
def R():
    import torch

    from paper_1811_09953_b200 import ring

    assert torch.cuda.is_available()
    return ring


@pytest.mark.parametrize("name", ["n4", "n16", "n1024", "n4096", "n8192", "n16384", "t65537_n1024"])
def test_ntt_matches_reference_golden(R, name, golden_meta, golden_npz):
    d = golden_npz("ntt")
    m = golden_meta["ntt"][name]
    ctx = R.RingContext.create(m["n"], m["primes"])
    assert [l.root for l in ctx.limbs] == m["roots"]
    x = R.RingPoly(ctx, d[f"{name}_in"])
    f = R.ntt_forward(x)
    assert np.array_equal(f.host(), d[f"{name}_fwd"])
    g = R.ntt_inverse(R.RingPoly(ctx, d[f"{name}_in"], R.NTT))
    assert np.array_equal(g.host(), d[f"{name}_inv"])
    assert R.ntt_inverse(f) == x


@pytest.mark.parametrize("n", [4, 8, 32, 64, 256, 2048, 32768])
def test_ntt_all_degrees_vs_oracle(R, n):
    rng = np.random.default_rng(n)
    from oracle import nt

    primes = tuple(nt.ntt_primes(n, 2, bits=55))
    ctx = R.RingContext.create(n, primes)
    x = orn.random_uniform(primes, n, rng)
    f = R.ntt_forward(R.RingPoly(ctx, x))
    assert np.array_equal(f.host(), orn.ntt(x, primes))
    assert np.array_equal(R.ntt_inverse(R.RingPoly(ctx, x, R.NTT)).host(), orn.intt(x, primes))
    assert np.array_equal(R.ntt_inverse(f).host(), x)


def test_ntt_extreme_values(R):
    # all-(q-1) rows and 61-bit primes exercise the lazy [0,4q) ranges
    from oracle import nt

    n = 4096
    primes = tuple(nt.ntt_primes(n, 2, bits=61))
    ctx = R.RingContext.create(n, primes)
    x = np.stack([np.full(n, q - 1, dtype=np.uint64) for q in primes])
    assert np.array_equal(R.ntt_forward(R.RingPoly(ctx, x)).host(), orn.ntt(x, primes))
    assert np.array_equal(R.ntt_inverse(R.RingPoly(ctx, x, R.NTT)).host(), orn.intt(x, primes))


def _primes_below_2_51(n, count):
    """NTT primes just below 2^51 (the auxiliary-base rule of libfcn):
    the tightest case of the FP64 kernels' |x| < 3.86 q < 2^53 bound."""
    from oracle import nt

    step = 2 * n
    p = ((1 << 51) // step) * step + 1
    out = []
    while len(out) < count:
        p -= step
        if nt.is_prime(p):
            out.append(p)
    return tuple(out)


def _largest_primes_with_schedule(n, rs, count):
    """The largest NTT primes for which the FP64 NTT picks reduction
    schedule rs (ntt.cu f64_schedule): the tightest case of its bound."""
    from oracle import nt
    from paper_1811_09953_b200 import _lib

    L = _lib.load()
    logn = n.bit_length() - 1
    lo, hi = 1 << 30, (1 << 51) - 1
    while hi - lo > 1:  # largest q with schedule >= rs
        mid = (lo + hi) // 2
        if L.fcn_ntt_f64_schedule(logn, mid) >= rs:
            lo = mid
        else:
            hi = mid
    step = 2 * n
    p = (lo // step) * step + 1
    out = []
    while len(out) < count:
        if p <= lo and nt.is_prime(p) and L.fcn_ntt_f64_schedule(logn, p) == rs:
            out.append(p)
        p -= step
    return tuple(out)


def _extreme_rows(n, primes):
    rng = np.random.default_rng(n)
    return [
        [np.full(n, q - 1, dtype=np.uint64) for q in primes],
        [np.full(n, (q - 1) // 2, dtype=np.uint64) for q in primes],
        [np.full(n, (q + 1) // 2, dtype=np.uint64) for q in primes],
        [np.where(np.arange(n) % 2 == 0, 0, q - 1).astype(np.uint64) for q in primes],
        [rng.integers(0, q, n, dtype=np.uint64) for q in primes],
    ]


@pytest.mark.parametrize("n", [1024, 8192, 16384])
def test_ntt_fp64_extreme_values_near_2_51(R, n):
    """FP64 NTT (q < 2^51) on rows that maximise every intermediate:
    all q-1, all (q-1)/2, all (q+1)/2, alternating 0 / q-1, and random."""
    primes = _primes_below_2_51(n, 2)
    ctx = R.RingContext.create(n, primes)
    for rows in _extreme_rows(n, primes):
        x = np.stack(rows)
        assert np.array_equal(R.ntt_forward(R.RingPoly(ctx, x)).host(), orn.ntt(x, primes))
        assert np.array_equal(R.ntt_inverse(R.RingPoly(ctx, x, R.NTT)).host(), orn.intt(x, primes))


@pytest.mark.parametrize("rs", [1, 2])
@pytest.mark.parametrize("n", [1024, 2048, 4096, 8192, 16384])
def test_ntt_fp64_reduced_schedules_at_their_limit(R, n, rs):
    """The cheaper FP64 reduction schedules (one reduction per transform,
    none) on the largest primes that select them, with extreme rows; also
    the epilogue inverse through mul_ct is covered by the cfg tests."""
    primes = _largest_primes_with_schedule(n, rs, 2)
    ctx = R.RingContext.create(n, primes)
    for rows in _extreme_rows(n, primes):
        x = np.stack(rows)
        assert np.array_equal(R.ntt_forward(R.RingPoly(ctx, x)).host(), orn.ntt(x, primes))
        assert np.array_equal(R.ntt_inverse(R.RingPoly(ctx, x, R.NTT)).host(), orn.intt(x, primes))


def test_ring_ops_match_reference(R, golden_meta, golden_npz):
    d = golden_npz("ringops")
    m = golden_meta["ringops"]
    ctx = R.RingContext.create(m["n"], m["primes"])
    a, b = R.RingPoly(ctx, d["a"]), R.RingPoly(ctx, d["b"])
    assert np.array_equal(R.poly_add(a, b).host(), d["add"])
    assert np.array_equal(R.poly_sub(a, b).host(), d["sub"])
    assert np.array_equal(R.poly_neg(a).host(), d["neg"])
    assert np.array_equal(R.scalar_mul(a, -12345).host(), d["scalar_m12345"])
    fa, fb = R.ntt_forward(a), R.ntt_forward(b)
    assert np.array_equal(R.pointwise_mul(fa, fb).host(), d["pointwise"])
    assert np.array_equal(R.poly_mul_ntt(a, b).host(), d["polymul"])
    for i, (k, c) in enumerate(m["monomials"]):
        assert np.array_equal(R.poly_mul_monomial(a, k, c).host(), d[f"mono{i}"])
    ctx64 = R.RingContext.create(64, m["sb_primes"])
    xy = R.poly_mul_ntt(R.RingPoly(ctx64, d["sb_x"]), R.RingPoly(ctx64, d["sb_y"]))
    assert np.array_equal(xy.host(), d["sb_xy"])


def test_hand_known_answers(R):
    ctx = R.RingContext.create(4, (17,))
    p = R.RingPoly.from_int_coeffs(ctx, [1, 1])
    assert R.poly_mul_ntt(p, p).host()[0].tolist() == [1, 2, 1, 0]
    x3 = R.RingPoly.from_int_coeffs(ctx, [0, 0, 0, 1])
    x1 = R.RingPoly.from_int_coeffs(ctx, [0, 1])
    assert R.poly_mul_ntt(x3, x1).host()[0].tolist() == [16, 0, 0, 0]
    assert R.poly_mul_monomial(x3, 1, 1).host()[0].tolist() == [16, 0, 0, 0]
    one = R.RingPoly.from_int_coeffs(ctx, [1])
    assert R.poly_mul_monomial(one, 0, -1).host()[0].tolist() == [16, 0, 0, 0]


def test_monomial_equals_ntt_product(R):
    # reference tests/test_ring.py:124-136 and acceptance A3 (n=8192)
    from oracle import nt

    rng = np.random.default_rng(3)
    for n, cnt in ((512, 20), (8192, 8)):
        primes = tuple(nt.ntt_primes(n, 2, bits=55))
        ctx = R.RingContext.create(n, primes)
        t = 1099511922689
        for _ in range(cnt):
            c = R.RingPoly(ctx, orn.random_uniform(primes, n, rng))
            k = int(rng.integers(0, n))
            coeff = int(rng.integers(-(t // 2), t // 2 + 1))
            mono = [0] * (k + 1)
            mono[k] = coeff
            want = R.poly_mul_ntt(c, R.RingPoly.from_int_coeffs(ctx, mono))
            assert R.poly_mul_monomial(c, k, coeff) == want


def test_errors(R):
    ctx = R.RingContext.create(4, (17,))
    p = R.RingPoly.zero(ctx)
    with pytest.raises(R.RingError):
        R.ntt_inverse(p)
    with pytest.raises(R.RingError):
        R.ntt_forward(R.ntt_forward(p))
    with pytest.raises(R.RingError):
        R.poly_mul_monomial(p, 4, 1)
    with pytest.raises(R.RingError):
        R.RingContext.create(4, (19,))  # 19 != 1 mod 8
    with pytest.raises(R.RingError):
        R.RingContext.create(1000, (17,))


def test_batched_rows_many_polys(R):
    """One launch over a [B][2][k][n] batch equals per-row oracle transforms."""
    import torch

    from oracle import nt
    from paper_1811_09953_b200 import _lib
    from paper_1811_09953_b200 import device as dev

    n, k, B = 8192, 4, 12
    primes = tuple(nt.ntt_primes(n, k, bits=50))
    ctx = R.RingContext.create(n, primes)
    rng = np.random.default_rng(9)
    x = np.stack([orn.random_uniform(primes, n, rng) for _ in range(2 * B)]).reshape(B, 2, k, n)
    d = dev.to_device(x)
    _lib.check(_lib.lib().fcn_ntt_forward(ctx.handle().ptr, d.data_ptr(), B * 2 * k, k, 0, dev.stream_ptr()))
    got = dev.to_host(d)
    for b in (0, 5, B - 1):
        for p in range(2):
            assert np.array_equal(got[b, p], orn.ntt(x[b, p], primes))
    _lib.check(_lib.lib().fcn_ntt_inverse(ctx.handle().ptr, d.data_ptr(), B * 2 * k, k, 0, dev.stream_ptr()))
    torch.cuda.synchronize()
    assert np.array_equal(dev.to_host(d), x)
