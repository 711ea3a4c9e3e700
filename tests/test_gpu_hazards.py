"""Memory-safety and race checks of the hot kernels without compute-sanitizer
(closed on this GPU pool): guard bands around every output buffer, repeated
launches that must reproduce the same bytes, and launches with many more rows
than resident CTAs so every persistent CTA runs the barrier-elided paths of
the FP64 NTT (the next row's cp.async issued before the copy-out barrier,
the per-warp copy-out) many times; results against the oracle."""

import numpy as np
import pytest
import torch

from oracle import bfv as ob
from oracle import rns as orn
from paper_1811_09953_b200 import _lib, configs, engine, fv, mac_tc
from paper_1811_09953_b200 import device as dev

pytestmark = pytest.mark.gpu

SENTINEL = 0x5A5A5A5A5A5A5A5A
GUARD = 4096


def _guarded(shape, fill=None):
    """A view of `shape` inside a buffer with GUARD words of sentinel on both sides."""
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * GUARD,), SENTINEL, dtype=torch.int64, device="cuda")
    view = buf[GUARD:GUARD + n].view(shape)
    if fill is not None:
        view.copy_(fill)
    return buf, view


def _guards_intact(buf):
    torch.cuda.synchronize()
    return bool((buf[:GUARD] == SENTINEL).all()) and bool((buf[-GUARD:] == SENTINEL).all())


@pytest.mark.parametrize("n,k", [(1024, 4), (8192, 4), (16384, 3)])
def test_ntt_many_rows_guarded_repeatable(n, k):
    primes = tuple(configs.find_ntt_primes(n, k, bits=50))
    P = fv.EncryptionParams(n, primes, (65537,), 1 << 32)
    h = P.native()
    L = _lib.lib()
    rng = np.random.default_rng(n + k)
    rows = 148 * 6 * k  # several rows per resident CTA (prefetch / copy-out paths)
    host = np.stack([orn.random_uniform(primes, n, rng) for _ in range(rows // k)]).reshape(rows, n)
    buf, x = _guarded((rows, n), torch.from_numpy(host.view(np.int64)).cuda())
    ref = None
    for rep in range(5):
        x.copy_(torch.from_numpy(host.view(np.int64)).cuda())
        _lib.check(L.fcn_ntt_forward(h.ring_ptr, x.data_ptr(), rows, k, 0, dev.stream_ptr()))
        fwd = x.clone()
        _lib.check(L.fcn_ntt_inverse(h.ring_ptr, x.data_ptr(), rows, k, 0, dev.stream_ptr()))
        assert _guards_intact(buf)
        assert np.array_equal(dev.to_host(x), host), "inverse(forward(x)) != x"
        if ref is None:
            ref = fwd
            fh = dev.to_host(fwd)
            for r in (0, 1, rows // 2, rows - 1):  # spot rows against the oracle
                want = orn.ntt(host[r - r % k:r - r % k + k], primes)[r % k]
                assert np.array_equal(fh[r], want)
        else:
            assert torch.equal(fwd, ref), "forward NTT not reproducible"


@pytest.mark.parametrize("n,k,count,chunk", [(1024, 4, 300, 16), (8192, 4, 40, 16), (16384, 6, 48, 48)])
def test_square_pipeline_guarded_repeatable(n, k, count, chunk):
    primes = tuple(configs.find_ntt_primes(n, k, bits=50))
    P = fv.EncryptionParams(n, primes, (65537,), 1 << 32)
    sk, pk, ek = fv.keygen(P, 7)
    rng = np.random.default_rng(count)
    cts = np.stack([np.stack([orn.random_uniform(primes, n, rng) for _ in range(2)]) for _ in range(count)])
    x = dev.to_device(cts)
    buf, out = _guarded(tuple(x.shape))
    # the cfg3 shape runs one chunk of 48: 384 (poly, limb) units of the paired inverse over 148 resident CTAs
    ws_bytes = _lib.lib().fcn_mul_ct_workspace_bytes(P.native().ptr, chunk)
    wbuf, ws = _guarded((ws_bytes // 8 + 1,))
    first = None
    for rep in range(3):
        fv.mul_ct_batch(P, ek, 0, x, out=out, workspace=ws, act=(8, -2))  # chunks through the workspace
        assert _guards_intact(buf) and _guards_intact(wbuf)
        if first is None:
            first = out.clone()
        else:
            assert torch.equal(out, first), "square pipeline not reproducible"
    OP = ob.Params(n, primes, (65537,), 1 << 32)
    K = ob.Keys(sk.s.host(), pk.p0.host(), pk.p1.host(), [a.host() for a in ek.a], [g.host() for g in ek.g])
    got = dev.to_host(first)
    for b in (0, count // 2, count - 1):
        c = ob.Ct(cts[b, 0], cts[b, 1], 0, 6, 0)
        sq = ob.mul_ct(OP, c, c, K)
        a2 = ob.mul_pt(OP, sq, [8], 6)
        w = ob.add_ct(OP, a2, ob.mul_pt(OP, c, [65535], a2.scale - c.scale))
        assert np.array_equal(got[b], np.stack([w.c0, w.c1]))


@pytest.mark.parametrize("tc", [False, True])
def test_linear_layers_guarded_repeatable(tc):
    n, k = 1024, 4
    primes = tuple(configs.find_ntt_primes(n, k, bits=50))
    P = fv.EncryptionParams(n, primes, (65537,), 1 << 32)
    plan = configs.mac_sweep_plan(n_out=300, n_in=257, terms=60, seed=4)
    mac, _, _ = engine._lower_linear(plan, 65537, n, "batched")
    rng = np.random.default_rng(5)
    xin = dev.to_device(np.stack([np.stack([orn.random_uniform(primes, n, rng) for _ in range(2)]) for _ in range(257)]))
    want = engine._mac_out(P, mac, xin, None)
    tcp = mac_tc.build(mac, 257, _lib.lib().fcn_tc_planes(P.native().ptr), 2 * k * n, force=True) if tc else None
    buf, out = _guarded(tuple(want.shape))
    for rep in range(4):
        out.fill_(0)
        if tc:
            mac_tc.run(P, tcp, xin, out)
        else:
            engine._mac_out(P, mac, xin, None, out=out)
        assert _guards_intact(buf)
        assert torch.equal(out, want)


def test_split_planes_guarded():
    n, k = 1024, 4
    primes = tuple(configs.find_ntt_primes(n, k, bits=50))
    P = fv.EncryptionParams(n, primes, (65537,), 1 << 32)
    h = P.native()
    L = _lib.lib()
    rng = np.random.default_rng(6)
    count = 37
    x = dev.to_device(np.stack([np.stack([orn.random_uniform(primes, n, rng) for _ in range(2)]) for _ in range(count)]))
    nbytes = L.fcn_tc_planes_bytes(h.ptr, count)
    pad = torch.full((nbytes + 2 * GUARD,), 0xA5, dtype=torch.uint8, device="cuda")
    planes = pad[GUARD:GUARD + nbytes]
    _lib.check(L.fcn_split_planes(h.ptr, x.data_ptr(), count, planes.data_ptr(), dev.stream_ptr()))
    torch.cuda.synchronize()
    assert bool((pad[:GUARD] == 0xA5).all()) and bool((pad[-GUARD:] == 0xA5).all())
    P_ = L.fcn_tc_planes(h.ptr)
    cols = 2 * k * n
    pitch = cols + 256
    pl = planes.view(count, P_, pitch)[:, :, :cols].cpu().numpy().astype(np.uint64)
    xs = dev.to_host(x).reshape(count, cols)
    rebuilt = sum(pl[:, b, :] << np.uint64(8 * b) for b in range(P_))
    assert np.array_equal(rebuilt, xs)
