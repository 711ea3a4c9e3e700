"""Small runs of every hot kernel for compute-sanitizer (memcheck / racecheck /
synccheck): the FP64 NTTs (fwd, inv, the barrier-elided next-row prefetch,
the per-warp copy-out), the fused square pipeline (lift, fwd_sq, prescaled
INTT, rescale, digit NTT, key MAC, INTT epilogue), the sparse MAC
(mac_fast_kernel) and the tensor-core MAC (split_planes, mac_tc_kernel), at
n = 1024 and n = 8192; each result is checked against the oracle.

usage: compute-sanitizer --tool memcheck python tools/sanitize.py [n ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import bfv as ob  # noqa: E402
from oracle import rns as orn  # noqa: E402
from paper_1811_09953_b200 import configs, engine, fv, mac_tc, ring  # noqa: E402
from paper_1811_09953_b200 import device as dev  # noqa: E402


def run(n: int):
    rng = np.random.default_rng(n)
    primes = tuple(configs.find_ntt_primes(n, 4, bits=50))
    P = fv.EncryptionParams(n, primes, (65537,), 1 << 32)
    # NTT fwd / inv over several rows (row prefetch + copy-out paths)
    ctx = ring.RingContext.create(n, primes)
    x = orn.random_uniform(primes, n, rng)
    f = ring.ntt_forward(ring.RingPoly(ctx, x)).host()
    assert np.array_equal(f, orn.ntt(x, primes)), "NTT"
    rows = dev.to_device(np.stack([orn.random_uniform(primes, n, rng) for _ in range(3)]).reshape(-1, n))
    h = P.native()
    from paper_1811_09953_b200 import _lib

    L = _lib.lib()
    before = rows.clone()
    _lib.check(L.fcn_ntt_forward(h.ring_ptr, rows.data_ptr(), rows.shape[0], 4, 0, dev.stream_ptr()))
    _lib.check(L.fcn_ntt_inverse(h.ring_ptr, rows.data_ptr(), rows.shape[0], 4, 0, dev.stream_ptr()))
    torch.cuda.synchronize()
    assert torch.equal(rows, before), "NTT round trip"
    # square pipeline with the activation epilogue, 3 ciphertexts
    sk, pk, ek = fv.keygen(P, 5)
    K = ob.Keys(sk.s.host(), pk.p0.host(), pk.p1.host(), [a.host() for a in ek.a], [g.host() for g in ek.g])
    OP = ob.Params(n, primes, (65537,), 1 << 32)
    cts = np.stack([np.stack([orn.random_uniform(primes, n, rng) for _ in range(2)]) for _ in range(3)])
    out = dev.to_host(fv.mul_ct_batch(P, ek, 0, dev.to_device(cts)))
    w = ob.mul_ct(OP, ob.Ct(cts[0, 0], cts[0, 1]), ob.Ct(cts[0, 0], cts[0, 1]), K)
    assert np.array_equal(out[0], np.stack([w.c0, w.c1])), "mul_ct"
    fv.mul_ct_batch(P, ek, 0, dev.to_device(cts), act=(8, -2))
    torch.cuda.synchronize()
    # linear layers: sparse kernel and tensor cores on the same plan
    plan = configs.mac_sweep_plan(n_out=130, n_in=70, terms=20, seed=n)
    mac, _, _ = engine._lower_linear(plan, 65537, n, "batched")
    xin = dev.to_device(np.stack([np.stack([orn.random_uniform(primes, n, rng) for _ in range(2)]) for _ in range(70)]))
    want = engine._mac_out(P, mac, xin, None)
    tcp = mac_tc.build(mac, 70, L.fcn_tc_planes(h.ptr), 2 * 4 * n, force=True)
    got = torch.empty_like(want)
    mac_tc.run(P, tcp, xin, got)
    torch.cuda.synchronize()
    assert torch.equal(got, want), "tensor-core MAC"
    print(f"n={n} ok", flush=True)


if __name__ == "__main__":
    for n in [int(a) for a in sys.argv[1:]] or [1024, 8192]:
        run(n)
