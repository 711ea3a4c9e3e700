"""Kernel micro-benchmarks: batched NTT at a workload's ring shape.

usage: python tools/kbench.py [workload] [iters]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1811_09953_b200 import _lib, configs, fv  # noqa: E402
from paper_1811_09953_b200 import device as dev  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    W = configs.WORKLOADS[wl]
    P = fv.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    h = P.native()
    K = len(P.limb_primes) + len(h.aux)
    n = P.n
    rows = max(K, (512 << 20) // (n * 8) // K * K)
    g = torch.Generator(device="cuda").manual_seed(0)
    buf = torch.randint(0, 1 << 50, (rows, n), device="cuda", dtype=torch.int64, generator=g)
    L = _lib.lib()
    st = dev.stream_ptr()
    for name, fn in (("fwd", L.fcn_ntt_forward), ("inv", L.fcn_ntt_inverse)):
        for _ in range(2):
            _lib.check(fn(h.ring_ptr, buf.data_ptr(), rows, K, 0, st))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            _lib.check(fn(h.ring_ptr, buf.data_ptr(), rows, K, 0, st))
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / iters
        gbs = 2 * rows * n * 8 / (t / 1e3) / 1e9
        print(f"{wl} n={n} rows={rows} {name}: {t:.3f} ms/launch  {gbs:.0f} GB/s")


if __name__ == "__main__":
    main()
