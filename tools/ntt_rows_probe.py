"""NTT time per row against the launch's row count (L2-resident vs HBM-streaming rows).

usage: python tools/ntt_rows_probe.py [workload]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1811_09953_b200 import _lib, configs, fv  # noqa: E402
from paper_1811_09953_b200 import device as dev  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    W = configs.WORKLOADS[wl]
    P = fv.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    h = P.native()
    K = len(P.limb_primes) + len(h.aux)
    n = P.n
    per_sm = 16384 // n
    L = _lib.lib()
    st = dev.stream_ptr()
    g = torch.Generator(device="cuda").manual_seed(0)
    for waves in (1, 2, 4, 8, 28):
        rows = 148 * per_sm * waves
        buf = torch.randint(0, 1 << 50, (rows, n), device="cuda", dtype=torch.int64, generator=g)
        for name, fn in (("fwd", L.fcn_ntt_forward), ("inv", L.fcn_ntt_inverse)):
            iters = max(4, 400 // waves)
            for _ in range(3):
                _lib.check(fn(h.ring_ptr, buf.data_ptr(), rows, K, 0, st))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                _lib.check(fn(h.ring_ptr, buf.data_ptr(), rows, K, 0, st))
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / iters
            print(f"{wl} n={n} rows={rows} ({rows * n * 8 / 2**20:.0f} MiB, {waves} rows per CTA) {name}: "
                  f"{t * 1e3:.1f} us/launch, {t * 1e3 / waves:.2f} us per wave")
        del buf


if __name__ == "__main__":
    main()
