"""Phase timeline of ntt_f64_fwd (a -DFCN_NTT_PROF build of libfcn):
clock64 deltas of warp 0 of every CTA, summed over rows and CTAs.

usage: python tools/ab_variant.py prof -DFCN_NTT_PROF
       FCN_LIB_PATH=abvar/prof/libfcn.so python tools/ntt_phase_prof.py [workload]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1811_09953_b200 import _lib, configs, fv  # noqa: E402
from paper_1811_09953_b200 import device as dev  # noqa: E402

NAMES = ["load wait + conversions + pass 1 + barrier", "exchange 1 stores + barrier", "pass 2 (loads, butterflies, stores)",
         "exchange 2 barrier", "pass 3 + reduction + staging stores", "next-row loads issued + copy-out"]


INV_NAMES = ["wait for the streamed row + barrier", "loads + pass 1 + stores + barrier", "pass 2 (loads, butterflies, stores)",
             "exchange 2 barrier", "strided loads + next-row copies + pass 3", "twist + reduction + stores"]


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    inv = len(sys.argv) > 2 and sys.argv[2] == "inv"
    W = configs.WORKLOADS[wl]
    P = fv.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    h = P.native()
    K = len(P.limb_primes) + len(h.aux)
    n = P.n
    rows = max(K, (512 << 20) // (n * 8) // K * K)
    g = torch.Generator(device="cuda").manual_seed(0)
    buf = torch.randint(0, 1 << 50, (rows, n), device="cuda", dtype=torch.int64, generator=g)
    L = C.CDLL(os.environ["FCN_LIB_PATH"]) if "FCN_LIB_PATH" in os.environ else _lib.lib()
    lib = _lib.lib()
    fn = lib.fcn_ntt_inverse if inv else lib.fcn_ntt_forward
    names = INV_NAMES if inv else NAMES
    st = dev.stream_ptr()
    out = (C.c_ulonglong * 16)()
    for _ in range(2):
        _lib.check(fn(h.ring_ptr, buf.data_ptr(), rows, K, 0, st))
    torch.cuda.synchronize()
    lib.fcn_ntt_prof_read.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    lib.fcn_ntt_prof_read(out, 1)
    iters = 5
    for _ in range(iters):
        _lib.check(fn(h.ring_ptr, buf.data_ptr(), rows, K, 0, st))
    torch.cuda.synchronize()
    lib.fcn_ntt_prof_read(out, 0)
    tot = sum(out[i] for i in range(6))
    print(f"{wl} {'inverse' if inv else 'forward'} n={n} rows={rows}: {tot / (rows * iters):.0f} clocks per row (warp 0 of each CTA)")
    for i, nm in enumerate(names):
        print(f"  {100 * out[i] / tot:5.1f}%  {out[i] / (rows * iters):8.0f} clk  {nm}")


if __name__ == "__main__":
    main()
