"""One warm mul_ct_batch (square + relinearisation) at a workload's shape (ncu launch lists).

usage: python tools/profile_mulct.py [workload] [count]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1811_09953_b200 import configs, fv  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    W = configs.WORKLOADS[wl]
    P = fv.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    sk, pk, ek = fv.keygen(P, configs.SEED_KEYS)
    k, n = len(W.primes), W.n
    g = torch.Generator(device="cuda").manual_seed(0)
    qs = torch.tensor(list(W.primes), dtype=torch.int64, device="cuda").view(1, 1, k, 1)
    x = (torch.randint(0, 1 << 62, (B, 2, k, n), device="cuda", generator=g, dtype=torch.int64) % qs).contiguous()
    ws = fv.mul_ct_workspace(P, B)
    out = torch.empty_like(x)
    fv.mul_ct_batch(P, ek, 0, x, None, out=out, workspace=ws)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    fv.mul_ct_batch(P, ek, 0, x, None, out=out, workspace=ws)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("done")


if __name__ == "__main__":
    main()
