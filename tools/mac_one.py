"""Run one linear layer of a workload on the tensor-core MAC (for ncu captures).

usage: python tools/mac_one.py cfg5 [layer-index]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import macbench  # noqa: E402  (tools/ on sys.path when run as a script)
from paper_1811_09953_b200 import _lib, configs, engine, fv, mac_tc  # noqa: E402


def main():
    wl = sys.argv[1]
    idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    W = configs.WORKLOADS[wl]
    P = fv.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    k, n = len(W.primes), W.n
    name, plan, n_in = macbench.layers(wl)[idx]
    mac, _, _ = engine._lower_linear(plan, W.t, n, "batched")
    qs = torch.tensor(list(W.primes), dtype=torch.int64, device="cuda").view(1, 1, k, 1)
    x = (torch.randint(0, 1 << 62, (n_in, 2, k, n), device="cuda", dtype=torch.int64) % qs)
    tcp = mac_tc.build(mac, n_in, _lib.lib().fcn_tc_planes(P.native().ptr), 2 * k * n, force=True)
    out = torch.empty((mac.n_out, 2, k, n), dtype=torch.int64, device="cuda")
    for _ in range(2):
        mac_tc.run(P, tcp, x, out)
    torch.cuda.synchronize()
    print(name, "done")


if __name__ == "__main__":
    main()
