"""Run one warm evaluation step of a workload (for ncu launch lists / captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_09953_b200 import engine  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    W, P, sk, pk, ek, net, cfg, x, tensor = bench._setup(wl)
    engine.eval_encrypted(net, tensor, ek, cfg, encoding="batched")
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(steps):
        engine.eval_encrypted(net, tensor, ek, cfg, encoding="batched")
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("done")


if __name__ == "__main__":
    main()
