"""cProfile of the host side of eager eval_encrypted calls (where the Python
time per layer goes).  usage: python tools/host_profile.py [workload] [calls]"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_09953_b200 import engine  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
W, P, sk, pk, ek, net, cfg, x, tensor = bench._setup(wl)
for _ in range(3):
    engine.eval_encrypted(net, tensor, ek, cfg, encoding="batched")
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    engine.eval_encrypted(net, tensor, ek, cfg, encoding="batched")
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
