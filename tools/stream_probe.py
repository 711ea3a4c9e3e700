"""Where does evaluate_stream spend host time per batch? (diagnostic)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_09953_b200 import engine  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
W, P, sk, pk, ek, net, cfg, x, tensor = bench._setup(wl)
hb = [tensor.buf.cpu().pin_memory() for _ in range(2)]
N = 12
stamps = []
t_prev = time.perf_counter()
gen = engine.evaluate_stream(net, (hb[i % 2] for i in range(N)), ek, cfg, P, tensor.shape, tensor.scale_exponent)
for r in gen:
    t = time.perf_counter()
    stamps.append(1e3 * (t - t_prev))
    t_prev = t
print(wl, "per-yield ms:", [round(s, 2) for s in stamps])
torch.cuda.synchronize()
# eval only, with a fresh device input each time (upload on the same stream)
d = torch.empty_like(tensor.buf)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(N):
    d.copy_(hb[i % 2], non_blocking=True)
    out, _ = engine.eval_encrypted(net, engine.CipherTensor(tensor.shape, scale_exponent=tensor.scale_exponent, buf=d,
                                                             params=P, lane=0), ek, cfg, encoding="batched")
torch.cuda.synchronize()
print(wl, "serial upload+eval ms/batch:", round(1e3 * (time.perf_counter() - t0) / N, 2))
