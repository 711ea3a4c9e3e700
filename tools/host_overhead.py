"""Host (Python + ctypes) time per eval_encrypted call vs GPU time, per workload."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_09953_b200 import engine  # noqa: E402

for wl in sys.argv[1:] or ["cfg1", "cfg2"]:
    W, P, sk, pk, ek, net, cfg, x, tensor = bench._setup(wl)
    for _ in range(3):
        engine.eval_encrypted(net, tensor, ek, cfg, encoding="batched")
    torch.cuda.synchronize()
    N = 10
    t0 = time.perf_counter()
    for _ in range(N):
        engine.eval_encrypted(net, tensor, ek, cfg, encoding="batched")
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{wl}: host enqueue {1e3 * (t1 - t0) / N:.2f} ms/call, wall incl. GPU {1e3 * (t2 - t0) / N:.2f} ms/call")
    hb = [tensor.buf.cpu().pin_memory() for _ in range(2)]
    t0 = time.perf_counter()
    for _ in engine.evaluate_stream(net, (hb[i % 2] for i in range(N)), ek, cfg, P, tensor.shape, tensor.scale_exponent):
        pass
    t1 = time.perf_counter()
    print(f"{wl}: evaluate_stream {1e3 * (t1 - t0) / N:.2f} ms/batch over {N} batches")

# pieces of the streaming loop (last workload)
N = 10
t0 = time.perf_counter()
for _ in range(N):
    r = torch.empty(tensor.buf.shape, dtype=torch.int64, pin_memory=True)
t1 = time.perf_counter()
print(f"pinned alloc of a result-sized buffer: {1e3 * (t1 - t0) / N:.3f} ms")
copy = torch.cuda.Stream()
d = torch.empty(hb[0].shape, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(N):
    with torch.cuda.stream(copy):
        d.copy_(hb[i % 2], non_blocking=True)
copy.synchronize()
t1 = time.perf_counter()
print(f"H2D on copy stream: {1e3 * (t1 - t0) / N:.2f} ms per batch ({hb[0].numel() * 8 / 1e6:.0f} MB)")
