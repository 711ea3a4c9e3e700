import torch, time
x = torch.empty(411*1024*1024//8, dtype=torch.int64).pin_memory()
d = torch.empty_like(x, device='cuda')
for _ in range(3): d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): d.copy_(x, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms=e0.elapsed_time(e1)/10
print("H2D one stream: %.2f ms per 411MB = %.1f GB/s" % (ms, 411*1.048576/ms))
# two streams, halves
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
h=x.numel()//2
torch.cuda.synchronize()
t0=time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): d[:h].copy_(x[:h], non_blocking=True)
    with torch.cuda.stream(s2): d[h:].copy_(x[h:], non_blocking=True)
torch.cuda.synchronize()
ms=(time.perf_counter()-t0)*1e3/10
print("H2D two streams: %.2f ms = %.1f GB/s" % (ms, 411*1.048576/ms))
y = torch.empty(5*1024*1024//8, dtype=torch.int64).pin_memory()
dd = torch.empty_like(y, device='cuda')
e0.record()
for _ in range(10): y.copy_(dd, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("D2H 5MB: %.3f ms" % (e0.elapsed_time(e1)/10))
