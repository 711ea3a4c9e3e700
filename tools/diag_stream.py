import sys, time, os
sys.path.insert(0, '/root/repo')
import torch, bench
from paper_1811_09953_b200 import engine
W, P, sk, pk, ek, net, cfg, x, tensor = bench._setup('cfg2')
host = [tensor.buf.cpu().pin_memory() for _ in range(2)]
print('pinned', host[0].is_pinned())
def t(fn, n=5):
    torch.cuda.synchronize(); s=time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter()-s)/n*1e3
print('h2d', t(lambda: host[0].to('cuda', non_blocking=True)))
copy = torch.cuda.Stream()
def h2d_side():
    with torch.cuda.stream(copy):
        d = host[0].to('cuda', non_blocking=True)
    copy.synchronize()
print('h2d side stream', t(h2d_side))
print('eval', t(lambda: engine.eval_encrypted(net, tensor, ek, cfg, encoding='batched')))
def both():
    with torch.cuda.stream(copy):
        d = host[0].to('cuda', non_blocking=True)
    engine.eval_encrypted(net, tensor, ek, cfg, encoding='batched')
    copy.synchronize()
print('eval+concurrent h2d', t(both))
def stream():
    for _ in engine.evaluate_stream(net, (host[i%2] for i in range(5)), ek, cfg, P, tensor.shape, tensor.scale_exponent): pass
print('stream x5 per step', t(stream, 1)/5)
