"""Linear-layer kernels at the workloads' shapes: the sparse CUDA-core MAC
(mac_fast_kernel) vs the tensor-core MAC (split_planes + mac_tc_kernel),
timed with CUDA events on random residues (outputs compared bit for bit).

usage: python tools/macbench.py [cfg2|cfg3|cfg4|cfg5 ...]
"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

from paper_1811_09953_b200 import _lib, configs, engine, fv, mac_tc, netplan  # noqa: E402
from paper_1811_09953_b200 import device as dev  # noqa: E402


def timed(fn, iters=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters / 1e3


def layers(wl):
    W = configs.WORKLOADS[wl]
    if wl == "cfg5":
        return [("mac1024", configs.mac_sweep_plan(n_out=4096, n_in=4096, terms=1024, seed=1), 4096)]
    comp = netplan.compile_network(configs.build_network(wl), W.fixed_point())
    out, n_in = [], None
    shapes = {"cfg2": 784, "cfg3": 3072, "cfg4": 2048}
    n_in = shapes[wl]
    for p in comp.plans:
        if type(p).__name__ == "LinearPlan":
            out.append((p.name, p, n_in))
            n_in = len(p.outputs)
    return out


def main():
    wls = sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"]
    res = []
    for wl in wls:
        W = configs.WORKLOADS[wl]
        P = fv.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
        k, n = len(W.primes), W.n
        cols = 2 * k * n
        planes = _lib.lib().fcn_tc_planes(P.native().ptr)
        for name, plan, n_in in layers(wl):
            mac, _, _ = engine._lower_linear(plan, W.t, n, "batched")
            g = torch.Generator(device="cuda").manual_seed(1)
            qs = torch.tensor(list(W.primes), dtype=torch.int64, device="cuda").view(1, 1, k, 1)
            x = (torch.randint(0, 1 << 62, (n_in, 2, k, n), device="cuda", generator=g, dtype=torch.int64) % qs)
            t_sp = timed(lambda: engine._mac_out(P, mac, x, None), iters=1 if wl == "cfg5" else 3)
            want = engine._mac_out(P, mac, x, None)
            tcp = mac_tc.build(mac, n_in, planes, cols, force=True)
            got = torch.empty_like(want)
            t_tc = timed(lambda: mac_tc.run(P, tcp, x, got))
            ok = bool(torch.equal(got, want))
            pl = torch.empty(_lib.lib().fcn_tc_planes_bytes(P.native().ptr, n_in), dtype=torch.uint8, device="cuda")
            t_split = timed(lambda: _lib.check(_lib.lib().fcn_split_planes(P.native().ptr, x.data_ptr(), n_in,
                                                                          pl.data_ptr(), dev.stream_ptr())))
            nnz = mac.n_terms
            r = {"workload": wl, "layer": name, "n_in": n_in, "n_out": mac.n_out, "nnz": nnz, "planes": planes,
                 "groups": tcp.n_groups, "split": tcp.split, "sparse_ms": t_sp * 1e3, "tc_ms": t_tc * 1e3,
                 "split_planes_ms": t_split * 1e3, "est_tc_ms": tcp.est_tc * 1e3, "est_sparse_ms": tcp.est_sparse * 1e3,
                 "bit_identical": ok, "hbm_bytes": (n_in + mac.n_out) * cols * 8,
                 "tc_frac_hbm": (n_in + mac.n_out) * cols * 8 / t_tc / 1e9 / 6547.8}
            print(json.dumps(r), flush=True)
            res.append(r)
            del x, want, got, pl
            torch.cuda.empty_cache()
    return res


if __name__ == "__main__":
    main()
