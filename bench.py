#!/usr/bin/env python
"""Throughput of the homomorphic evaluation path on B200.

Default workload: BASELINE.json configs[1] ("cfg2"), the MNIST-shaped
Faster-CryptoNets network at N=8192 with 4 RNS limbs and t=65537 batching,
one synthetic image per slot (8,192 images per pass).  A step is one
`engine.eval_encrypted` pass over the encrypted batch.

  value  -- encrypted images/s with the input ciphertexts resident in HBM
  e2e    -- the same through the public API with host (pinned) ciphertext
            buffers: H2D of the inputs and D2H of the outputs inside the
            timed region
  roofline -- the batched NTT kernel (dominant kernel of the path), timed
            live with CUDA events, algorithmic bytes vs measured HBM copy BW
  cpu_baseline -- the CPU oracle port (oracle/) timed on this host on a
            bounded sample, extrapolated with the plan's HOP counts

`--impl reference` times the CPU oracle port (the reference's algorithm
restated in numpy + Python big ints) with all host cores instead.

Multi-GPU (torchrun, one rank per GPU): `--shard outputs` (default) splits
every layer's outputs across ranks (strong scaling of one batch); with
`--transport p2p` (default) each stage's last kernel stores its block into
every rank's buffer over NVLink (symmetric memory, no collective on the data
path), with `--transport nccl` the blocks are all-gathered with NCCL.
`--shard replicas` runs an independent batch per rank (weak scaling, no
collective).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["fcn", "reference"], default="fcn")
    ap.add_argument("--workload", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4"])
    ap.add_argument("--shard", choices=["outputs", "replicas"], default="outputs")
    ap.add_argument("--transport", choices=["p2p", "nccl"], default="p2p")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of one CUDA graph per step")
    ap.add_argument("--force-sharded", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the cpu_baseline sample")
    return ap.parse_args()


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = (
        "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
        "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
        "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
    )

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[4:8]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, fl in rows for i, f in enumerate(fl) if f.lower() == "active"})
        sm = sorted(r[0] for r in rows)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons, "samples": len(rows)}


def _peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _fp64_peak():
    p = os.path.join(REPO, "profiles", "fp64_peak.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f)


def _int_peak():
    p = os.path.join(REPO, "profiles", "int_peak.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f)


def _config(W, workload, ws, shard, hops=None, l2=None):
    cfg = {
        "workload": workload,
        "n": W.n,
        "limbs": len(W.primes),
        "t": W.t,
        "slots": W.slots,
        "encoding": "batched",
        "parallelism": f"{shard}{ws}" if ws > 1 else "single",
    }
    if hops is not None:
        cfg["hops"] = {"pt_ct_mul": hops.pt_ct_mul, "ct_ct_add": hops.ct_ct_add, "ct_ct_mul": hops.ct_ct_mul,
                       "pt_ct_add": hops.pt_ct_add}
    if l2 is not None:
        cfg["l2"] = l2
    return cfg


def _profile_traffic(name: str):
    """dram bytes per launch of a kernel from the committed ncu summary."""
    p = os.path.join(REPO, "profiles", "kernel_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f).get(name)


# ------------------------------------------------------------------ setup


def _setup(workload: str, seed_offset: int = 0):
    import torch

    from paper_1811_09953_b200 import configs, engine, fv

    W = configs.WORKLOADS[workload]
    P = fv.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    sk, pk, ek = fv.keygen(P, configs.SEED_KEYS)
    net = configs.build_network(workload)
    cfg = W.fixed_point()
    x = configs.build_inputs(workload)
    tensor = engine.encrypt_tensor_batched(pk, P, x, cfg, 0, configs.SEED_ENC + seed_offset)
    torch.cuda.synchronize()
    return W, P, sk, pk, ek, net, cfg, x, tensor


def _ntt_roofline(P, iters: int = 20):
    """Average duration of the batched NTT kernel over > L2 of rows."""
    import torch

    from paper_1811_09953_b200 import _lib
    from paper_1811_09953_b200 import device as dev

    h = P.native()
    K = len(P.limb_primes) + len(h.aux)
    n = P.n
    rows = max(K, (512 << 20) // (n * 8) // K * K)  # ~512 MB of rows: > L2
    g = torch.Generator(device="cuda").manual_seed(0)
    buf = torch.randint(0, 1 << 50, (rows, n), device="cuda", dtype=torch.int64, generator=g)
    st = dev.stream_ptr()
    L = _lib.lib()
    for _ in range(3):
        _lib.check(L.fcn_ntt_forward(h.ring_ptr, buf.data_ptr(), rows, K, 0, st))
        _lib.check(L.fcn_ntt_inverse(h.ring_ptr, buf.data_ptr(), rows, K, 0, st))
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    for _ in range(iters):
        _lib.check(L.fcn_ntt_forward(h.ring_ptr, buf.data_ptr(), rows, K, 0, st))
    e1.record()
    for _ in range(iters):
        _lib.check(L.fcn_ntt_inverse(h.ring_ptr, buf.data_ptr(), rows, K, 0, st))
    e2.record()
    torch.cuda.synchronize()
    t_f = e0.elapsed_time(e1) / iters / 1e3
    t_i = e1.elapsed_time(e2) / iters / 1e3
    bytes_per_launch = 2 * rows * n * 8
    return {"rows": rows, "n": n, "bytes": bytes_per_launch, "t_fwd_s": t_f, "t_inv_s": t_i}


def _keyswitch_roofline(P, ek, count: int = 256, iters: int = 20):
    """Average duration of the key-switching inner product (fcn_key_mac) over
    `count` ciphertexts of NTT-domain digits (> L2): bytes = digits read +
    accumulators written (keys excluded, SURVEY 8(d) convention)."""
    import torch

    from paper_1811_09953_b200 import _lib
    from paper_1811_09953_b200 import device as dev

    h = P.native()
    kh = ek.native(P)
    k, n, D = len(P.limb_primes), P.n, P.ell + 1
    g = torch.Generator(device="cuda").manual_seed(1)
    dig = torch.randint(0, 1 << 50, (count, D, k, n), device="cuda", dtype=torch.int64, generator=g)
    acc = torch.empty((count, 2, k, n), device="cuda", dtype=torch.int64)
    st = dev.stream_ptr()
    L = _lib.lib()
    for _ in range(3):
        _lib.check(L.fcn_key_mac(h.ptr, kh.ptr, dig.data_ptr(), acc.data_ptr(), count, st))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        _lib.check(L.fcn_key_mac(h.ptr, kh.ptr, dig.data_ptr(), acc.data_ptr(), count, st))
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / iters / 1e3
    return {"count": count, "digits": D, "bytes": count * (D * k + 2 * k) * n * 8, "t_s": t}


# ----------------------------------------------------------------- CPU leg


def _cpu_sample(workload: str, seconds: float, hops_tot, slots: int):
    """Oracle (numpy + big-int) per-op times at the workload's ring shape on a
    bounded sample, extrapolated by the plan's HOP counts to one pass."""
    from oracle import bfv as ob
    from oracle import rns as orn
    from paper_1811_09953_b200 import configs

    W = configs.WORKLOADS[workload]
    OP = ob.Params(W.n, W.primes, (W.t,), W.beta)
    K = ob.keygen(OP, configs.SEED_KEYS)
    rng = np.random.default_rng(11)
    cts = [ob.Ct(orn.random_uniform(W.primes, W.n, rng), orn.random_uniform(W.primes, W.n, rng)) for _ in range(4)]
    t_end = time.perf_counter() + seconds * 0.7
    n_mul, t0 = 0, time.perf_counter()
    while n_mul < 2 or (time.perf_counter() < t_end and n_mul < 64):
        ob.mul_ct(OP, cts[n_mul % 4], cts[n_mul % 4], K)
        n_mul += 1
    t_mul = (time.perf_counter() - t0) / n_mul
    t_end = time.perf_counter() + seconds * 0.3
    n_pt, t0 = 0, time.perf_counter()
    acc = cts[0]
    while n_pt < 8 or (time.perf_counter() < t_end and n_pt < 4096):
        term = ob.mul_pt(OP, cts[n_pt % 4], [8], 0)
        acc = ob.add_ct(OP, acc, term)
        n_pt += 1
    t_pair = (time.perf_counter() - t0) / n_pt
    # add_pt at most once per output; cost ~ one add (bounded by the pair time)
    t_pass = hops_tot.ct_ct_mul * t_mul + hops_tot.pt_ct_mul * t_pair + hops_tot.pt_ct_add * t_pair
    sample = f"{n_mul} mul_ct + {n_pt} (mul_pt+add_ct) at n={W.n}, k={len(W.primes)}; extrapolated by HOP counts"
    return slots / t_pass, t_pass, sample, {"t_mul_ct_s": t_mul, "t_mulpt_addct_s": t_pair}


def _ref_worker(job):
    kind, workload, count = job
    from oracle import bfv as ob
    from oracle import rns as orn
    from paper_1811_09953_b200 import configs

    st = _ref_worker.state
    OP, K, cts = st
    t0 = time.perf_counter()
    if kind == "mul":
        for i in range(count):
            ob.mul_ct(OP, cts[i % len(cts)], cts[i % len(cts)], K)
    else:
        acc = cts[0]
        for i in range(count):
            acc = ob.add_ct(OP, acc, ob.mul_pt(OP, cts[i % len(cts)], [8], 0))
    return time.perf_counter() - t0


def _ref_init(workload):
    from oracle import bfv as ob
    from oracle import rns as orn
    from paper_1811_09953_b200 import configs

    W = configs.WORKLOADS[workload]
    OP = ob.Params(W.n, W.primes, (W.t,), W.beta)
    K = ob.keygen(OP, configs.SEED_KEYS)
    rng = np.random.default_rng(11 + os.getpid() % 7)
    cts = [ob.Ct(orn.random_uniform(W.primes, W.n, rng), orn.random_uniform(W.primes, W.n, rng)) for _ in range(2)]
    _ref_worker.state = (OP, K, cts)


def _host_cpu() -> dict:
    """The host the CPU numbers ran on (count, physical cores, model)."""
    info = {"os_cpu_count": os.cpu_count()}
    try:
        import psutil

        info["physical_cores"] = psutil.cpu_count(logical=False)
    except Exception:  # noqa: BLE001 - optional
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["model"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return info


def run_reference(args, ws, rank):
    """CPU oracle port on all host cores (multiprocessing over independent outputs)."""
    if rank != 0:
        return
    import multiprocessing as mp

    from paper_1811_09953_b200 import configs, netplan

    W = configs.WORKLOADS[args.workload]
    comp = netplan.compile_network(configs.build_network(args.workload), W.fixed_point())
    tot = netplan.plan_hops(comp, "batched", W.t).totals
    cores = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_ref_init, initargs=(args.workload,)) as pool:
        def step():
            t0 = time.perf_counter()
            pool.map(_ref_worker, [("mul", args.workload, 1)] * cores)
            t_mul = time.perf_counter() - t0
            t0 = time.perf_counter()
            pool.map(_ref_worker, [("pt", args.workload, 16)] * cores)
            t_pt = time.perf_counter() - t0
            # cores ops in t_mul; 16*cores pairs in t_pt
            return tot.ct_ct_mul * t_mul / cores + (tot.pt_ct_mul + tot.pt_ct_add) * t_pt / (16 * cores)

        for _ in range(args.warmup):
            step()
        t0 = time.perf_counter()
        passes = [step() for _ in range(args.steps)]
        wall = time.perf_counter() - t0
    t_pass = float(np.mean(passes))
    value = W.slots / t_pass
    line = {
        "impl": "reference",
        "metric": "encrypted images/sec",
        "value": value,
        "unit": "images/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": wall / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic (seeded uniform ciphertexts at the workload's ring shape)",
        "config": _config(W, args.workload, ws, args.shard, tot,
                          "inputs larger than L2 (%d MB of input ciphertexts per step)" % (784 * 2 * len(W.primes) * W.n * 8 >> 20)
                          if args.workload in ("cfg1", "cfg2") else None),
        "cpu_baseline": {
            "value": value,
            "unit": "images/s",
            "cores": cores,
            "kind": "port",
            "host": _host_cpu(),
            "sample": f"per step: {cores} mul_ct + {16 * cores} (mul_pt+add_ct) across a {cores}-process pool; "
            f"pass time extrapolated by the plan's HOP counts ({tot.ct_ct_mul} ct_ct_mul, {tot.pt_ct_mul} pt_ct_mul)",
        },
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg


def run_gpu(args, ws, rank, local):
    import torch
    import torch.distributed as dist

    from paper_1811_09953_b200 import _lib, engine

    torch.cuda.set_device(local)
    _lib.load()
    W, P, sk, pk, ek, net, cfg, x, tensor = _setup(args.workload, seed_offset=rank if args.shard == "replicas" else 0)
    comp = engine.compile_network(net, cfg)
    plan = comp  # evaluations take the compiled plan (no per-call content hash of the weights)
    # --force-sharded: the sharded code path at world size 1 (checks the
    # multi-GPU plumbing -- pre-flight, transports, timing -- on one GPU)
    sharded = (ws > 1 or args.force_sharded) and args.shard == "outputs"
    if sharded:
        from paper_1811_09953_b200 import dist as fdist

        transport = args.transport
        if transport == "p2p":
            # pre-flight: every rank must be able to map the symmetric buffers
            # and produce the same bytes as the NCCL all-gather schedule
            ok = 1
            try:
                got = fdist.eval_encrypted_sharded(plan, tensor, ek, cfg, encoding="batched", transport="p2p")[0]
                want = fdist.eval_encrypted_sharded(plan, tensor, ek, cfg, encoding="batched", transport="nccl")[0]
                if not torch.equal(got.buf, want.buf):
                    ok = 0
                    args.transport_note = "p2p result differs from the NCCL schedule"
            except Exception as exc:  # noqa: BLE001 - reported in config
                ok = 0
                args.transport_note = f"p2p unavailable ({type(exc).__name__}: {exc})"[:200]
            flag = torch.tensor([ok], device="cuda", dtype=torch.int32)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 0:
                transport = "nccl"
        args.transport_used = transport
        evaluate = lambda t: fdist.eval_encrypted_sharded(plan, t, ek, cfg, encoding="batched",  # noqa: E731
                                                          transport=transport)[0]
    else:
        evaluate = lambda t: engine.eval_encrypted(plan, t, ek, cfg, encoding="batched")[0]  # noqa: E731
        if not args.no_graph:
            # the whole network as one CUDA graph over the resident input buffer
            try:
                g = engine.EvalGraph(plan, tensor, ek, cfg, encoding="batched")
                ref = evaluate(tensor)
                if torch.equal(g.replay().buf, ref.buf):
                    evaluate = lambda t: g.replay() if t is tensor else engine.eval_encrypted(  # noqa: E731
                        plan, t, ek, cfg, encoding="batched")[0]
                    args.graph_used = True
                    args.graph_kernels = g.kernels
                else:
                    args.graph_note = "graph replay differs from eager evaluation"
            except Exception as exc:  # noqa: BLE001 - reported in config
                args.graph_note = f"graph capture failed ({type(exc).__name__}: {exc})"[:200]

    def barrier():
        if ws > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        out = evaluate(tensor)
    torch.cuda.synchronize()
    barrier()
    L = _lib.lib()
    n0 = L.fcn_launch_count()
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            out = evaluate(tensor)
        e1.record()
        torch.cuda.synchronize()
        barrier()
    launches = (L.fcn_launch_count() - n0) // args.steps
    if getattr(args, "graph_used", False):
        launches = args.graph_kernels  # replays launch the captured kernels, not through the host counter
    t_step = e0.elapsed_time(e1) / 1e3 / args.steps
    if ws > 1:
        tt = torch.tensor([t_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
    images = W.slots * (ws if args.shard == "replicas" else 1)
    value = images / t_step

    check = None

    # e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # public streaming API: pinned host batches in, host results out; each step's
        # H2D (double-buffered on a copy stream) and D2H are inside the timed loop
        host_in = [tensor.buf.cpu().pin_memory() for _ in range(2)]
        h2d = host_in[0].numel() * 8
        d2h = 0
        if sharded:
            from paper_1811_09953_b200 import dist as fdist

            n_in = tensor.buf.shape[0]
            parts = fdist.partition(n_in, ws)
            lo, hi = parts[rank]
            block = parts[0][1] - parts[0][0]
            copy = torch.cuda.Stream()

            def stream(batches):
                # each rank uploads its 1/world of batch i+1 on a copy stream
                # while batch i computes; an NVLink all-gather assembles it
                # (dist.upload_sharded, split in two for the overlap)
                def up(hb):
                    with torch.cuda.stream(copy):
                        loc = hb[lo:hi].to("cuda", non_blocking=True)
                        ev = torch.cuda.Event()
                        ev.record(copy)
                    return loc, ev

                it = iter(batches)
                hb = next(it, None)
                nxt = up(hb) if hb is not None else None
                while nxt is not None:
                    loc, ev = nxt
                    torch.cuda.current_stream().wait_event(ev)
                    loc.record_stream(torch.cuda.current_stream())
                    hb = next(it, None)
                    nxt = up(hb) if hb is not None else None
                    full = fdist._torch_gather(loc, n_in, block)
                    t_in = engine.CipherTensor(tensor.shape, scale_exponent=tensor.scale_exponent, buf=full, params=P,
                                               lane=0)
                    yield evaluate(t_in).buf.to("cpu")
        else:
            # result ring allocated once, like a server would (pinned allocation is slow)
            out_shape = (int(np.prod(comp.out_shape)), 2, len(P.limb_primes), P.n)
            ring = [torch.empty(out_shape, dtype=torch.int64, pin_memory=True) for _ in range(3)]

            def stream(batches):
                return engine.evaluate_stream(plan, batches, ek, cfg, P, tensor.shape, tensor.scale_exponent,
                                              host_out=ring)
        for _ in stream(host_in[i % 2] for i in range(2)):
            pass
        barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # at least 20 batches so the pipeline fill (one upload not overlapped
        # with compute) is amortised as in a serving loop
        n_e2e = max(args.steps, 20)
        s0.record()
        for res in stream(host_in[i % 2] for i in range(n_e2e)):
            d2h = res.numel() * 8
        s1.record()
        torch.cuda.synchronize()
        barrier()
        t_e2e = s0.elapsed_time(s1) / 1e3 / n_e2e
        if ws > 1:
            tt = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        e2e = {"value": images / t_e2e, "unit": "images/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": t_e2e * 1e3, "batches": n_e2e,
               "api": "engine.evaluate_stream (pinned host batches in, host result bodies out)" if not sharded else
               "dist.upload_sharded (each rank uploads 1/world of the pinned batch, NVLink all-gather) + "
               "dist.eval_encrypted_sharded + host result bodies out"}

    if rank != 0:
        return
    peak, peak_kind = _peaks()
    r = _ntt_roofline(P)
    t_avg = (r["t_fwd_s"] + r["t_inv_s"]) / 2
    achieved = r["bytes"] / t_avg / 1e9
    tr = _profile_traffic(f"ntt_{args.workload}")
    fp = _fp64_peak()
    bfly = r["rows"] * (r["n"] // 2) * (r["n"].bit_length() - 1)
    fp_roof = None
    if fp:
        ach = bfly / t_avg
        # the reduction schedule the launch used (one reduction per transform for limbs just above 2^50)
        from paper_1811_09953_b200 import _lib

        h = P.native()
        qmax = max(tuple(P.limb_primes) + tuple(h.aux))
        rs = _lib.load().fcn_ntt_f64_schedule(int(r["n"]).bit_length() - 1, qmax)
        pk = fp.get("butterfly_rs1_per_s", fp["butterfly_per_s"]) if rs >= 1 else fp["butterfly_per_s"]
        fp_roof = {"achieved_butterflies_per_s": ach, "peak_butterflies_per_s": pk, "frac": ach / pk,
                   "schedule": rs, "ceiling_frac_of_hbm": pk * r["bytes"] / bfly / 1e9 / peak,
                   "peak_source": "profiles/fp64_peak.json (measured register-resident FP64 butterfly with the "
                                  "launch's reduction schedule, tools/fp64bench.cu)"}
    roofline = {
        "kernel": "ntt_f64_fwd / ntt_f64_inv (batched negacyclic NTT on the FP64 pipe, one CTA per row slot)",
        "bound": "hbm",
        "achieved": achieved,
        "peak": peak,
        "peak_kind": peak_kind,
        "unit": "GB/s",
        "frac": achieved / peak,
        "traffic": tr,
        "algorithmic_bytes_per_launch": r["bytes"],
        "rows_per_launch": r["rows"],
        "ms_fwd": r["t_fwd_s"] * 1e3,
        "ms_inv": r["t_inv_s"] * 1e3,
        "fp64_roofline": fp_roof,
        "note": "the NTT is FP64-pipe bound on B200 (one exact signed modmul = 5 DP ops + FRND per butterfly): "
                "fp64_roofline.ceiling_frac_of_hbm is the register-resident butterfly ceiling as a fraction of HBM",
    }
    ks = _keyswitch_roofline(P, ek)
    ks_ach = ks["bytes"] / ks["t_s"] / 1e9
    keyswitch = {
        "kernel": "keymac_f64_kernel (fcn_key_mac: sum_d key_d * digit_d, NTT domain)",
        "bound": "hbm",
        "achieved": ks_ach,
        "peak": peak,
        "unit": "GB/s",
        "frac": ks_ach / peak,
        "algorithmic_bytes_per_launch": ks["bytes"],
        "ciphertexts_per_launch": ks["count"],
        "digits": ks["digits"],
        "ms": ks["t_s"] * 1e3,
    }
    hops = engine.plan_hops(comp, "batched", W.t).totals
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        # cpu_baseline leg: the oracle also checks the decrypted timed output
        from oracle import drivers as od

        slots = engine.decrypt_tensor_slots(sk, out)
        check = bool(np.array_equal(slots, od.plain_model_batched(comp, x << cfg.precision_bits, W.t)))
        v, t_pass, sample, per = _cpu_sample(args.workload, args.cpu_seconds, hops, W.slots)
        cpu = {"value": v, "unit": "images/s", "cores": 1, "kind": "port", "sample": sample, "seconds_per_pass": t_pass,
               "host": _host_cpu(), **per}
    line = {
        "metric": "encrypted images/sec",
        "value": value,
        "unit": "images/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": t_step * 1e3,
        "higher_is_better": True,
        "scaling": "weak" if (ws == 1 or args.shard == "replicas") else "strong",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic (seeded uint8 images, one per slot; random-init pruned pow2 weights)",
        "config": dict(_config(W, args.workload, ws, args.shard, hops,
                               "inputs larger than L2 (%d MB of input ciphertexts per step)" % (tensor.buf.numel() * 8 >> 20)),
                       cuda_graph=bool(getattr(args, "graph_used", False)),
                       **({"graph_note": args.graph_note} if getattr(args, "graph_note", None) else {}),
                       **({"transport": getattr(args, "transport_used", args.transport)} if sharded else {}),
                       **({"transport_note": args.transport_note} if getattr(args, "transport_note", None) else {})),
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "decrypt_check": check,
        "roofline": roofline,
        "keyswitch_roofline": keyswitch,
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    print(json.dumps(line), flush=True)


def main():
    args = _args()
    ws, rank, local = _dist()
    group = ws > 1 or (args.force_sharded and args.impl != "reference")
    if group:
        import torch
        import torch.distributed as dist

        backend = "gloo" if args.impl == "reference" else "nccl"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_gpu(args, ws, rank, local)
    if group:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
