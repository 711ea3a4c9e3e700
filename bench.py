#!/usr/bin/env python
"""Throughput of the homomorphic evaluation path on B200.

Default workload: BASELINE.json configs[2] ("cfg3"), the largest network
configuration (CIFAR-shaped, N=16384, 6 RNS limbs, t=65537 batching, one
synthetic image per slot: 16,384 images per pass); `--workload` selects
cfg1/cfg2/cfg4 (the other network configs) or cfg5 (the primitive sweep:
NTT fwd+inv, square + relinearisation with dnum=3 keys, the 1024-term sparse
pow2 MAC over 4,096 ciphertexts).  A step is one `engine.eval_encrypted`
pass over the encrypted batch (cfg5: one pass of the three primitives).

  value  -- encrypted images/s with the input ciphertexts resident in HBM
  e2e    -- the same through the public API with host (pinned) ciphertext
            buffers: H2D of the inputs and D2H of the outputs inside the
            timed region
  roofline -- the batched NTT kernel (dominant kernel of the path), timed
            live with CUDA events, algorithmic bytes vs measured HBM copy BW
  keyswitch_roofline -- relinearisation (digit NTT + key MAC + INTT with
            the add) with SURVEY 8(d)'s bytes 2.5 B P + keys, and square +
            relinearisation end to end with 2 B P + keys
  cpu_baseline -- the reference package itself (baseline/_ref, `hecnet`)
            on one host core, on a bounded sample extrapolated with the
            plan's HOP counts (refarm.py)

`--impl reference` runs the reference (`hecnet` from baseline/_ref) on all
host cores: a fork pool over each layer's independent outputs (the value),
plus its as-shipped one-core loop and its own ThreadPool (refarm.py).

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
    ap.add_argument("--workload", default="cfg3", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--shard", choices=["outputs", "replicas"], default="outputs")
    ap.add_argument("--transport", choices=["p2p", "nccl"], default="p2p")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of one CUDA graph per step")
    ap.add_argument("--force-sharded", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="budget of the cpu_baseline sample")
    ap.add_argument("--ref-mode-seconds", type=float, default=12.0,
                    help="budget of each of the reference arm's one-core and ThreadPool samples")
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
                rows.append((float(parts[0]), float(parts[1]), parts[4:8], float(parts[2])))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, f in enumerate(r[2]) if f.lower() == "active"})
        sm = sorted(r[0] for r in rows)
        pw = sorted(r[3] for r in rows)
        # power: the FP64 step runs at the board's limit, which is what sw_power_cap reports
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons, "samples": len(rows),
                "power_w": pw[len(pw) // 2], "power_w_max": pw[-1]}


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
    accumulators written (keys excluded).  A sub-kernel figure."""
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
    del dig, acc
    return {"count": count, "digits": D, "bytes": count * (D * k + 2 * k) * n * 8, "t_s": t}


STAGES = ("lift", "forward_ntt_tensor", "tensor_intt", "rescale_digits", "digit_ntt", "key_mac", "final_intt_add")


def _square_relin_stages(P, ek, count: int, iters: int = 3, act=(8, 131072)):
    """Squares + relinearisation of `count` random ciphertexts (fcn_mul_ct_ex,
    the activation epilogue of the workloads) with per-stage CUDA events
    (fcn_stage_timing), averaged over `iters` calls after a warm-up."""
    import ctypes as C

    import torch

    from paper_1811_09953_b200 import _lib, fv

    k, n = len(P.limb_primes), P.n
    g = torch.Generator(device="cuda").manual_seed(2)
    hi = min(P.limb_primes)
    x = torch.randint(0, hi, (count, 2, k, n), device="cuda", dtype=torch.int64, generator=g)
    out = torch.empty_like(x)
    L = _lib.lib()
    ws = fv.mul_ct_workspace(P, count)
    fv.mul_ct_batch(P, ek, 0, x, out=out, workspace=ws, act=act)
    torch.cuda.synchronize()
    L.fcn_stage_timing(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fv.mul_ct_batch(P, ek, 0, x, out=out, workspace=ws, act=act)
    e1.record()
    torch.cuda.synchronize()
    ms = (C.c_double * len(STAGES))()
    _lib.check(L.fcn_stage_times(ms, len(STAGES)))
    L.fcn_stage_timing(0)
    total = e0.elapsed_time(e1) / iters / 1e3
    stages = {name: ms[i] / iters / 1e3 for i, name in enumerate(STAGES)}
    del x, out, ws
    torch.cuda.empty_cache()
    return total, stages


def _keyswitch_objects(P, ek, peak, count: int):
    """relinearisation bytes 2.5 B P + 2 dnum k n 8 over the digit
    NTT + key MAC + INTT-with-add chain; square + relin 2 B P + keys over the
    whole fcn_mul_ct_ex call.  Both chains are FP64-pipe bound,
    so the fractions relate the in/out/key bytes to the time."""
    k, n, D = len(P.limb_primes), P.n, P.ell + 1
    Pb = 2 * k * n * 8
    keys = 2 * D * k * n * 8
    total, st = _square_relin_stages(P, ek, count)
    t_ks = st["digit_ntt"] + st["key_mac"] + st["final_intt_add"]
    ks_bytes = 2.5 * count * Pb + keys
    sq_bytes = 2.0 * count * Pb + keys
    import ctypes as C

    from paper_1811_09953_b200 import _lib

    pv = C.c_int64()
    _lib.check(_lib.lib().fcn_ctx_query(P.native().ptr, 7, C.byref(pv)))
    pair = bool(pv.value)
    keyswitch = {
        "kernel": ("relinearisation chain, shared prime pair: ntt_f64_fwd (digits under q_0, q_1) + "
                   "keymac_pair_f64_kernel + ntt_f64_inv_epi (limbs 0, 1) + ntt_f64_inv_pair (two-residue CRT)") if pair
        else "relinearisation chain: ntt_f64_fwd (digits) + keymac_f64_kernel + ntt_f64_inv_epi",
        "shared_pair": pair,
        "transformed_rows_per_ciphertext": (2 * D + 4 * k - 4) if pair else k * (D + 2),
        "bound": "hbm",
        "achieved": ks_bytes / t_ks / 1e9,
        "peak": peak,
        "unit": "GB/s",
        "frac": ks_bytes / t_ks / 1e9 / peak,
        "algorithmic_bytes": ks_bytes,
        "formula": "2.5 B P + 2 dnum k n 8 (SURVEY 8(d))",
        "ciphertexts": count,
        "digits": D,
        "ms": t_ks * 1e3,
    }
    square = {
        "kernel": "square + relinearisation end to end (fcn_mul_ct_ex with the activation epilogue)",
        "achieved": sq_bytes / total / 1e9,
        "peak": peak,
        "unit": "GB/s",
        "frac": sq_bytes / total / 1e9 / peak,
        "algorithmic_bytes": sq_bytes,
        "formula": "2 B P + keys (SURVEY 8(d))",
        "ciphertexts": count,
        "ms": total * 1e3,
        "ciphertexts_per_s": count / total,
        "stage_ms": {name: v * 1e3 for name, v in st.items()},
    }
    return keyswitch, square


# ----------------------------------------------------------------- CPU leg


def run_reference(args, ws, rank):
    """The reference package on this host's cores (refarm.py): the value is
    mode (c), a fork pool over each layer's independent outputs; modes (a)
    one core as shipped and (b) the shipped ThreadPool are reported beside it."""
    if rank != 0:
        return
    import refarm

    if args.workload == "cfg5":
        print(json.dumps({"impl": "reference", "unavailable": "cfg5 is a primitive sweep with no network pass; "
                          "the reference arm times the network workloads cfg1-cfg4"}), flush=True)
        return
    cores = os.cpu_count() or 1
    st = refarm.RefState(args.workload)
    pool = refarm.ProcessPool(st, cores)
    try:
        for _ in range(args.warmup):
            pool.step()
        t0 = time.perf_counter()
        steps = [pool.step() for _ in range(args.steps)]
        wall = time.perf_counter() - t0
    finally:
        pool.close()
    t_pass = float(np.mean([r["seconds_per_pass"] for r in steps]))
    value = st.W.slots / t_pass
    seq = refarm.sequential(st, args.ref_mode_seconds)
    thr = refarm.threadpool(st, cores, args.ref_mode_seconds, seq["t_act_output_s"])
    tot = st.hop_totals()
    sample = (f"per step: {cores} activation outputs (mul_ct + mul_pt + mul_pt + add_ct) and {cores} x 32 linear taps "
              f"(mul_pt + add_ct) over a {cores}-process fork pool, pass time extrapolated by the plan's HOP structure "
              f"({tot.ct_ct_mul} ct_ct_mul, {tot.pt_ct_mul} pt_ct_mul)")
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
        "data": "synthetic (seeded uint8 images encrypted by the reference's own fv.encrypt; reference keygen)",
        "config": _config(st.W, args.workload, ws, args.shard, tot),
        "cpu_baseline": {
            "value": value,
            "unit": "images/s",
            "cores": cores,
            "kind": st.kind,
            "host": refarm.host_cpu(),
            "sample": sample,
            "seconds_per_pass": t_pass,
            "t_act_output_s": float(np.mean([r["t_act_output_s"] for r in steps])),
            "t_tap_s": float(np.mean([r["t_tap_s"] for r in steps])),
            "modes": {"workers1": seq, "threadpool": thr,
                      "process_pool": {"images_per_s": value, "seconds_per_pass": t_pass, "cores": cores}},
            "implementation": "hecnet (reference package, unmodified, baseline/_ref)" if st.kind == "reference"
            else "oracle port (baseline/_ref missing)",
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
            # capability check that cannot fail on one rank only: every rank
            # votes (symmetric-memory module present, peer access to every
            # local GPU) before any rank enters the collective rendezvous
            cap = 1
            try:
                import torch.distributed._symmetric_memory  # noqa: F401

                n_local = torch.cuda.device_count()
                for peer in range(n_local):
                    if peer != local and not torch.cuda.can_device_access_peer(local, peer):
                        cap = 0
            except Exception:  # noqa: BLE001 - vote 0
                cap = 0
            flag = torch.tensor([cap], device="cuda", dtype=torch.int32)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 0:
                transport = "nccl"
                args.transport_note = "p2p capability vote failed on some rank"
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
    keyswitch, square = _keyswitch_objects(P, ek, peak, 256 if P.n <= 8192 else 128)
    keyswitch["inner_product_subkernel"] = {
        "kernel": "keymac_f64_kernel alone (per-limb form, fcn_key_mac: sum_d key_d * digit_d, NTT domain; "
                  "bytes = digits + accumulators)",
        "achieved": ks["bytes"] / ks["t_s"] / 1e9, "frac": ks["bytes"] / ks["t_s"] / 1e9 / peak,
        "ciphertexts_per_launch": ks["count"], "ms": ks["t_s"] * 1e3}
    hops = engine.plan_hops(comp, "batched", W.t).totals
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        # cpu_baseline leg: the reference package (baseline/_ref) on one host
        # core; the oracle's plain mod-t model also checks the decrypted output
        import refarm
        from oracle import drivers as od

        slots = engine.decrypt_tensor_slots(sk, out)
        check = bool(np.array_equal(slots, od.plain_model_batched(comp, x << cfg.precision_bits, W.t)))
        rst = refarm.RefState(args.workload)
        seq = refarm.sequential(rst, args.cpu_seconds)
        cpu = {"value": seq["images_per_s"], "unit": "images/s", "cores": 1, "kind": rst.kind,
               "sample": seq["sample"] + "; pass time extrapolated by the plan's HOP structure",
               "seconds_per_pass": seq["seconds_per_pass"], "host": refarm.host_cpu(),
               "t_act_output_s": seq["t_act_output_s"], "t_mul_pt_s": seq["t_mul_pt_s"], "t_add_ct_s": seq["t_add_ct_s"],
               "implementation": "hecnet (reference package, unmodified, baseline/_ref)" if rst.kind == "reference"
               else "oracle port (baseline/_ref missing)"}
    try:
        import refarm

        digest = refarm.output_digest(out.buf)
    except Exception:  # noqa: BLE001 - informational
        digest = None
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
        "square_relin": square,
        "cpu_baseline": cpu,
        "output_sha256": digest,
        "e2e": e2e,
    }
    print(json.dumps(line), flush=True)


def run_sweep(args, ws, rank, local):
    """cfg5: the primitive pass (NTT fwd+inv, square + relinearisation with
    dnum = 3 keys, the 1024-term sparse pow2 MAC) over 4,096 uniform
    ciphertexts, sharded over the ranks by ciphertext with one all-gather of
    the squares before the MAC (paper_1811_09953_b200/sweep.py).
    value = ciphertexts through the whole pass per second."""
    import torch
    import torch.distributed as dist

    from paper_1811_09953_b200 import _lib, configs, dist as fdist, fv, sweep

    torch.cuda.set_device(local)
    _lib.load()
    W = configs.WORKLOADS["cfg5"]
    P = fv.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
    sk, pk, ek = fv.keygen(P, configs.SEED_KEYS)
    B, terms = 4096, 1024
    plan = configs.mac_sweep_plan(n_out=B, n_in=B, terms=terms, seed=1)
    group = dist.group.WORLD if ws > 1 else None
    pp = sweep.PrimitivePass(P, ek, plan, rank, ws, group)
    x = sweep.uniform_batch(P, B, seed=0)
    lo, hi = fdist.partition(B, ws)[rank]
    x_local = x[lo:hi].contiguous()
    del x
    torch.cuda.empty_cache()

    def barrier():
        if ws > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        nt, sq, mac = pp.run(x_local)
    torch.cuda.synchronize()
    ntt_ok = bool(torch.equal(nt, x_local))
    L = _lib.lib()
    n0 = L.fcn_launch_count()
    per_op = []
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            nt, sq, mac = pp.run(x_local)
            e1.record()
            e1.synchronize()
            per_op.append(pp.times())
        e1.record()
        torch.cuda.synchronize()
        barrier()
    launches = (L.fcn_launch_count() - n0) // args.steps
    t_step = e0.elapsed_time(e1) / 1e3 / args.steps
    if ws > 1:
        tt = torch.tensor([t_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
    ops = {k: float(np.mean([d[k] for d in per_op])) for k in per_op[0]}
    if ws > 1:
        for k_ in list(ops):
            tt = torch.tensor([ops[k_]], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ops[k_] = float(tt.item())
    # e2e through the same API: the rank's block of ciphertexts from pinned
    # host memory in, its MAC output rows out, every step
    e2e = None
    if not args.no_e2e:
        host_in = x_local.cpu().pin_memory()
        host_out = torch.empty(mac.shape, dtype=torch.int64, pin_memory=True)
        dev_in = torch.empty_like(x_local)
        barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_e2e = max(1, min(args.steps, 5))
        s0.record()
        for _ in range(n_e2e):
            dev_in.copy_(host_in, non_blocking=True)
            _, _, m = pp.run(dev_in)
            host_out.copy_(m, non_blocking=True)
        s1.record()
        torch.cuda.synchronize()
        barrier()
        t_e2e = s0.elapsed_time(s1) / 1e3 / n_e2e
        if ws > 1:
            tt = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        e2e = {"value": B / t_e2e, "unit": "ciphertexts/s", "h2d_bytes_per_step": host_in.numel() * 8,
               "d2h_bytes_per_step": host_out.numel() * 8, "ms_per_step": t_e2e * 1e3, "batches": n_e2e,
               "api": "sweep.PrimitivePass.run (pinned host block in, host MAC rows out)"}
        del host_in, host_out, dev_in
    if rank != 0:
        return
    peak, _ = _peaks()
    k, n = len(W.primes), W.n
    Pb = 2 * k * n * 8
    b_loc = hi - lo
    keys = 2 * (P.ell + 1) * k * n * 8
    fp = _fp64_peak()
    h = P.native()
    rs = L.fcn_ntt_f64_schedule(n.bit_length() - 1, max(tuple(W.primes)))
    bfly = 2 * (2 * b_loc * k) * (n // 2) * (n.bit_length() - 1)
    pk_b = (fp.get("butterfly_rs1_per_s", fp["butterfly_per_s"]) if rs >= 1 else fp["butterfly_per_s"]) if fp else None
    o_loc = fdist.partition(B, ws)[0][1]
    term_coeffs = o_loc * terms * 2 * k * n
    per_op_roof = {
        "ntt_fwd_inv": {"ms": ops["ntt_fwd_inv_s"] * 1e3, "bytes": 4 * b_loc * Pb,
                        "achieved_gbs": 4 * b_loc * Pb / ops["ntt_fwd_inv_s"] / 1e9,
                        "frac": 4 * b_loc * Pb / ops["ntt_fwd_inv_s"] / 1e9 / peak,
                        "frac_fp64_butterfly_peak": (bfly / ops["ntt_fwd_inv_s"] / pk_b) if pk_b else None},
        "square_relin": {"ms": ops["square_relin_s"] * 1e3, "bytes": 2 * b_loc * Pb + keys,
                         "achieved_gbs": (2 * b_loc * Pb + keys) / ops["square_relin_s"] / 1e9,
                         "frac": (2 * b_loc * Pb + keys) / ops["square_relin_s"] / 1e9 / peak,
                         "ciphertexts_per_s": b_loc / ops["square_relin_s"]},
        "mac_1024_terms": {"ms": ops["mac_s"] * 1e3, "bytes": (B + o_loc) * Pb,
                           "achieved_gbs": (B + o_loc) * Pb / ops["mac_s"] / 1e9,
                           "frac": (B + o_loc) * Pb / ops["mac_s"] / 1e9 / peak,
                           "term_coeffs_per_s": term_coeffs / ops["mac_s"]},
        "allgather": {"ms": ops["allgather_s"] * 1e3, "bytes_per_rank": (B - b_loc) * Pb},
    }
    ks, square = _keyswitch_objects(P, ek, peak, 128)
    line = {
        "metric": "cfg5 primitive pass (NTT fwd+inv, square+relin dnum=3, 1024-term MAC)",
        "value": B / t_step,
        "unit": "ciphertexts/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": t_step * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic (4,096 seeded uniform ciphertexts; MAC plan seed 1)",
        "config": {"workload": "cfg5", "n": n, "limbs": k, "t": W.t, "beta_log2": 134, "dnum": P.ell + 1,
                   "ciphertexts": B, "mac_terms": terms, "parallelism": f"ciphertext-shard{ws}" if ws > 1 else "single",
                   "l2": "inputs larger than L2 (%d MB of ciphertexts per rank)" % (b_loc * Pb >> 20)},
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "ntt_roundtrip_identity": ntt_ok,
        "per_op": per_op_roof,
        "roofline": dict(per_op_roof["ntt_fwd_inv"], kernel="ntt_f64_fwd / ntt_f64_inv", bound="hbm",
                         achieved=per_op_roof["ntt_fwd_inv"]["achieved_gbs"], peak=peak, unit="GB/s",
                         traffic=_profile_traffic("ntt_cfg5")),
        "keyswitch_roofline": ks,
        "square_relin": square,
        "cpu_baseline": None,
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
            # NCCL's own init log (nranks / transport per rank) on stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries only the JSON line
        dist.init_process_group(backend)
        if backend == "nccl":
            probe = torch.ones(1, device="cuda")
            dist.all_reduce(probe)  # creates the communicator now
            print(f"[bench] rank {rank}/{ws} local {local} nccl communicator nranks={int(probe.item())} "
                  f"device={torch.cuda.get_device_name(local)}", file=sys.stderr, flush=True)
    if args.impl == "reference":
        run_reference(args, ws, rank)
    elif args.workload == "cfg5":
        run_sweep(args, ws, rank, local)
    else:
        run_gpu(args, ws, rank, local)
    if group:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
