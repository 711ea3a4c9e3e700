"""Reference CPU arm of `bench.py`: the reference package `hecnet` itself,
timed on this host's cores.

Measurement infrastructure, not product code.  The reference is installed
unmodified into `baseline/_ref` (`pip install --no-index --no-deps --target
baseline/_ref <copy of /root/reference/pkg>`); that
directory travels to the GPU box with the repo snapshot.  When it is missing
the CPU oracle port (`oracle/`) stands in and every line says
`kind: "port"`.

The batched (SIMD) workloads are evaluated exactly as the reference's
`engine.eval_encrypted` walks a compiled plan (engine.py:651-774) -- per
linear output a chain of `fv.mul_pt` + `fv.add_ct` (+ `fv.add_pt`), per
activation `fv.mul_ct(x, x)` -> `mul_pt(a2)` -> `+ mul_pt(x, a1)` ->
`add_pt(a0)` -- with the integer constants encoded as constant plaintexts
`PlainPoly(t, [z mod t])` (the slot encoding), so the CPU
does the same homomorphic operations as the GPU path on the same
ciphertexts.  The plan is the reference's own `compile_network` of the
workload's network.

Three CPU modes:
  (a) ``workers1``   -- the evaluation loop on one core (reference as shipped);
  (b) ``threadpool`` -- the reference's own ThreadPool with workers = cores
                        (engine.py:682-690; GIL-bound);
  (c) ``process_pool`` -- a fork pool over each layer's independent outputs,
                        calling the same reference functions (best honest
                        CPU number).
Per-op costs are measured on a bounded sample and extrapolated with the
plan's HOP counts (the reference's `project_hops` rule); `full_pass` runs a
whole network (cfg1/cfg2/cfg4) through mode (c) and returns the digest of
the output ciphertext bytes for a byte-for-byte comparison with the GPU.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(REPO, "baseline", "_ref")


def load_reference():
    """Import the installed reference package (None when it is absent)."""
    if os.path.isdir(REF_DIR) and REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        from hecnet import approx, encode, engine, fv, ring  # noqa: F401
    except Exception:  # noqa: BLE001 - absent or broken install -> port
        return None
    import hecnet

    return hecnet


def host_cpu() -> dict:
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


# ----------------------------------------------------------------- backends


class _Hecnet:
    """The reference's own types and operations."""

    kind = "reference"

    def __init__(self, W):
        from hecnet import fv, ring

        self.fv, self.ring = fv, ring
        self.t = W.t
        self.P = fv.EncryptionParams(W.n, W.primes, (W.t,), W.beta)
        self.sk, self.pk, self.ek = fv.keygen(self.P, _seeds().SEED_KEYS)
        self.tctx = ring.RingContext.create(W.n, (W.t,))

    def const(self, z: int):
        return self.fv.PlainPoly(self.t, np.array([int(z) % self.t], dtype=np.uint64))

    def mul_ct(self, a, b):
        return self.fv.mul_ct(a, b, self.ek)

    def mul_pt(self, ct, m, s):
        return self.fv.mul_pt(ct, m, s)

    def add_ct(self, a, b):
        return self.fv.add_ct(a, b)

    def add_pt(self, ct, m):
        return self.fv.add_pt(ct, m)

    def scale(self, ct):
        return ct.scale_exponent

    def zero(self, scale):
        return self.fv.Ciphertext.zero(self.P, 0, scale)

    def encrypt_slots(self, z, scale, rng):
        """Slot vector -> inverse NTT over Z_t -> fv.encrypt."""
        v = np.zeros((1, self.P.n), dtype=np.uint64)
        v[0, : z.size] = np.mod(np.asarray(z, dtype=np.int64), self.t).astype(np.uint64)
        coeffs = self.ring.ntt_inverse(self.ring.RingPoly(self.tctx, v, self.ring.NTT)).data[0]
        return self.fv.encrypt(self.pk, self.P, self.fv.PlainPoly(self.t, coeffs), 0, scale, rng)

    def arrays(self, ct):
        return ct.c0.data, ct.c1.data

    def from_arrays(self, c0, c1, scale, depth):
        R = self.ring.RingPoly
        return self.fv.Ciphertext(R(self.P.ctx, c0), R(self.P.ctx, c1), self.P, 0, scale, depth)

    def depth(self, ct):
        return ct.mul_depth

    def compile(self, net, cfg):
        from hecnet import approx, encode, engine

        def tr(L):
            k = type(L).__name__
            if k == "Conv2d":
                return engine.Conv2d(L.weights, L.bias, L.stride, L.padding, L.mask)
            if k == "Dense":
                return engine.Dense(L.weights, L.bias, L.mask)
            if k == "ScaledAvgPool":
                return engine.ScaledAvgPool(L.window, L.stride, L.padding, L.reciprocal)
            if k == "PolyActivation":
                c = tuple(float(v) for v in L.poly.coeffs)
                return engine.PolyActivation(approx.PolyApprox(2, c, 4.0, 0.0))
            raise KeyError(k)

        rnet = engine.NetworkSpec(net.input_shape, [tr(L) for L in net.layers])
        return engine.compile_network(rnet, encode.FixedPointConfig(tuple(cfg.t_lanes), cfg.precision_bits))


class _Port:
    """The CPU oracle port (oracle/), used only when the reference is absent."""

    kind = "port"

    def __init__(self, W):
        from oracle import bfv as ob

        self.ob = ob
        self.t = W.t
        self.P = ob.Params(W.n, W.primes, (W.t,), W.beta)
        self.K = ob.keygen(self.P, _seeds().SEED_KEYS)

    def const(self, z):
        return [int(z) % self.t]

    def mul_ct(self, a, b):
        return self.ob.mul_ct(self.P, a, b, self.K)

    def mul_pt(self, ct, m, s):
        return self.ob.mul_pt(self.P, ct, m, s)

    def add_ct(self, a, b):
        return self.ob.add_ct(self.P, a, b)

    def add_pt(self, ct, m):
        return self.ob.add_pt(self.P, ct, m)

    def scale(self, ct):
        return ct.scale

    def zero(self, scale):
        z = np.zeros((len(self.P.primes), self.P.n), dtype=np.uint64)
        return self.ob.Ct(z, z.copy(), 0, scale, 0)

    def encrypt_slots(self, z, scale, rng):
        from oracle import drivers as od

        coeffs = od.slot_encode(np.asarray(z), self.t, self.P.n)
        return self.ob.encrypt(self.P, self.K, coeffs, 0, scale, rng)

    def arrays(self, ct):
        return ct.c0, ct.c1

    def from_arrays(self, c0, c1, scale, depth):
        return self.ob.Ct(c0, c1, 0, scale, depth)

    def depth(self, ct):
        return ct.depth

    def compile(self, net, cfg):
        from paper_1811_09953_b200 import netplan

        return netplan.compile_network(net, cfg)


def _seeds():
    if REPO not in sys.path:
        sys.path.insert(0, REPO)
    from paper_1811_09953_b200 import configs

    return configs


# ---------------------------------------------------------- plan evaluation


def _plan_kind(plan) -> str:
    return type(plan).__name__


def linear_output(B, plan_out, cur, scale, prec):
    """One linear output: mul_pt + add_ct chain (+ add_pt bias) (engine.py:698-717)."""
    acc = None
    for tap in plan_out.taps:
        term = B.mul_pt(cur[tap.in_index], B.const(tap.weight_int), prec)
        acc = term if acc is None else B.add_ct(acc, term)
    if acc is None:
        acc = B.zero(scale + prec)
    if plan_out.bias_int is not None:
        acc = B.add_pt(acc, B.const(plan_out.bias_int))
    return acc


def act_output(B, plan, x, prec):
    """One activation output (engine.py:744-770) with constant plaintexts."""
    sq = B.mul_ct(x, x)
    acc = B.mul_pt(sq, B.const(plan.a2_int), prec) if plan.a2_int is not None else sq
    if plan.a1_mult_int is not None:
        lin = B.mul_pt(x, B.const(plan.a1_mult_int), B.scale(acc) - B.scale(x))
        acc = B.add_ct(acc, lin)
    if plan.a0_add_int is not None:
        acc = B.add_pt(acc, B.const(plan.a0_add_int))
    return acc


class RefState:
    """Per-process state of a workload: backend, keys, plan, sample inputs."""

    def __init__(self, workload: str, n_inputs: int = 4, prefer_reference: bool = True):
        cfgs = _seeds()
        self.W = cfgs.WORKLOADS[workload]
        self.workload = workload
        hec = load_reference() if prefer_reference else None
        self.B = _Hecnet(self.W) if hec is not None else _Port(self.W)
        self.kind = self.B.kind
        self.net = cfgs.build_network(workload)
        self.cfg = self.W.fixed_point()
        self.prec = self.cfg.precision_bits
        self.plan = self.B.compile(self.net, self.cfg)
        self.x = cfgs.build_inputs(workload)
        rng = np.random.default_rng(cfgs.SEED_ENC)
        z = self.x[:n_inputs] << self.prec
        self.cts = [self.B.encrypt_slots(z[i], self.prec, rng) for i in range(n_inputs)]
        acts = [p for p in self.plan.plans if _plan_kind(p) == "ActPlan"]
        self.act = acts[0] if acts else None
        lins = [p for p in self.plan.plans if _plan_kind(p) == "LinearPlan"]
        self.weights = [tp.weight_int for p in lins for o in p.outputs for tp in o.taps][:4096]

    # ---- per-op samples
    def run_act(self, i: int = 0):
        return act_output(self.B, self.act, self.cts[i % len(self.cts)], self.prec)

    def run_linear(self, taps: int, seed: int = 0):
        """A linear output of `taps` terms over the sample inputs (returns (t_mul_pt, t_add_ct))."""
        B, cts = self.B, self.cts
        tm = ta = 0.0
        acc = None
        for j in range(taps):
            w = self.weights[(seed * 131 + j) % len(self.weights)]
            t0 = time.perf_counter()
            term = B.mul_pt(cts[j % len(cts)], B.const(w), self.prec)
            t1 = time.perf_counter()
            acc = term if acc is None else B.add_ct(acc, term)
            t2 = time.perf_counter()
            tm += t1 - t0
            ta += t2 - t1 if j else 0.0
        return tm, ta

    # ---- extrapolation by the plan's HOP structure
    def pass_seconds(self, t_act: float, t_mulpt: float, t_add: float) -> float:
        """One evaluation pass: per-activation-output cost x nodes + per-tap costs
        (the reference's project_hops structure, engine.py:535-581)."""
        tot = 0.0
        for p in self.plan.plans:
            k = _plan_kind(p)
            if k == "LinearPlan":
                taps = sum(len(o.taps) for o in p.outputs)
                adds = sum(max(0, len(o.taps) - 1) + (o.bias_int is not None) for o in p.outputs)
                tot += taps * t_mulpt + adds * t_add
            elif k == "PoolPlan":
                tot += sum(max(0, len(o) - 1) for o in p.outputs) * t_add
                if p.reciprocal_int is not None:
                    tot += len(p.outputs) * t_mulpt
            elif k == "ActPlan":
                tot += p.nodes * t_act
        return tot

    def hop_totals(self):
        """HOP totals of the plan in batched mode (engine.py:535-581 rules;
        counted by plan type name, so it reads the reference's plans too)."""
        from paper_1811_09953_b200.netplan import LayerCounts

        c = LayerCounts()
        for p in self.plan.plans:
            k = _plan_kind(p)
            if k == "LinearPlan":
                for o in p.outputs:
                    c.pt_ct_mul += len(o.taps)
                    c.ct_ct_add += max(0, len(o.taps) - 1)
                    c.pt_ct_add += o.bias_int is not None
            elif k == "PoolPlan":
                for o in p.outputs:
                    c.ct_ct_add += max(0, len(o) - 1)
                    c.pt_ct_mul += p.reciprocal_int is not None
            elif k == "ActPlan":
                c.ct_ct_mul += p.nodes
                c.pt_ct_mul += p.nodes * ((p.a2_int is not None) + (p.a1_mult_int is not None))
                c.ct_ct_add += p.nodes * (p.a1_mult_int is not None)
                c.pt_ct_add += p.nodes * (p.a0_add_int is not None)
        return c


# ------------------------------------------------------------------ modes

_STATE: RefState | None = None


def _init_worker(workload, prefer_reference):
    global _STATE
    if _STATE is None or _STATE.workload != workload:
        _STATE = RefState(workload, prefer_reference=prefer_reference)


def _job_act(i):
    t0 = time.perf_counter()
    _STATE.run_act(i)
    return time.perf_counter() - t0


def _job_lin(args):
    taps, seed = args
    return _STATE.run_linear(taps, seed)


def sequential(st: RefState, budget_s: float) -> dict:
    """Mode (a): one core, the evaluation loop as shipped (workers=1)."""
    n_act, t0 = 0, time.perf_counter()
    while n_act < 1 or (time.perf_counter() - t0 < 0.7 * budget_s and n_act < 16):
        st.run_act(n_act)
        n_act += 1
    t_act = (time.perf_counter() - t0) / n_act
    n_taps, tm, ta, t0 = 0, 0.0, 0.0, time.perf_counter()
    while n_taps < 16 or (time.perf_counter() - t0 < 0.3 * budget_s and n_taps < 4096):
        a, b = st.run_linear(16, n_taps)
        tm, ta, n_taps = tm + a, ta + b, n_taps + 16
    t_mulpt, t_add = tm / n_taps, ta / (n_taps - n_taps // 16)
    t_pass = st.pass_seconds(t_act, t_mulpt, t_add)
    return {"images_per_s": st.W.slots / t_pass, "seconds_per_pass": t_pass, "cores": 1,
            "t_act_output_s": t_act, "t_mul_pt_s": t_mulpt, "t_add_ct_s": t_add,
            "sample": f"{n_act} activation outputs + {n_taps} linear taps on one core"}


def threadpool(st: RefState, workers: int, budget_s: float, t_act_seq: float) -> dict:
    """Mode (b): the reference's ThreadPool over a layer's outputs (engine.py:682-690)."""
    from concurrent.futures import ThreadPoolExecutor

    n_act = max(2, min(workers, int(budget_s * 0.7 / max(t_act_seq, 1e-3))))
    with ThreadPoolExecutor(max_workers=workers) as pool:
        t0 = time.perf_counter()
        list(pool.map(lambda i: st.run_act(i), range(n_act)))
        t_act = (time.perf_counter() - t0) / n_act
        taps = 32
        t0 = time.perf_counter()
        list(pool.map(lambda i: st.run_linear(taps, i), range(workers)))
        t_lin = (time.perf_counter() - t0) / (workers * taps)
    t_pass = st.pass_seconds(t_act, t_lin, 0.0)
    return {"images_per_s": st.W.slots / t_pass, "seconds_per_pass": t_pass, "cores": workers,
            "t_act_output_s": t_act, "t_tap_s": t_lin,
            "sample": f"ThreadPool(max_workers={workers}): {n_act} activation outputs, "
                      f"{workers} linear outputs x {taps} taps"}


class ProcessPool:
    """Mode (c): fork pool over independent outputs calling the reference's functions."""

    def __init__(self, st: RefState, cores: int):
        import multiprocessing as mp

        global _STATE
        _STATE = st  # forked workers inherit the keys and sample ciphertexts
        self.st = st
        self.cores = cores
        self.pool = mp.get_context("fork").Pool(cores)

    def step(self, taps: int = 32) -> dict:
        c = self.cores
        t0 = time.perf_counter()
        self.pool.map(_job_act, range(c), chunksize=1)
        t_act = (time.perf_counter() - t0) / c
        t0 = time.perf_counter()
        self.pool.map(_job_lin, [(taps, i) for i in range(c)], chunksize=1)
        t_tap = (time.perf_counter() - t0) / (c * taps)
        t_pass = self.st.pass_seconds(t_act, t_tap, 0.0)
        return {"seconds_per_pass": t_pass, "t_act_output_s": t_act, "t_tap_s": t_tap}

    def close(self):
        self.pool.terminate()
        self.pool.join()


# ------------------------------------------------------------- full pass

_LAYER = None


def _full_job(i):
    B, kind, plan, cur, scale, prec = _LAYER
    if kind == "LinearPlan":
        ct = linear_output(B, plan.outputs[i], cur, scale, prec)
    else:
        ct = act_output(B, plan, cur[i], prec)
    c0, c1 = B.arrays(ct)
    return c0, c1, B.scale(ct), B.depth(ct)


def full_pass(workload: str, cores: int | None = None, log=None) -> dict:
    """Encrypt the workload's inputs with the reference (seed SEED_ENC, the
    reference's draw order) and evaluate the whole network with mode (c).
    Returns wall times and the SHA-256 of the output ciphertext bodies
    ([B][2][k][n] little-endian u64, the GPU buffer layout)."""
    import multiprocessing as mp

    global _LAYER
    cores = cores or os.cpu_count() or 1
    st = RefState(workload, n_inputs=1)
    B = st.B
    cfgs = _seeds()
    rng = np.random.default_rng(cfgs.SEED_ENC)
    z = st.x << st.prec
    t0 = time.perf_counter()
    cur = [B.encrypt_slots(z[i], st.prec, rng) for i in range(z.shape[0])]
    t_enc = time.perf_counter() - t0
    scale = st.prec
    layers = []
    t_eval = 0.0
    for plan in st.plan.plans:
        kind = _plan_kind(plan)
        count = len(plan.outputs) if kind == "LinearPlan" else plan.nodes
        _LAYER = (B, kind, plan, cur, scale, st.prec)
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(cores) as pool:
            res = pool.map(_full_job, range(count), chunksize=max(1, count // (cores * 8)))
        dt = time.perf_counter() - t0
        t_eval += dt
        cur = [B.from_arrays(c0, c1, s, d) for c0, c1, s, d in res]
        scale = B.scale(cur[0])
        layers.append({"layer": plan.name, "kind": kind, "outputs": count, "seconds": dt})
        if log:
            log(f"[refarm] {workload} {plan.name}: {count} outputs in {dt:.1f} s")
    h = hashlib.sha256()
    for ct in cur:
        c0, c1 = B.arrays(ct)
        h.update(np.ascontiguousarray(c0, dtype="<u8").tobytes())
        h.update(np.ascontiguousarray(c1, dtype="<u8").tobytes())
    return {"kind": st.kind, "workload": workload, "cores": cores, "encrypt_s": t_enc, "eval_s": t_eval,
            "images_per_s": st.W.slots / t_eval, "layers": layers, "out_sha256": h.hexdigest(),
            "out_scale": scale, "host": host_cpu()}


def output_digest(buf) -> str:
    """SHA-256 of a [B][2][k][n] device/host buffer in the same byte order."""
    import torch

    a = buf.detach().to("cpu").contiguous() if isinstance(buf, torch.Tensor) else np.asarray(buf)
    arr = a.numpy() if hasattr(a, "numpy") else a
    return hashlib.sha256(np.ascontiguousarray(arr.view(np.uint64), dtype="<u8").tobytes()).hexdigest()
