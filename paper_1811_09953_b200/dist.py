"""Multi-GPU evaluation: output sharding + NCCL all-gather (one process per GPU).

Every output ciphertext of a layer is an independent unit (reference
engine.py:682-690 evaluates them in any order and merges counters by sum;
SPEC ordering contract).  `eval_encrypted_sharded` therefore

  * splits the outputs of each linear / pool layer into contiguous,
    equally sized blocks (`partition`), one per rank;
  * runs the following activation on the rank's own block (it is
    elementwise), so a "stage" = linear-or-pool (+ activation);
  * all-gathers the stage's output blocks over NCCL (torch.distributed,
    NVLink / NVSwitch) so every rank holds the next layer's full input.

Metadata (per-ciphertext depth and scale) and the HOP counter are computed
on every rank from the full plan, exactly as the single-GPU evaluator does,
so the result is byte-identical for any world size.

`run_stages` holds the partition / gather schedule independently of the
compute, which is what the CPU (gloo) tests exercise.
"""

from __future__ import annotations

import math

import numpy as np


def partition(count: int, world: int) -> list:
    """Contiguous blocks of ceil(count/world) outputs; trailing ranks may be short or empty."""
    block = max(1, math.ceil(count / world)) if count else 0
    out = []
    for r in range(world):
        lo = min(count, r * block)
        hi = min(count, lo + block)
        out.append((lo, hi))
    return out


def stages(plans) -> list:
    """Group plan indices into stages: [linear|pool (+ act)] or [act]."""
    out, i = [], 0
    kinds = [type(p).__name__ for p in plans]
    while i < len(plans):
        if kinds[i] in ("LinearPlan", "PoolPlan") and i + 1 < len(plans) and kinds[i + 1] == "ActPlan":
            out.append([i, i + 1])
            i += 2
        else:
            out.append([i])
            i += 1
    return out


def stage_outputs(plan) -> int:
    kind = type(plan).__name__
    if kind == "ActPlan":
        return plan.nodes
    return len(plan.outputs)


def run_stages(plans, inputs, rank: int, world: int, compute, gather):
    """Generic sharded schedule.

    compute(stage_plan_indices, cur_full, lo, hi) -> local block (rows lo..hi)
    gather(local_block, count, block_size) -> full rows 0..count
    """
    cur = inputs
    for st in stages(plans):
        count = stage_outputs(plans[st[-1]])
        parts = partition(count, world)
        lo, hi = parts[rank]
        block = parts[0][1] - parts[0][0]
        local = compute(st, cur, lo, hi)
        cur = gather(local, count, block)
    return cur


def _torch_gather(local, count: int, block: int, group=None):
    """All-gather equally padded blocks of [rows][2][k][n] (NCCL / gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    shape = tuple(local.shape[1:])
    pad = local.new_zeros((block,) + shape)
    if local.shape[0]:
        pad[: local.shape[0]].copy_(local)
    full = local.new_empty((block * world,) + shape)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, pad.contiguous(), group=group)
    else:
        chunks = list(full.chunk(world))
        dist.all_gather(chunks, pad.contiguous(), group=group)
        full = torch.cat(chunks)
    return full[:count].contiguous()


def upload_sharded(host_batch, group=None, device=None):
    """One input batch onto every rank with 1/world of the PCIe traffic each.

    Rank r copies its contiguous block of the [count][...] host rows
    (pinned memory: asynchronous) to its own GPU, and the blocks are
    all-gathered over NVLink (NCCL) into the full device batch on every rank
    -- the first layer reads all inputs, so every rank needs the whole batch,
    but no rank's PCIe link carries more than its share.  gloo groups gather
    on the CPU (tests)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    count = host_batch.shape[0]
    parts = partition(count, world)
    lo, hi = parts[rank]
    block = parts[0][1] - parts[0][0]
    if device is None:
        device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    local = host_batch[lo:hi].to(device, non_blocking=True)
    return _torch_gather(local, count, block, group)


def _prepare(net, tensor, cfg, encoding):
    from . import engine

    params, lane = tensor.params, tensor.lane
    t = int(params.t_lanes[lane])
    compiled = engine._compiled(net, cfg)
    counter = engine._hops(compiled, encoding, t)
    low = engine._lowered(compiled, t, params.n, encoding)
    prec = cfg.precision_bits
    depths, scales = tensor.depths.copy(), tensor.scales.copy()
    scale, factor = tensor.scale_exponent, tensor.scale_factor
    for p, lw in zip(compiled.plans, low):
        depths, scales, scale, factor = engine._meta_step(p, lw, depths, scales, scale, factor, prec)
    return compiled, counter, low, (depths, scales, scale, factor)


def _stage(params, lane, ek, plans, low, st, cur, lo, hi, encoding, mul_chunk, out=None, fanout=()):
    """Rows [lo, hi) of one stage; its last layer writes `out` (+ fan-out)."""
    from . import engine

    res = cur
    for j, idx in enumerate(st):
        last = j == len(st) - 1
        res = engine._layer_range(params, lane, ek, plans[idx], low[idx], res if j else cur, lo, hi, encoding, mul_chunk,
                                  out=out if last else None, fanout=fanout if last else ())
    return res


def _result(net, tensor, cfg, encoding, compiled, counter, meta, out, events):
    from . import engine
    from .netplan import TimedLayerCounts

    for st, a, b in events:
        for idx in st:
            counter.layer_counts[idx] = TimedLayerCounts(counter.layer_counts[idx], (a, b, 1.0 / len(st)))
    depths, scales, scale, factor = meta
    res = engine.CipherTensor(compiled.out_shape, scale_exponent=scale, scale_factor=factor, buf=out,
                              params=tensor.params, lane=tensor.lane, depths=depths, scales=scales)
    return res, counter


def eval_encrypted_sharded(net, tensor, ek, cfg, encoding: str = "integer", group=None, mul_chunk=None,
                           transport: str = "nccl"):
    """Same result as engine.eval_encrypted, computed across the ranks of `group`.

    transport="nccl": each stage's block is all-gathered with NCCL.
    transport="p2p": each stage's last kernel writes its block straight into
    every rank's copy of the next layer's input (torch symmetric memory
    mapped over NVLink; fcn_*_multi fan-out stores), followed by a
    device-side barrier -- no separate collective on the data path."""
    import torch
    import torch.distributed as dist

    if transport == "p2p":
        return _eval_p2p(net, tensor, ek, cfg, encoding, group, mul_chunk)
    if transport != "nccl":
        raise ValueError(f"unknown transport {transport!r}")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    params, lane = tensor.params, tensor.lane
    compiled, counter, low, meta = _prepare(net, tensor, cfg, encoding)
    plans = compiled.plans
    events = []

    def compute(st, cur, lo, hi):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        out = _stage(params, lane, ek, plans, low, st, cur, lo, hi, encoding, mul_chunk)
        ev1.record()
        events.append((st, ev0, ev1))
        return out

    out = run_stages(plans, tensor.buf, rank, world, compute, lambda loc, c, b: _torch_gather(loc, c, b, group))
    return _result(net, tensor, cfg, encoding, compiled, counter, meta, out, events)


def _max_rows(plans, world: int) -> int:
    rows = 0
    for st in stages(plans):
        count = stage_outputs(plans[st[-1]])
        block = partition(count, world)[0][1] - partition(count, world)[0][0]
        rows = max(rows, block * world)
    return max(rows, 1)


_P2P_BUFFERS: dict = {}  # (shape, group, device) -> (two symmetric buffers, their handles)


def _eval_p2p(net, tensor, ek, cfg, encoding, group, mul_chunk):
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm

    from . import device as dev
    from . import engine

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world > 8:
        raise ValueError("fan-out transport supports up to 8 ranks (FCN_MAX_FANOUT)")
    params, lane = tensor.params, tensor.lane
    compiled, counter, low, meta = _prepare(net, tensor, cfg, encoding)
    plans = compiled.plans
    shape = (_max_rows(plans, world), 2, len(params.limb_primes), params.n)
    gname = group.group_name if group is not None else dist.group.WORLD.group_name
    key = (shape, gname, dev.current_device())
    ws = _P2P_BUFFERS.get(key)
    if ws is None:
        bufs = [symm.empty(shape, dtype=torch.int64, device=torch.device("cuda", dev.current_device())) for _ in range(2)]
        ws = (bufs, [symm.rendezvous(b, gname) for b in bufs])
        _P2P_BUFFERS[key] = ws
    bufs, hdls = ws
    # no rank may overwrite a peer's buffers while that peer still reads the
    # previous call's result out of them
    hdls[0].barrier(channel=1)
    rb = engine._row_bytes(params)
    events = []
    cur = tensor.buf
    for s_i, st in enumerate(stages(plans)):
        count = stage_outputs(plans[st[-1]])
        lo, hi = partition(count, world)[rank]
        dst, h = bufs[s_i % 2], hdls[s_i % 2]
        peers = [int(h.buffer_ptrs[r]) + lo * rb for r in range(world) if r != rank]
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        if hi > lo:
            _stage(params, lane, ek, plans, low, st, cur, lo, hi, encoding, mul_chunk, out=dst[lo:hi], fanout=peers)
        h.barrier(channel=0)  # every rank's block has landed in every buffer
        ev1.record()
        events.append((st, ev0, ev1))
        cur = dst[:count]
    out = cur.clone()
    return _result(net, tensor, cfg, encoding, compiled, counter, meta, out, events)


def simulate_fanout(net, tensor, ek, cfg, encoding: str, world: int, mul_chunk=None):
    """Single-GPU check of the fan-out schedule: the `world` ranks' stage
    blocks are computed one after another (no rank ever waits on another)
    and each writes its block into all `world` full buffers, exactly as
    _eval_p2p does over NVLink.  Returns the per-rank final buffers."""
    from . import device as dev
    from . import engine

    params, lane = tensor.params, tensor.lane
    compiled, counter, low, meta = _prepare(net, tensor, cfg, encoding)
    plans = compiled.plans
    shape = (_max_rows(plans, world), 2, len(params.limb_primes), params.n)
    bufs = [[dev.empty(shape) for _ in range(world)] for _ in range(2)]
    rb = engine._row_bytes(params)
    cur = [tensor.buf] * world
    for s_i, st in enumerate(stages(plans)):
        count = stage_outputs(plans[st[-1]])
        dst = bufs[s_i % 2]
        for rank in range(world):
            lo, hi = partition(count, world)[rank]
            if hi > lo:
                peers = [dst[r].data_ptr() + lo * rb for r in range(world) if r != rank]
                _stage(params, lane, ek, plans, low, st, cur[rank], lo, hi, encoding, mul_chunk, out=dst[rank][lo:hi],
                       fanout=peers)
        cur = [dst[r][:count] for r in range(world)]
    return [c.clone() for c in cur]
