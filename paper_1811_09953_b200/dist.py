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


def eval_encrypted_sharded(net, tensor, ek, cfg, encoding: str = "integer", group=None, mul_chunk=None):
    """Same result as engine.eval_encrypted, computed across the ranks of `group`."""
    import torch
    import torch.distributed as dist

    from . import engine

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    params, lane = tensor.params, tensor.lane
    t = int(params.t_lanes[lane])
    compiled = engine._compiled(net, cfg)
    counter = engine._hops(compiled, encoding, t)
    low = engine._lowered(compiled, t, params.n, encoding)
    prec = cfg.precision_bits
    depths, scales = tensor.depths.copy(), tensor.scales.copy()
    scale, factor = tensor.scale_exponent, tensor.scale_factor
    plans = compiled.plans
    for p, lw in zip(plans, low):
        depths, scales, scale, factor = engine._meta_step(p, lw, depths, scales, scale, factor, prec)

    events = []

    def compute(st, cur, lo, hi):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        out = cur
        for j, idx in enumerate(st):
            plan, lw = plans[idx], low[idx]
            if j == 0:
                out = engine._layer_range(params, lane, ek, plan, lw, cur, lo, hi, encoding, mul_chunk)
            else:  # activation on the rank's own block
                out = engine._layer_range(params, lane, ek, plan, lw, out, lo, hi, encoding, mul_chunk)
        ev1.record()
        events.append((st, ev0, ev1))
        return out

    out = run_stages(plans, tensor.buf, rank, world, compute, lambda loc, c, b: _torch_gather(loc, c, b, group))
    from .netplan import TimedLayerCounts

    for st, a, b in events:
        for idx in st:
            counter.layer_counts[idx] = TimedLayerCounts(counter.layer_counts[idx], (a, b, 1.0 / len(st)))
    res = engine.CipherTensor(compiled.out_shape, scale_exponent=scale, scale_factor=factor, buf=out, params=params,
                              lane=lane, depths=depths, scales=scales)
    return res, counter
