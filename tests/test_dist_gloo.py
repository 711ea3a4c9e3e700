"""CPU (gloo, world_size 2) tests of the multi-GPU schedule: output
partitioning, stage grouping and the all-gather, with the CPU oracle as the
per-rank compute.  The sharded result must be byte-identical to the
single-process evaluation (reference engine.py:682-690 ordering contract)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_09953_b200 import dist as fdist


def test_partition_and_stages():
    assert fdist.partition(10, 4) == [(0, 3), (3, 6), (6, 9), (9, 10)]
    assert fdist.partition(3, 4) == [(0, 1), (1, 2), (2, 3), (3, 3)]
    assert fdist.partition(0, 2) == [(0, 0), (0, 0)]
    for count in range(0, 40):
        for world in (1, 2, 3, 8):
            parts = fdist.partition(count, world)
            covered = [i for lo, hi in parts for i in range(lo, hi)]
            assert covered == list(range(count))

    class L:  # stand-ins with the reference plan type names
        pass

    Linear = type("LinearPlan", (), {})
    Pool = type("PoolPlan", (), {})
    Act = type("ActPlan", (), {})
    plans = [Linear(), Act(), Pool(), Linear(), Act(), Act(), Linear()]
    assert fdist.stages(plans) == [[0, 1], [2], [3, 4], [5], [6]]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup():
    from oracle import bfv as ob
    from oracle import nt
    from paper_1811_09953_b200 import netplan as L
    from paper_1811_09953_b200.encode import FixedPointConfig

    n = 1024
    primes = tuple(nt.ntt_primes(n, 3, bits=36))
    P = ob.Params(n, primes, (65537,))
    K = ob.keygen(P, 2)
    rng = np.random.default_rng(4)
    conv_w = rng.choice([0.0, 0.25, -0.5, 1.0], size=(3, 1, 3, 3), p=[0.5, 0.2, 0.2, 0.1])
    dense_w = rng.choice([0.0, 0.5, -0.25], size=(5, 27), p=[0.5, 0.25, 0.25])
    net = L.NetworkSpec(
        (1, 5, 5),
        [
            L.Conv2d(conv_w, np.array([0.5, -0.25, 0.125]), 1, 0),
            L.PolyActivation(L.PolyApprox(2, (0.0, 0.5, 0.125))),
            L.Dense(dense_w, np.array([0.25, -1.0, 0.5, 0.0, 1.0])),
            L.PolyActivation(L.square_activation()),
        ],
    )
    cfg = FixedPointConfig((65537,), 3)
    comp = L.compile_network(net, cfg)
    crng = np.random.default_rng(9)
    from oracle import rns as orn

    cts = [ob.Ct(orn.random_uniform(primes, n, crng), orn.random_uniform(primes, n, crng), 0, 3, 0) for _ in range(25)]
    return P, K, comp, cts


def _sub_plan(plan, lo, hi):
    import dataclasses

    kind = type(plan).__name__
    if kind in ("LinearPlan", "PoolPlan"):
        return dataclasses.replace(plan, outputs=plan.outputs[lo:hi])
    return dataclasses.replace(plan, nodes=hi - lo)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import bfv as ob
        from oracle import drivers as od
        from paper_1811_09953_b200.netplan import CompiledNet

        P, K, comp, cts = _setup()
        plans = comp.plans

        def compute(st, cur, lo, hi):
            first = plans[st[0]]
            inputs = cur if type(first).__name__ != "ActPlan" else cur[lo:hi]
            sub = [_sub_plan(plans[i], lo, hi) for i in st]
            out, _, _ = od.run_plan(P, CompiledNet(tuple(sub), 3, 0, 1, ()), inputs, K, 3, "batched")
            body = torch.from_numpy(np.stack([np.stack([c.c0, c.c1]) for c in out]).view(np.int64)) if out else \
                torch.zeros((0, 2, len(P.primes), P.n), dtype=torch.int64)
            meta = [(c.scale, c.depth) for c in out]
            return body, meta

        def gather(local, count, block):
            body, meta = local
            full = fdist._torch_gather(body, count, block)
            metas = [None] * world
            dist.all_gather_object(metas, meta)
            flat = [m for part in metas for m in part]
            arr = full.numpy().view(np.uint64)
            return [ob.Ct(arr[i, 0].copy(), arr[i, 1].copy(), 0, flat[i][0], flat[i][1]) for i in range(count)]

        res = fdist.run_stages(plans, cts, rank, world, compute, gather)
        if rank == 0:
            q.put([(np.stack([c.c0, c.c1]).tobytes(), c.scale, c.depth) for c in res])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_schedule_matches_single_process(world):
    from oracle import drivers as od

    P, K, comp, cts = _setup()
    want, _, _ = od.run_plan(P, comp, cts, K, 3, "batched")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert len(got) == len(want)
    for (body, scale, depth), w in zip(got, want):
        assert body == np.stack([w.c0, w.c1]).tobytes()
        assert (scale, depth) == (w.scale, w.depth)


def _upload_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for count in (7, 2, 1):
            g = torch.Generator().manual_seed(count)
            host = torch.randint(0, 1 << 50, (count, 2, 3, 16), generator=g, dtype=torch.int64)
            full = fdist.upload_sharded(host)
            q.put((rank, count, bool(torch.equal(full, host))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_upload_sharded_reassembles_the_batch(world):
    """dist.upload_sharded: every rank copies only its block of the host batch
    and the all-gather hands every rank the whole batch, including counts
    smaller than the world size (empty blocks)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_upload_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(3 * world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, _, ok in res), res


# ---------------------------------------------------------------- cfg5 split


def _sweep_setup():
    """A miniature cfg5: uniform ciphertexts at n=1024 over 3 limbs, a
    dnum-style large beta, and a sparse pow2 MAC plan (configs.mac_sweep_plan)."""
    from oracle import bfv as ob
    from oracle import nt
    from oracle import rns as orn
    from paper_1811_09953_b200 import configs

    n = 1024
    primes = tuple(nt.ntt_primes(n, 3, bits=36))
    P = ob.Params(n, primes, (65537,), 1 << 40)
    K = ob.keygen(P, 2)
    rng = np.random.default_rng(0)
    B = 5
    cts = [ob.Ct(orn.random_uniform(primes, n, rng), orn.random_uniform(primes, n, rng), 0, 6, 0) for _ in range(B)]
    plan = configs.mac_sweep_plan(n_out=B, n_in=B, terms=3, seed=1)
    return P, K, cts, plan


def _sweep_compute(P, K, plan):
    from oracle import bfv as ob
    from oracle import rns as orn

    def body(cs):
        if not cs:
            return torch.zeros((0, 2, len(P.primes), P.n), dtype=torch.int64)
        return torch.from_numpy(np.stack([np.stack([c.c0, c.c1]) for c in cs]).view(np.int64))

    def cts_of(t, scale, depth):
        arr = t.numpy().view(np.uint64)
        return [ob.Ct(arr[i, 0].copy(), arr[i, 1].copy(), 0, scale, depth) for i in range(arr.shape[0])]

    def ntt_roundtrip(x):
        out = []
        for c in cts_of(x, 6, 0):
            out.append(ob.Ct(orn.intt(orn.ntt(c.c0, P.primes), P.primes), orn.intt(orn.ntt(c.c1, P.primes), P.primes)))
        return body(out)

    def square(x):
        return body([ob.mul_ct(P, c, c, K) for c in cts_of(x, 6, 0)])

    def mac_rows(full, lo, hi):
        ins = cts_of(full, 12, 1)
        outs = []
        for o in plan.outputs[lo:hi]:
            acc = None
            for tp in o.taps:
                term = ob.mul_pt(P, ins[tp.in_index], [tp.weight_int % 65537], 0)
                acc = term if acc is None else ob.add_ct(P, acc, term)
            outs.append(acc)
        return body(outs)

    return ntt_roundtrip, square, mac_rows


def _sweep_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1811_09953_b200 import sweep

        P, K, cts, plan = _sweep_setup()
        ntt_roundtrip, square, mac_rows = _sweep_compute(P, K, plan)
        B = len(cts)
        lo, hi = fdist.partition(B, world)[rank]
        x = torch.from_numpy(np.stack([np.stack([c.c0, c.c1]) for c in cts[lo:hi]]).view(np.int64)) if hi > lo else \
            torch.zeros((0, 2, len(P.primes), P.n), dtype=torch.int64)
        nt, sq, mac = sweep.primitive_schedule(x, rank, world, B, len(plan.outputs), ntt_roundtrip, square,
                                               lambda loc, c, b: fdist._torch_gather(loc, c, b), mac_rows)
        parts = fdist.partition(B, world)
        blk = parts[0][1] - parts[0][0]
        full = [fdist._torch_gather(t, B, blk) for t in (nt, sq, mac)]
        if rank == 0:
            q.put([t.numpy().tobytes() for t in full])
    finally:
        dist.destroy_process_group()


def test_cfg5_split_matches_single_process():
    """SURVEY 8(e)'s cfg5 split (ciphertext shards for the NTT and square +
    relinearisation, one all-gather of the squares, partitioned MAC rows)
    at world size 2 is byte-identical to one process."""
    from paper_1811_09953_b200 import sweep

    P, K, cts, plan = _sweep_setup()
    ntt_roundtrip, square, mac_rows = _sweep_compute(P, K, plan)
    x = torch.from_numpy(np.stack([np.stack([c.c0, c.c1]) for c in cts]).view(np.int64))
    want = sweep.primitive_schedule(x, 0, 1, len(cts), len(plan.outputs), ntt_roundtrip, square,
                                   lambda loc, c, b: loc, mac_rows)
    assert torch.equal(want[0], x)  # the NTT round trip is the identity
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sweep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got == [t.numpy().tobytes() for t in want]
