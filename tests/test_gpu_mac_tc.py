"""The tensor-core linear layer (tcgen05 kind::i8 over byte planes,
csrc/mac_tc.cu) is bit-identical to the sparse CUDA-core kernel and to the
oracle's restatement of the reference chain (engine.py:698-717: fv.mul_pt
with constant plaintexts + fv.add_ct) on dense, convolution-shaped and
cfg5-shaped plans, at 5, 7 and 8 byte planes, with output row ranges,
fan-out destinations and extreme residues / coefficients."""

import numpy as np
import pytest
import torch

from paper_1811_09953_b200 import configs, engine, fv, mac_tc, netplan
from paper_1811_09953_b200 import device as dev

pytestmark = pytest.mark.gpu


def _params(k, bits, n=1024):
    primes = tuple(configs.find_ntt_primes(n, k, bits=bits))
    return fv.EncryptionParams(n, primes, (65537,), 1 << 32)


def _inputs(P, count, seed, extreme=False):
    k = len(P.limb_primes)
    g = torch.Generator(device="cuda").manual_seed(seed)
    qs = torch.tensor(list(P.limb_primes), dtype=torch.int64, device="cuda").view(1, 1, k, 1)
    x = torch.randint(0, 1 << 62, (count, 2, k, P.n), device="cuda", generator=g, dtype=torch.int64) % qs
    if extreme:
        x[: count // 2] = (qs - 1).expand(count // 2, 2, k, P.n)
    return x.contiguous()


def _low(plan, P):
    mac, bias, _ = engine._lower_linear(plan, 65537, P.n, "batched")
    return mac, bias


def _sparse(P, mac, x):
    return engine._mac_out(P, mac, x, None)


def _oracle_rows(P, plan, x, rows):
    from oracle import bfv as ob

    xs = dev.to_host(x)
    out = {}
    for o in rows:
        acc = None
        for tp in plan.outputs[o].taps:
            c = ob.Ct(xs[tp.in_index, 0], xs[tp.in_index, 1])
            term = ob.mul_pt(ob.Params(P.n, P.limb_primes, (65537,)), c, [tp.weight_int % 65537], 0)
            acc = term if acc is None else ob.add_ct(ob.Params(P.n, P.limb_primes, (65537,)), acc, term)
        out[o] = np.stack([acc.c0, acc.c1])
    return out


def _plans():
    rng = np.random.default_rng(5)
    w = rng.choice([0.0, 0.5, -0.25, 1.0, -0.015625, 0.0625], size=(200, 300), p=[0.85, 0.03, 0.03, 0.03, 0.03, 0.03])
    dense = netplan.compile_network(netplan.NetworkSpec((300,), [netplan.Dense(w, None)]),
                                    configs.WORKLOADS["cfg2"].fixed_point()).plans[0]
    conv = netplan.compile_network(configs.build_network("cfg2"), configs.WORKLOADS["cfg2"].fixed_point()).plans[0]
    sweep = configs.mac_sweep_plan(n_out=256, n_in=300, terms=100, seed=2)
    return {"dense": (dense, 300), "conv": (conv, 784), "sweep": (sweep, 300)}


@pytest.mark.parametrize("k,bits", [(2, 50), (3, 36), (2, 60)])
@pytest.mark.parametrize("which", ["dense", "conv", "sweep"])
def test_tc_mac_matches_sparse_kernel_and_oracle(k, bits, which):
    P = _params(k, bits)
    plan, n_in = _plans()[which]
    mac, _ = _low(plan, P)
    planes = 5 if bits == 36 else (8 if bits == 60 else 7)
    assert engine._lib.lib().fcn_tc_planes(P.native().ptr) == planes
    tcp = mac_tc.build(mac, n_in, planes, 2 * k * P.n, force=True)
    assert tcp is not None
    x = _inputs(P, n_in, seed=k * 100 + bits, extreme=True)
    want = _sparse(P, mac, x)
    got = torch.empty_like(want)
    mac_tc.run(P, tcp, x, got)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    rows = [0, len(plan.outputs) // 2, len(plan.outputs) - 1]
    ref = _oracle_rows(P, plan, x, rows)
    gh = dev.to_host(got)
    for o in rows:
        assert np.array_equal(gh[o], ref[o])


def test_tc_mac_row_range_and_fanout():
    P = _params(2, 50)
    plan, n_in = _plans()["conv"]
    mac, _ = _low(plan, P)
    tcp = mac_tc.build(mac, n_in, 7, 4 * P.n, force=True)
    x = _inputs(P, n_in, seed=7)
    want = _sparse(P, mac, x)
    lo, hi = 100, 700
    a = torch.zeros((hi - lo,) + tuple(want.shape[1:]), dtype=torch.int64, device="cuda")
    b = torch.zeros_like(a)
    mac_tc.run(P, tcp, x, a, fanout=(b.data_ptr(),), lo=lo, hi=hi)
    torch.cuda.synchronize()
    assert torch.equal(a, want[lo:hi]) and torch.equal(b, want[lo:hi])


def test_tc_mac_extreme_coefficients():
    """|c| = 127 on every term of long rows, every input at q - 1 (largest
    byte-plane sums), both signs."""
    P = _params(2, 50)
    n_in = 640
    outs = []
    for o in range(130):
        sgn = 1 if o % 2 == 0 else -1
        taps = tuple(netplan.TapPlan(i, sgn * 127) for i in range(o % 3, n_in, 1 + o % 2))
        outs.append(netplan.LinearOut(taps, None))
    plan = netplan.LinearPlan("extreme", tuple(outs))
    mac, _ = _low(plan, P)
    tcp = mac_tc.build(mac, n_in, 7, 4 * P.n, force=True)
    assert tcp is not None
    x = _inputs(P, n_in, seed=9, extreme=True)
    x[:] = x[0:1]  # all inputs q - 1
    want = _sparse(P, mac, x)
    got = torch.empty_like(want)
    mac_tc.run(P, tcp, x, got)
    torch.cuda.synchronize()
    assert torch.equal(got, want)


def test_engine_uses_tc_path_bit_exact():
    """eval_encrypted with the tensor-core MAC forced on equals the sparse path."""
    import os

    W = configs.WORKLOADS["cfg2"]
    P = fv.EncryptionParams(1024, tuple(configs.find_ntt_primes(1024, 4, bits=50)), (65537,), 1 << 32)
    sk, pk, ek = fv.keygen(P, 3)
    net = configs.build_network("cfg2")
    cfg = W.fixed_point()
    x = configs.build_inputs("cfg2", slots=1024)
    tensor = engine.encrypt_tensor_batched(pk, P, x, cfg, 0, 4)
    comp = engine.compile_network(net, cfg)
    old = os.environ.get("FCN_MAC_TC")
    try:
        os.environ["FCN_MAC_TC"] = "0"
        want = engine.eval_encrypted(comp, tensor, ek, cfg, encoding="batched")[0].buf.clone()
        os.environ["FCN_MAC_TC"] = "1"
        got = engine.eval_encrypted(comp, tensor, ek, cfg, encoding="batched")[0].buf
    finally:
        if old is None:
            os.environ.pop("FCN_MAC_TC", None)
        else:
            os.environ["FCN_MAC_TC"] = old
    assert torch.equal(got, want)


def test_tc_mac_empty_rows():
    P = _params(2, 50)
    outs = [netplan.LinearOut((), None) for _ in range(200)]
    outs[3] = netplan.LinearOut((netplan.TapPlan(2, 8), netplan.TapPlan(5, -4)), None)
    outs[150] = netplan.LinearOut((netplan.TapPlan(0, 1),), None)
    plan = netplan.LinearPlan("sparse", tuple(outs))
    mac, _ = _low(plan, P)
    tcp = mac_tc.build(mac, 6, 7, 4 * P.n, force=True)
    x = _inputs(P, 6, seed=11)
    want = _sparse(P, mac, x)
    got = torch.full_like(want, -1)
    mac_tc.run(P, tcp, x, got)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    assert int(got[0].abs().sum()) == 0


def test_cfg5_split_simulated_on_one_gpu():
    """sweep.primitive_schedule (SURVEY 8(e)'s cfg5 split) with the GPU
    kernels, ranks of a world of 2 and 3 computed one after another on one
    GPU (no rank waits on another) and gathered by concatenation: every
    rank's pieces equal the single-process pass byte for byte."""
    from paper_1811_09953_b200 import dist as fdist
    from paper_1811_09953_b200 import sweep

    P = _params(4, 50)
    sk, pk, ek = fv.keygen(P, 4)
    B = 7
    plan = configs.mac_sweep_plan(n_out=B, n_in=B, terms=4, seed=3)
    x = sweep.uniform_batch(P, B, seed=5)
    one = sweep.PrimitivePass(P, ek, plan, 0, 1)
    want = [t.clone() for t in one.run(x)]
    for world in (2, 3):
        passes = [sweep.PrimitivePass(P, ek, plan, r, world) for r in range(world)]
        parts = fdist.partition(B, world)
        sq_blocks = [fv.mul_ct_batch(P, ek, 0, x[lo:hi]) if hi > lo else x[:0].clone() for lo, hi in parts]
        full = torch.cat(sq_blocks)
        got_nt, got_sq, got_mac = [], [], []
        for r in range(world):
            lo, hi = parts[r]
            nt, sq, mac = sweep.primitive_schedule(
                x[lo:hi].contiguous(), r, world, B, B, passes[r]._ntt,
                lambda xl, r=r: sq_blocks[r], lambda loc, c, b: full,
                lambda f, a, b, r=r: engine._layer_range(P, 0, ek, plan, ("linear",) + tuple(passes[r].low[:2]), f,
                                                         a, b, "batched") if b > a else f[:0].clone())
            got_nt.append(nt.clone())
            got_sq.append(sq)
            got_mac.append(mac)
        assert torch.equal(torch.cat(got_nt), want[0])
        assert torch.equal(torch.cat(got_sq), want[1])
        assert torch.equal(torch.cat(got_mac), want[2])
