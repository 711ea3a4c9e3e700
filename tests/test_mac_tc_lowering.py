"""CPU checks of the tensor-core MAC lowering (paper_1811_09953_b200/mac_tc.py):
the grouped int8 tiles hold exactly the plan's terms in the canonical
layout the kernel reads, for dense, convolution-shaped and cfg5-shaped
plans, and the cost model picks the positions split of a convolution."""

import numpy as np
import pytest

from paper_1811_09953_b200 import configs, engine, mac_tc, netplan


def _host_mac(plan, t=65537):
    outs = plan.outputs
    counts = np.array([len(o.taps) for o in outs])
    rowptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    col = np.array([tp.in_index for o in outs for tp in o.taps], dtype=np.int64)
    w = np.array([tp.weight_int for o in outs for tp in o.taps], dtype=np.int64) % t
    coef = np.where(w > t // 2, w - t, w)
    return engine._Mac(None, None, None, None, len(outs), len(col), True, int(np.abs(coef).max()),
                       (rowptr, col, coef))


def _check(plan, n_in, P=7, cols=2 * 4 * 1024):
    mac = _host_mac(plan)
    tcp = mac_tc.build(mac, n_in, P, cols, force=True, device="cpu")
    assert tcp is not None
    rowptr, col, coef = mac.host
    want = sorted((o, int(col[e]), int(coef[e])) for o in range(mac.n_out) for e in range(rowptr[o], rowptr[o + 1]))
    assert mac_tc.decode(tcp) == want
    return tcp


def test_dense_plan_tiles():
    rng = np.random.default_rng(0)
    w = rng.choice([0.0, 0.5, -0.25, 1.0, -0.015625], size=(300, 333), p=[0.8, 0.05, 0.05, 0.05, 0.05])
    net = netplan.NetworkSpec((333,), [netplan.Dense(w, None)])
    plan = netplan.compile_network(net, configs.WORKLOADS["cfg2"].fixed_point()).plans[0]
    tcp = _check(plan, 333)
    assert tcp.n_groups >= 3  # at most 128 rows per group


def test_conv_plan_groups_by_position():
    net = configs.build_network("cfg2")
    comp = netplan.compile_network(net, configs.WORKLOADS["cfg2"].fixed_point())
    conv = comp.plans[0]
    tcp = _check(conv, 784)
    # 5 channels x 169 positions: the cost model groups all channels of a few
    # positions (a receptive-field union), not consecutive outputs
    assert tcp.split == 169
    kg = tcp.groups.numpy()[:, 3]
    assert kg.max() <= 5 * 25 * 2  # a few overlapping 5x5 windows


def test_cfg5_shaped_plan():
    plan = configs.mac_sweep_plan(n_out=256, n_in=512, terms=64, seed=3)
    tcp = _check(plan, 512)
    assert tcp.n_groups == 2


def test_ineligible_plans_fall_back():
    plan = configs.mac_sweep_plan(n_out=8, n_in=16, terms=4, seed=3)
    mac = _host_mac(plan)
    mac.max_abs_coef = 200
    assert mac_tc.build(mac, 16, 7, 2048, force=True, device="cpu") is None
    mac = _host_mac(plan)
    assert mac_tc.build(mac, 16, 4, 2048, force=True, device="cpu") is None  # limbs below 2^32


def test_empty_rows_and_groups():
    """Rows without taps (engine.py:711-712 emits Ciphertext.zero) and a whole
    group of them keep one zero-weight chunk, so the kernel writes zeros."""
    outs = [netplan.LinearOut((), None) for _ in range(130)]
    outs[3] = netplan.LinearOut((netplan.TapPlan(2, 8), netplan.TapPlan(5, -4)), None)
    plan = netplan.LinearPlan("sparse", tuple(outs))
    tcp = _check(plan, 6)
    grp = tcp.groups.numpy()
    assert (grp[:, 3] >= 1).all()
