"""Host-side edge cases (CPU): exact rounding of huge weights, matching the
reference's Python-int rounding (encode.py:96-98) instead of wrapping in int64."""

import numpy as np

from paper_1811_09953_b200 import encode, netplan


def test_round_half_away_array_large_magnitudes():
    v = np.array([2.0 ** 70 + 0.0, -(2.0 ** 63), 2.5, -2.5, 0.49999999999999994])
    got = encode.round_half_away_array(v)
    assert [int(x) for x in got] == [encode.round_half_away(x) for x in v]
    assert int(got[0]) == 2 ** 70
    small = encode.round_half_away_array(np.array([1.5, -1.5, 0.0]))
    assert small.dtype == np.int64 and small.tolist() == [2, -2, 0]


def test_compile_network_huge_weight_is_exact():
    w = np.array([[2.0 ** 60, 0.5], [0.0, -1.0]])
    net = netplan.NetworkSpec((2,), [netplan.Dense(w, None)])
    comp = netplan.compile_network(net, encode.FixedPointConfig((65537,), 6))
    taps = comp.plans[0].outputs[0].taps
    assert int(taps[0].weight_int) == 2 ** 66  # would wrap to a garbage tap in int64


def _hecnet():
    import os
    import sys

    import pytest

    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        from hecnet import approx, encode as henc, engine
    except Exception:  # noqa: BLE001
        pytest.skip("reference package not installed in baseline/_ref")
    return approx, henc, engine


def test_compile_network_equals_reference_on_random_networks():
    """netplan.compile_network vs the reference's compile_network (engine.py:437-529)
    on random networks with biases, reciprocal / power-of-two / factor pools
    (a bias after a non-pow2 pool exercises the float evaluation order) and
    activations with every coefficient present."""
    approx, henc, E = _hecnet()
    rng = np.random.default_rng(17)
    for trial in range(6):
        wconv = rng.choice([0.0, 0.5, -0.25, 0.75, 1.5, -0.0625], size=(3, 2, 3, 3))
        bconv = rng.normal(0, 1, 3)
        window = [2, 3][trial % 2]
        recip = trial % 3 == 0
        poly = (float(rng.normal()), float(rng.normal()), 0.125 if trial % 2 else 1.0)
        mine = [netplan.Conv2d(wconv, bconv, stride=1, padding=1),
                netplan.PolyActivation(netplan.PolyApprox(2, poly, 4.0, 0.0)),
                netplan.ScaledAvgPool(window, stride=2, padding=1, reciprocal=recip)]
        theirs = [E.Conv2d(wconv, bconv, 1, 1), E.PolyActivation(approx.PolyApprox(2, poly, 4.0, 0.0)),
                  E.ScaledAvgPool(window, stride=2, padding=1, reciprocal=recip)]
        shape = netplan.NetworkSpec((2, 6, 6), list(mine)).layers[-1].out_shape(
            netplan.Conv2d(wconv, bconv, 1, 1).out_shape((2, 6, 6)))
        n_flat = int(np.prod(shape))
        wd = rng.choice([0.0, 0.5, -1.0, 0.3], size=(4, n_flat))
        bd = rng.normal(0, 1, 4)
        mine.append(netplan.Dense(wd, bd))
        theirs.append(E.Dense(wd, bd))
        cfg = encode.FixedPointConfig((65537,), 5)
        a = netplan.compile_network(netplan.NetworkSpec((2, 6, 6), mine), cfg)
        b = E.compile_network(E.NetworkSpec((2, 6, 6), theirs), henc.FixedPointConfig((65537,), 5))
        assert (a.in_scale, a.out_scale, a.out_factor, tuple(a.out_shape)) == \
            (b.in_scale, b.out_scale, b.out_factor, tuple(b.out_shape)), trial
        for pa, pb in zip(a.plans, b.plans):
            assert type(pa).__name__ == type(pb).__name__ and pa.name == pb.name
            if type(pa).__name__ == "LinearPlan":
                assert [([(t.in_index, int(t.weight_int)) for t in o.taps], o.bias_int) for o in pa.outputs] == \
                    [([(t.in_index, int(t.weight_int)) for t in o.taps], o.bias_int) for o in pb.outputs], (trial, pa.name)
            elif type(pa).__name__ == "PoolPlan":
                assert (pa.outputs, pa.count, pa.pow2_shift, pa.factor_mult, pa.reciprocal_int) == \
                    (pb.outputs, pb.count, pb.pow2_shift, pb.factor_mult, pb.reciprocal_int), (trial, pa.name)
            else:
                assert (pa.nodes, pa.a2_int, pa.a1_mult_int, pa.a0_add_int, pa.scale_bump) == \
                    (pb.nodes, pb.a2_int, pb.a1_mult_int, pb.a0_add_int, pb.scale_bump), (trial, pa.name)
