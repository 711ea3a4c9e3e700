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
