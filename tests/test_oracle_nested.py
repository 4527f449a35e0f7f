"""Pins for oracle.nested: the literal nested procedure of P:98-114 equals Eq. 2.1 exactly."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import direct
from oracle.cooktoom import correlate_valid_1d
from oracle.nested import (Axis, Counter, TABLE_DIMS, composite, composite_conv2d,
                           nested_conv1d, nested_conv2d, plan_tables)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _ints(shape, seed, lo=-4, hi=5):
    return np.random.default_rng(seed).integers(lo, hi, size=shape).astype(object)


def test_fig3_worked_example():
    g = json.load(open(os.path.join(GOLD, "fig3_nested_f22.json")))
    x = [Fraction(v) for v in [3, -1, 4, 1, -5, 9, 2]]
    w = [Fraction(v) for v in [2, 7, -1, 8]]
    cnt, trace = Counter(), []
    y = nested_conv1d(x, w, m_o=2, m_i=2, r_i=2, counter=cnt, trace=trace)
    assert y == correlate_valid_1d(x, w)
    assert len(y) == g["outputs_per_slice"]
    assert cnt.mults == g["multiplications_per_slice"]
    ax = Axis(2, 2, 2, 2)
    assert ax.L == g["L"] and ax.l_i == g["l"]
    # input reordered matrix columns are the inner-slide windows
    X = trace[0][2]
    for j, cols in enumerate(g["input_reordered_columns"]):
        assert [X[s][j] for s in range(3)] == [x[c] for c in cols]


def test_delta_filter_1d():
    # length-7 x, w = [1,0,0,0], F(2,2), 2 levels -> x[0:4]
    x = [Fraction(v) for v in range(1, 8)]
    assert nested_conv1d(x, [1, 0, 0, 0], 2, 2, r_i=2) == x[:4]


def test_window_law():
    g = json.load(open(os.path.join(GOLD, "window_law.json")))
    for c in g["cases"]:
        ax = Axis(c["m"], c["r"], c["m"], c["r"])
        assert ax.l_i == c["l"] and ax.L == c["L"]


@pytest.mark.parametrize("m_o,r_o,m_i,r_i", [(2, 2, 2, 2), (3, 3, 3, 3), (2, 3, 2, 3), (2, 3, 3, 3),
                                             (4, 3, 3, 3), (3, 2, 3, 3), (6, 3, 6, 3), (2, 3, 4, 3),
                                             (1, 3, 3, 3), (3, 3, 1, 3)])
def test_1d_exact_all_lengths(m_o, r_o, m_i, r_i):
    rng = np.random.default_rng(m_o * 100 + m_i)
    for R in range(1, r_i * r_o + 1):
        x = [Fraction(int(v)) for v in rng.integers(-9, 10, size=40)]
        w = [Fraction(int(v)) for v in rng.integers(-9, 10, size=R)]
        assert nested_conv1d(x, w, m_o, m_i, r_o=r_o, r_i=r_i) == correlate_valid_1d(x, w)


def test_coverage_holes_for_mi_below_r():
    # positions r*t + s leave holes at 2, 5 for F(2,3) (x) F(2,3) (R6)
    ax = Axis(2, 3, 2, 3)
    assert sorted(set(ax.positions())) == [0, 1, 3, 4]
    assert ax.shifts == [0, 2] and ax.adv == 6
    covered = set()
    for ph, sh in enumerate(ax.shifts):
        for q, keep in enumerate(ax.keep(ph)):
            if keep:
                p = sh + ax.positions()[q]
                assert p not in covered
                covered.add(p)
    assert covered == set(range(6))


@pytest.mark.parametrize("K,pad,m_o,m_i,r_o", [(9, 4, 3, 3, 3), (5, 2, 3, 3, 3), (7, 3, 3, 3, 3),
                                               (5, 2, 2, 2, 3), (3, 1, 3, 3, 3), (9, 0, 2, 3, 3),
                                               (5, 2, 3, 3, 2), (4, 1, 3, 3, 2), (8, 3, 4, 3, 3)])
def test_2d_exact_equals_direct(K, pad, m_o, m_i, r_o):
    x = _ints((1, 2, 13, 11), K)
    w = _ints((2, 2, K, K), K + 1)
    cnt = Counter()
    y = nested_conv2d(x, w, pad, m_o, m_i, r_o=r_o, counter=cnt)
    ref = direct.conv2d(x.astype(np.float64), w.astype(np.float64), 1, pad)
    assert y.shape == ref.shape
    assert all(v == int(r) for v, r in zip(y.ravel(), ref.ravel()))
    ax = Axis(m_o, r_o, m_i)
    Ho, Wo = ref.shape[2:]
    slices = -(-Ho // ax.adv) * -(-Wo // ax.adv) * len(ax.shifts) ** 2
    # l^n multiplications per slice per (cin, cout), n = 4 axes here
    assert cnt.mults == slices * (ax.l_o * ax.l_i) ** 2 * 2 * 2


@pytest.mark.parametrize("K,m_o,m_i,r_o", [(9, 3, 3, 3), (5, 2, 2, 3), (5, 3, 3, 2), (7, 3, 3, 3)])
def test_composite_tables_reproduce_direct(K, m_o, m_i, r_o):
    # the integer/rational plan tables alone (what the library must match bit-exactly)
    tabs = plan_tables(K, 1, m_o, m_i, 2, 3, outer_taps=r_o)
    x = _ints((1, 2, 12, 14), 7)
    w = _ints((3, 2, K, K), 8)
    pad = K // 2
    y = composite_conv2d(x, w, pad, tabs)
    ref = direct.conv2d(x.astype(np.float64), w.astype(np.float64), 1, pad)
    assert all(v == int(r) for v, r in zip(y.ravel(), ref.ravel()))


def test_composite_shapes_33():
    ax = Axis(3, 3, 3, 3)
    BT, G, AT, gather = composite(ax)
    assert (len(BT), len(BT[0])) == (25, 17)
    assert (len(G), len(G[0])) == (25, 9)
    assert (len(AT), len(AT[0])) == (9, 25)
    assert gather == [3 * j + s for j in range(5) for s in range(5)]
    tabs = plan_tables(9, 1, 3, 3, 64, 64, pad=4)
    assert tabs[TABLE_DIMS][8:12] == [25, 17, 9, 625]


def test_float_path_close_to_exact():
    rng = np.random.default_rng(11)
    x = rng.standard_normal((1, 3, 10, 10))
    w = rng.standard_normal((2, 3, 9, 9))
    y = nested_conv2d(x, w, 4, 3, 3, exact=False)
    ref = direct.conv2d(x, w, 1, 4)
    assert np.max(np.abs(y - ref)) / np.max(np.abs(ref)) < 1e-12
