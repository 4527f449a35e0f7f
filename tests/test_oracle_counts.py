"""Pins for oracle.counts: closed forms vs the paper and vs the instrumented evaluators."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import counts
from oracle.nested import Counter, nested_conv2d
from oracle.ola import ola_conv2d

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_eq2_3_counts():
    # OLA 4 x F(2,2) = 12 multiplications vs nesting 3 x F(2,2) = 9, for 4 outputs
    assert counts.ola_per_axis(4, 2, 2) * 4 == 12
    assert counts.nested_per_axis(2, 2, 2, 2) * 4 == 9


def test_table1_ratios_within_3pct():
    g = json.load(open(os.path.join(GOLD, "table1_gops.json")))
    nested = counts.per_output_2d(counts.nested_per_axis(3, 3, 3, 3))
    assert nested == Fraction(625, 81)
    for row in g["rows"]:
        if row["type"] != "conv2d":
            continue  # depthwise 7x7: hardware-bound measurement (R16)
        K = row["K"]
        ola = counts.per_output_2d(counts.ola_per_axis(K, 3, 3))
        analytic = float(ola / nested)
        measured = row["gops_nested"] / row["gops_ola"]
        assert abs(measured - row["speedup"]) < 0.01
        assert abs(analytic - measured) / measured < g["tolerance_rel"]
    assert counts.per_output_2d(counts.ola_per_axis(5, 3, 3)) / nested == Fraction(144, 100)
    assert counts.per_output_2d(counts.ola_per_axis(9, 3, 3)) / nested == Fraction(324, 100)


def test_nested_beats_ola_and_direct_winograd_cell():
    # nested uses fewer multiplications than OLA "in most of the cases";
    # for F(2,2) and F(3,3) every R > r qualifies
    for (m, r) in [(2, 2), (3, 3)]:
        gaps = []
        for R in range(r + 1, 13):
            n = counts.nested_same_kernel_per_axis(R, m, r)
            o = counts.ola_per_axis(R, m, r)
            assert n <= o
            gaps.append(counts.per_output_2d(o) - counts.per_output_2d(n))
        assert gaps[-1] > gaps[0]    # "the gap increases when the filter size gets larger"
    # "direct Winograd algorithm has the highest efficiency in such case" (F(6,3), 5x5)
    dw = counts.direct_winograd_per_axis(5, 6)
    assert dw < counts.ola_per_axis(5, 6, 3) and dw < counts.nested_same_kernel_per_axis(5, 6, 3)


def test_f63_5x5_unpinned_values_recorded():
    # parity unpinned (R17): paper says +2.2%; conventions here give +30.6% / 0%
    same = counts.per_output_2d(counts.nested_same_kernel_per_axis(5, 6, 3))
    mixed = counts.per_output_2d(counts.nested_per_axis(6, 2, 6, 3))
    ola = counts.per_output_2d(counts.ola_per_axis(5, 6, 3))
    assert round(float(same / ola - 1), 3) == 0.306
    assert mixed == ola


@pytest.mark.parametrize("K,m_o,m_i", [(9, 3, 3), (5, 2, 2), (7, 3, 3)])
def test_counter_equals_closed_form(K, m_o, m_i):
    rng = np.random.default_rng(1)
    x = rng.integers(-2, 3, size=(1, 2, 10, 12)).astype(object)
    w = rng.integers(-2, 3, size=(3, 2, K, K)).astype(object)
    pad = K // 2
    cnt = Counter()
    nested_conv2d(x, w, pad, m_o, m_i, counter=cnt)
    assert cnt.mults == counts.layer_ewmm_nested(1, 10, 12, 2, 3, m_o, 3, m_i)
    c2 = Counter()
    ola_conv2d(x, w, pad, 3, counter=c2)
    assert c2.mults == counts.layer_ewmm_ola(1, 10, 12, 2, 3, K, 3)


def test_f23_both_levels_28_4_per_output():
    assert round(float(counts.per_output_2d(counts.nested_per_axis(2, 3, 2, 3))), 1) == 28.4
