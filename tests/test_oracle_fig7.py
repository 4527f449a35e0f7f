"""Pins for the Fig. 7 sweep (oracle.fig7) and its committed artefact."""
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import counts, fig7
from oracle.multilevel import Counter, conv1d, depth_for, levels
from oracle.nested import Counter as NCounter
from oracle.ola import ola_conv2d

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows():
    return {(c["method"], c["filter_side"], c["kernel_m"], c["kernel_r"]): c for c in fig7.sweep()}


def test_table_shape_and_artefact_reproduces():
    rows = fig7.sweep()
    assert len(rows) == 10 * 4 * 3
    # tests/golden/fig7_sweep.csv is written by tools/make_fig7.py, which calls oracle.fig7 only
    with open(os.path.join(GOLD, "fig7_sweep.csv")) as f:
        assert f.read() == fig7.to_csv(rows)


def test_small_filters_degenerate():
    # R <= r: one kernel application; nested and OLA coincide with the kernel itself
    t = _rows()
    for (m, r) in fig7.KERNELS:
        for R in range(3, r + 1):
            n, o = t[("nested", R, m, r)], t[("ola", R, m, r)]
            assert n["mults_per_output"] == o["mults_per_output"] == Fraction((m + r - 1) ** 2, m * m)


def test_closed_forms_match_oracle_counts():
    t = _rows()
    for (m, r) in fig7.KERNELS:
        for R in fig7.SIDES:
            assert t[("ola", R, m, r)]["mults_per_output"] == counts.per_output_2d(counts.ola_per_axis(R, m, r))
            assert t[("direct", R, m, r)]["mults_per_output"] == \
                counts.per_output_2d(counts.direct_winograd_per_axis(R, m))
            assert t[("nested", R, m, r)]["mults_per_output"] == \
                counts.per_output_2d(counts.nested_same_kernel_per_axis(R, m, r))


@pytest.mark.parametrize("R,m,r", [(5, 2, 2), (9, 3, 3), (7, 4, 4), (12, 3, 3), (10, 6, 3), (11, 2, 2)])
def test_nested_cell_equals_instrumented_counter(R, m, r):
    # per axis: the exact evaluator's EWMM count over whole slices; 2-D = square (separable)
    rng = np.random.default_rng(R)
    a = levels(m, r, depth_for(R, r))
    w = [int(v) for v in rng.integers(-3, 4, R)]
    n_slices = 3
    x = [int(v) for v in rng.integers(-3, 4, R - 1 + n_slices * a.advance())]
    cnt = Counter()
    y = conv1d(x, w, a, cnt)
    assert y == [sum(x[i + k] * w[k] for k in range(R)) for i in range(len(x) - R + 1)]
    per_axis = Fraction(cnt.mults, n_slices * a.advance())
    c = _rows()[("nested", R, m, r)]
    assert per_axis * per_axis == c["mults_per_output"]


@pytest.mark.parametrize("R", [5, 7])
def test_ola_cell_equals_instrumented_counter(R):
    rng = np.random.default_rng(R)
    x = rng.integers(-2, 3, size=(1, 1, 12, 12)).astype(object)
    w = rng.integers(-2, 3, size=(1, 1, R, R)).astype(object)
    cnt = NCounter()
    ola_conv2d(x, w, 0, 3, counter=cnt)
    Ho = 12 - R + 1
    tiles = (-(-Ho // 3)) ** 2
    c = _rows()[("ola", R, 3, 3)]
    assert cnt.mults == tiles * c["mults_per_tile"]


def test_paper_claims_p146_148():
    t = _rows()
    mpo = lambda meth, R, k: t[(meth, R) + k]["mults_per_output"]
    for k in [(2, 2), (3, 3)]:
        gaps = [mpo("ola", R, k) - mpo("nested", R, k) for R in fig7.SIDES if R > k[1]]
        assert all(g >= 0 for g in gaps)                       # "fewer multiplications ... in most cases"
        assert gaps[-1] > gaps[0]                              # "the gap increases when the filter size gets larger"
    # F(6,3) on 5x5: nested is not better than OLA, and direct Winograd is the cheapest of the three
    assert mpo("nested", 5, (6, 3)) >= mpo("ola", 5, (6, 3))
    assert mpo("direct", 5, (6, 3)) < min(mpo("ola", 5, (6, 3)), mpo("nested", 5, (6, 3)))
    # Table I's analytic ratios (F(3,3)): 1.44 at 5x5, 3.24 at 9x9
    assert mpo("ola", 5, (3, 3)) / mpo("nested", 5, (3, 3)) == Fraction(144, 100)
    assert mpo("ola", 9, (3, 3)) / mpo("nested", 9, (3, 3)) == Fraction(324, 100)
