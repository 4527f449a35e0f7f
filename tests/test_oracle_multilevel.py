"""Pins for oracle.multilevel (nesting to any depth) -- exact, brute force."""
import random
from fractions import Fraction

import pytest

from oracle.multilevel import Counter, conv1d, depth_for, leaf, levels, nest
from oracle.nested import Axis, composite


def _direct(x, w):
    return [sum(Fraction(x[i + k]) * w[k] for k in range(len(w))) for i in range(len(x) - len(w) + 1)]


@pytest.mark.parametrize("m_o,r_o,m_i", [(3, 3, 3), (4, 3, 3), (2, 3, 3), (4, 2, 3), (2, 2, 3)])
def test_two_levels_equal_oracle_nested_composite(m_o, r_o, m_i):
    # the recursive composite reproduces the two-level matrices of oracle.nested exactly
    ax = Axis(m_o, r_o, m_i, 3)
    BT, G, AT, gather = composite(ax)
    a = nest(m_o, r_o, leaf(m_i, 3))
    assert a.BT == BT and a.G == G and a.AT == AT
    assert a.L == ax.L and a.R == ax.reach
    assert a.pos == ax.positions()


@pytest.mark.parametrize("m,r,d", [(2, 2, 1), (2, 2, 2), (2, 2, 3), (2, 2, 4), (3, 3, 2), (3, 3, 3),
                                   (4, 4, 2), (6, 3, 2), (6, 3, 3), (3, 2, 3)])
def test_depth_d_equals_direct_exactly(m, r, d):
    rng = random.Random(m * 100 + r * 10 + d)
    a = levels(m, r, d)
    for R in sorted({a.R, max(1, a.R - 1), r ** (d - 1) + 1 if d > 1 else r}):
        w = [Fraction(rng.randint(-4, 4), rng.randint(1, 3)) for _ in range(R)]
        x = [Fraction(rng.randint(-5, 5)) for _ in range(R + 3 * a.advance() + 2)]
        cnt = Counter()
        assert conv1d(x, w, a, cnt) == _direct(x, w)
        slices = -(-(len(x) - R + 1) // a.advance())
        assert cnt.mults == slices * (m + r - 1) ** d          # l^d per slice


@pytest.mark.parametrize("m,r", [(2, 2), (3, 3), (4, 4), (6, 3), (5, 3)])
def test_distinct_output_recursion(m, r):
    # O_1 = m, O_j = (m - 1) r^(j-1) + O_(j-1) for m >= r (contiguous)
    O = m
    for d in range(1, 5 if m <= 4 else 4):
        if d > 1:
            O = (m - 1) * r ** (d - 1) + O
        a = levels(m, r, d)
        assert a.advance() == O
        assert a.L == r ** d + O - 1                          # window = reach + outputs - 1
        assert a.P == (m + r - 1) ** d


def test_fig3_worked_example_window():
    # P:108 / Fig. 3: F(2,2) at both levels -> window L = r(l-1) + l = 2*2 + 3 = 7, 9 products, 4 outputs
    a = levels(2, 2, 2)
    assert (a.L, a.P, a.advance(), a.R) == (7, 9, 4, 4)


def test_depth_for():
    assert [depth_for(R, 3) for R in (1, 3, 4, 9, 10, 27, 28)] == [1, 1, 2, 2, 3, 3, 4]
    assert [depth_for(R, 2) for R in (2, 3, 4, 5, 8, 9, 12)] == [1, 2, 2, 3, 3, 4, 4]
