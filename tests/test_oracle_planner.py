"""Pins for oracle.planner (section IV.B decomposition algorithm)."""
import json
import os
import random
from fractions import Fraction

import pytest

from oracle import planner
from oracle.fig7 import KERNELS

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _direct1(x, w, S):
    R = len(w)
    return [sum(Fraction(x[S * i + k]) * w[k] for k in range(R)) for i in range((len(x) - R) // S + 1)]


def test_eq4_1_tree_lengths_and_rpn():
    g = json.load(open(os.path.join(GOLD, "eq4_1_rpn.json")))
    p = planner.plan(g["R"], g["S"], g["m"], g["r"])
    assert planner.rpn_text(p) == g["rpn"]
    assert p.M == g["M"]
    # the nested term carries the 3-tap phase, the leaf the 2-tap phase (Eq. 2.7: 5 = 2*2 + 1)
    assert isinstance(p.terms[0], planner.Nest) and p.terms[0].taps == 3
    assert isinstance(p.terms[1], planner.Repeat) and p.terms[1].child.taps == 2


def test_eq4_1_fig6_example_executes():
    # "decomposing and accelerating a 5x5 stride-2 convolution by F(m=2, r=2)" -- 2-D, exact
    rng = random.Random(5)
    p = planner.plan(5, 2, 2, 2)
    x = [[rng.randint(-3, 3) for _ in range(17)] for _ in range(15)]
    w = [[rng.randint(-3, 3) for _ in range(5)] for _ in range(5)]
    y = planner.execute_plan2d(p, x, w, 2)
    ref = [[sum(x[2 * i + a][2 * j + b] * w[a][b] for a in range(5) for b in range(5))
            for j in range((17 - 5) // 2 + 1)] for i in range((15 - 5) // 2 + 1)]
    assert y == ref


@pytest.mark.parametrize("m,r", KERNELS)
@pytest.mark.parametrize("S", [1, 2, 3])
def test_execute_equals_direct_every_R(m, r, S):
    # every (R, S) in {3..12} x {1..3} and each kernel equals the direct conv (here exact)
    rng = random.Random(100 * m + 10 * r + S)
    for R in range(1, 13):
        p = planner.plan(R, S, m, r)
        w = [Fraction(rng.randint(-4, 4), rng.randint(1, 3)) for _ in range(R)]
        x = [rng.randint(-5, 5) for _ in range(R + S * (2 * p.M + 3))]
        assert planner.execute_plan(p, x, w, S) == _direct1(x, w, S), (R, S, m, r, planner.rpn_text(p))


@pytest.mark.parametrize("R,S,m,r", [(9, 3, 3, 3), (7, 2, 3, 3), (10, 1, 2, 2), (11, 2, 4, 4)])
def test_execute_2d_sample(R, S, m, r):
    rng = random.Random(R * S)
    p = planner.plan(R, S, m, r)
    n = (R + S * (p.M + 2))
    x = [[rng.randint(-2, 2) for _ in range(n + 1)] for _ in range(n)]
    w = [[rng.randint(-2, 2) for _ in range(R)] for _ in range(R)]
    y = planner.execute_plan2d(p, x, w, S)
    ref = [[sum(x[S * i + a][S * j + b] * w[a][b] for a in range(R) for b in range(R))
            for j in range((n + 1 - R) // S + 1)] for i in range((n - R) // S + 1)]
    assert y == ref


def test_sum_terms_equal_length_and_lcm():
    for (m, r) in KERNELS:
        for R in range(1, 13):
            for S in (1, 2, 3):
                p = planner.plan(R, S, m, r)
                if isinstance(p, planner.Sum):
                    assert len({t.M for t in p.terms}) == 1 and p.terms[0].M == p.M
                    for t in p.terms:
                        base = t.child.M if isinstance(t, planner.Repeat) else t.M
                        assert p.M % base == 0


def test_rpn_round_trip_and_malformed():
    for (m, r) in KERNELS:
        for R in range(1, 13):
            for S in (1, 2, 3):
                p = planner.plan(R, S, m, r)
                q = planner.parse_rpn(planner.rpn_text(p))
                assert planner.shape(q) == planner.shape(p)
    for bad in ["SUM2 K2,2", "K2,2 K2,2", "NEST2", "K2,2 SUM2", "REP2", "K2,2 X"]:
        with pytest.raises(ValueError):
            planner.parse_rpn(bad)


def test_degenerate_and_depth():
    assert planner.rpn_text(planner.plan(3, 1, 3, 3)) == "K3,3"             # R <= r: the kernel
    assert planner.rpn_text(planner.plan(10, 1, 2, 2)) == "K2,2 NEST4"      # 2^3 < 10 <= 2^4
    assert planner.rpn_text(planner.plan(12, 1, 3, 3)) == "K3,3 NEST3"      # depth-3 nesting, K > 9
    assert planner.plan(9, 1, 3, 3).M == 9 and planner.plan(27, 1, 3, 3).M == 27
    assert planner.rpn_text(planner.plan(9, 3, 3, 3)) == "K3,3 K3,3 K3,3 SUM3"  # stride 3: 3 x 3 taps


def test_multiplication_count_of_a_plan():
    # Eq. 4.1 with F(2,2) per axis: nested term 9 products / 4 outputs, leaf 2 x 3 products / 4 outputs
    p = planner.plan(5, 2, 2, 2)
    cnt = planner.Counter()
    x = list(range(4 * 2 + 5 + 40))
    planner.execute_plan(p, x, [1, 2, 3, 4, 5], 2, cnt)
    tiles = -(-((len(x) - 5) // 2 + 1) // p.M)
    assert cnt.mults == tiles * (9 + 2 * 3)
