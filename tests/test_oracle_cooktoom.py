"""Pins for oracle.cooktoom (exact Cook-Toom F(m, r))."""
import json
import os
from fractions import Fraction

import pytest

from oracle.cooktoom import (apply_1d, correlate_valid_1d, generate_kernel, make_points,
                             verify_kernel, INF)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_correlate_reference_examples():
    # SPEC S:204 (delta filter) -- pins the brute-force correlation itself
    assert correlate_valid_1d([1, 2, 3, 4], [1, 0]) == [1, 2, 3]
    assert correlate_valid_1d([1, 2, 3, 4], [0, 1]) == [2, 3, 4]
    assert correlate_valid_1d([1, 1, 1], [2, 3]) == [5, 5]


def test_points_order():
    assert make_points(1) == [0]
    assert make_points(4) == [0, 1, -1, INF]
    assert make_points(6) == [0, 1, -1, 2, -2, INF]
    assert make_points(8)[:7] == [0, 1, -1, 2, -2, Fraction(1, 2), Fraction(-1, 2)]


@pytest.mark.parametrize("m", range(1, 7))
@pytest.mark.parametrize("r", range(1, 7))
def test_exact_identity_all_small_kernels(m, r):
    if m + r - 1 > 9:
        pytest.skip("l > 9 outside the supported set")
    k = generate_kernel(m, r)
    assert k.l == m + r - 1
    assert verify_kernel(k, trials=30, seed=m * 10 + r)


def test_perturbed_kernel_fails():
    k = generate_kernel(2, 3)
    k.G[1][0] += Fraction(1, 1000)
    assert not verify_kernel(k, trials=10)


def test_lavin_gray_f23_up_to_infinity_sign():
    g = json.load(open(os.path.join(GOLD, "lavin_gray_f23.json")))
    k = generate_kernel(2, 3)
    BT = [row[:] for row in k.BT]
    AT = [row[:] for row in k.AT]
    BT[-1] = [-v for v in BT[-1]]
    for row in AT:
        row[-1] = -row[-1]
    assert BT == [[Fraction(v) for v in row] for row in g["BT"]]
    assert AT == [[Fraction(v) for v in row] for row in g["AT"]]
    assert k.G == [[Fraction(v) for v in row] for row in g["G"]]


@pytest.mark.parametrize("r", [1, 2, 3, 5])
def test_f1r_is_native(r):
    # with no overlap (F(1, r)) Winograd converges to the native convolution
    k = generate_kernel(1, r)
    x = [Fraction(i * 7 - 3, 5) for i in range(r)]
    w = [Fraction(11 - 2 * i, 3) for i in range(r)]
    assert apply_1d(k, x, w) == [sum(a * b for a, b in zip(x, w))]


def test_multiplication_count_below_native():
    for m in range(2, 7):
        for r in range(2, 7):
            if m + r - 1 <= 9:
                assert m + r - 1 < m * r


def test_integer_B_and_A_for_integer_points():
    # DESIGN.md#R3: B and A are integer, the fractions live in G
    for (m, r) in [(2, 3), (3, 3), (3, 2), (2, 2), (4, 3)]:
        k = generate_kernel(m, r)
        assert all(v.denominator == 1 for row in k.BT for v in row)
        assert all(v.denominator == 1 for row in k.AT for v in row)
