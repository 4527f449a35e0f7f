"""Pins for oracle.ola (Eq. 2.3)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import direct
from oracle.cooktoom import correlate_valid_1d
from oracle.nested import Counter, nested_conv1d
from oracle.ola import ola_conv1d, ola_conv2d

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_eq2_3_worked_example():
    g = json.load(open(os.path.join(GOLD, "eq2_3_ola_f22.json")))
    x = [Fraction(v) for v in [1, -2, 3, 5, -7, 2, 4]]
    w = [Fraction(v) for v in [3, 1, -1, 2]]
    cnt, trace = Counter(), []
    y = ola_conv1d(x, w, g["m"], g["r"], counter=cnt, trace=trace)
    assert y == correlate_valid_1d(x, w)
    offs = g["subvector_offsets"]
    assert trace == [(o, b, offs[name]) for o, b, name in g["ola_terms"]]
    assert cnt.mults == g["ola_multiplications"]
    cn = Counter()
    assert nested_conv1d(x, w, 2, 2, r_i=2, counter=cn) == y
    assert cn.mults == g["nested_multiplications"]


@pytest.mark.parametrize("R,m,r", [(9, 3, 3), (5, 3, 3), (7, 2, 3), (4, 2, 2), (3, 3, 3)])
def test_1d_exact(R, m, r):
    rng = np.random.default_rng(R * 10 + m)
    x = [Fraction(int(v)) for v in rng.integers(-9, 10, size=31)]
    w = [Fraction(int(v)) for v in rng.integers(-9, 10, size=R)]
    assert ola_conv1d(x, w, m, r) == correlate_valid_1d(x, w)


@pytest.mark.parametrize("K,pad,m", [(9, 4, 3), (5, 2, 3), (7, 3, 2)])
def test_2d_exact_equals_direct(K, pad, m):
    rng = np.random.default_rng(K)
    x = rng.integers(-4, 5, size=(1, 2, 11, 10)).astype(object)
    w = rng.integers(-4, 5, size=(2, 2, K, K)).astype(object)
    cnt = Counter()
    y = ola_conv2d(x, w, pad, m, counter=cnt)
    ref = direct.conv2d(x.astype(np.float64), w.astype(np.float64), 1, pad)
    assert all(v == int(r) for v, r in zip(y.ravel(), ref.ravel()))
    Ho, Wo = ref.shape[2:]
    nb = -(-K // 3)
    assert cnt.mults == (-(-Ho // m)) * (-(-Wo // m)) * nb * nb * (m + 2) ** 2 * 4
