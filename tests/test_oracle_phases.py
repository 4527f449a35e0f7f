"""Pins for oracle.phases (Eq. 2.7 and the transposed-conv output phases)."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import direct
from oracle.nested import phase_taps
from oracle.phases import (conv_transpose2d_phases, decompose, stride2_conv2d_direct_phases,
                           stride2_conv2d_nested, stride_phase_lengths)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_eq4_1_plan_shape():
    g = json.load(open(os.path.join(GOLD, "eq4_1_plan.json")))
    assert stride_phase_lengths(g["R"], g["S"]) == [tuple(v) for v in g["phase_lengths"]]

    def tolist(t):
        return [tolist(v) if isinstance(v, (tuple, list)) else v for v in t]
    assert tolist(decompose(g["R"], g["S"], g["r"])) == g["tree"]


@pytest.mark.parametrize("K,pad", [(7, 3), (9, 4), (5, 2), (3, 1)])
def test_stride2_polyphase_direct(K, pad):
    rng = np.random.default_rng(K)
    x = rng.standard_normal((2, 3, 21, 18))
    w = rng.standard_normal((4, 3, K, K))
    ref = torch.nn.functional.conv2d(torch.from_numpy(x), torch.from_numpy(w), stride=2, padding=pad).numpy()
    np.testing.assert_allclose(stride2_conv2d_direct_phases(x, w, pad), ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("K,pad", [(7, 3), (9, 4)])
def test_stride2_nested_exact(K, pad):
    rng = np.random.default_rng(K + 1)
    x = rng.integers(-3, 4, size=(1, 2, 15, 14)).astype(object)
    w = rng.integers(-3, 4, size=(2, 2, K, K)).astype(object)
    y = stride2_conv2d_nested(x, w, pad)
    ref = direct.conv2d(x.astype(np.float64), w.astype(np.float64), 2, pad)
    assert y.shape == ref.shape
    assert all(v == int(r) for v, r in zip(y.ravel(), ref.ravel()))


def test_transposed_taps_k9():
    t = phase_taps(9, 2, True, 4)
    assert t[:3] == [2, 2, 5]
    assert t[3] == 2 and t[4:9] == [8, 6, 4, 2, 0]
    assert t[9] == 2 and t[10:15] == [-1, 7, 5, 3, 1]


@pytest.mark.parametrize("K,pad,op", [(9, 4, 1), (5, 2, 1), (3, 1, 1)])
def test_transposed_phases_vs_torch(K, pad, op):
    rng = np.random.default_rng(K)
    x = rng.standard_normal((2, 3, 9, 7))
    w = rng.standard_normal((3, 2, K, K))
    ref = torch.nn.functional.conv_transpose2d(torch.from_numpy(x), torch.from_numpy(w), stride=2,
                                               padding=pad, output_padding=op).numpy()
    np.testing.assert_allclose(conv_transpose2d_phases(x, w, pad, op), ref, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(direct.conv_transpose2d(x, w, 2, pad, op), ref, rtol=1e-12, atol=1e-12)


def test_transposed_nested_exact():
    rng = np.random.default_rng(3)
    x = rng.integers(-3, 4, size=(1, 2, 6, 5)).astype(object)
    w = rng.integers(-3, 4, size=(2, 1, 9, 9)).astype(object)
    y = conv_transpose2d_phases(x, w, 4, 1, nested=True, exact=True)
    ref = direct.conv_transpose2d(x.astype(np.float64), w.astype(np.float64), 2, 4, 1)
    assert y.shape == ref.shape
    assert all(v == int(r) for v, r in zip(y.ravel(), ref.ravel()))
