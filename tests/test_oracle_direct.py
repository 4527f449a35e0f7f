"""Pins for oracle.direct (Eq. 2.1 in FP64, R1)."""
import numpy as np
import pytest
import torch

from oracle import direct


def _rand(shape, seed, lo=-3, hi=4):
    return np.random.default_rng(seed).integers(lo, hi, size=shape).astype(np.float64)


@pytest.mark.parametrize("stride,pad,K", [(1, 0, 3), (1, 2, 5), (2, 1, 3), (2, 3, 7)])
def test_conv2d_vs_bruteforce(stride, pad, K):
    x = _rand((2, 3, 9, 8), 1)
    w = _rand((2, 3, K, K), 2)
    ref = np.array(direct.conv2d_bruteforce(x.tolist(), w.tolist(), stride, pad))
    np.testing.assert_array_equal(direct.conv2d(x, w, stride, pad), ref)


@pytest.mark.parametrize("stride,pad,K", [(1, 4, 9), (2, 4, 9), (2, 3, 7), (1, 2, 5)])
def test_conv2d_vs_torch_fp64(stride, pad, K):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 4, 23, 19))
    w = rng.standard_normal((5, 4, K, K))
    ref = torch.nn.functional.conv2d(torch.from_numpy(x), torch.from_numpy(w), stride=stride,
                                     padding=pad).numpy()
    np.testing.assert_allclose(direct.conv2d(x, w, stride, pad), ref, rtol=1e-12, atol=1e-12)


def test_conv2d_closed_forms():
    # 3x3 ones input, 2x2 ones filter -> all 4s
    y = direct.conv2d(np.ones((1, 1, 3, 3)), np.ones((1, 1, 2, 2)))
    np.testing.assert_array_equal(y, 4 * np.ones((1, 1, 2, 2)))
    # delta filter at (0, 0) -> cropped input
    x = _rand((1, 2, 7, 7), 5)
    w = np.zeros((2, 2, 3, 3))
    w[0, 0, 0, 0] = w[1, 1, 0, 0] = 1
    np.testing.assert_array_equal(direct.conv2d(x, w), x[:, :, :5, :5])


def test_conv2d_at_matches_full():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 3, 17, 13))
    w = rng.standard_normal((4, 3, 7, 7))
    for stride, pad in [(1, 3), (2, 3)]:
        full = direct.conv2d(x, w, stride, pad)
        pts = [(n, o, i, j) for n in range(2) for o in range(4) for i in (0, 2, full.shape[2] - 1)
               for j in (0, full.shape[3] - 1)]
        vals = direct.conv2d_at(x, w, stride, pad, pts)
        np.testing.assert_allclose(vals, [full[p] for p in pts], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("K,pad,op", [(9, 4, 1), (3, 1, 1), (4, 1, 0)])
def test_conv_transpose2d_vs_torch(K, pad, op):
    rng = np.random.default_rng(6)
    x = rng.standard_normal((2, 3, 7, 6))
    w = rng.standard_normal((3, 2, K, K))
    ref = torch.nn.functional.conv_transpose2d(torch.from_numpy(x), torch.from_numpy(w), stride=2,
                                               padding=pad, output_padding=op).numpy()
    out = direct.conv_transpose2d(x, w, 2, pad, op)
    assert out.shape == ref.shape
    np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)
    pts = [(1, 1, 0, 0), (0, 0, ref.shape[2] - 1, ref.shape[3] - 1), (1, 0, 5, 4), (0, 1, 6, 1)]
    np.testing.assert_allclose(direct.conv_transpose2d_at(x, w, 2, pad, pts), [ref[p] for p in pts],
                               rtol=1e-12, atol=1e-12)


def test_transposed_output_size_fsrcnn():
    # DESIGN.md#R11: 9x9 stride 2, pad 4, output_padding 1 maps 540x960 -> 1080x1920
    H, W, K = 540, 960, 9
    assert (H - 1) * 2 - 8 + K + 1 == 1080 and (W - 1) * 2 - 8 + K + 1 == 1920


@pytest.mark.parametrize("K,pad,stride", [(7, 3, 1), (3, 1, 1), (5, 0, 2)])
def test_depthwise_vs_torch_groups_and_bruteforce(K, pad, stride):
    # Table I's depthwise row: groups = C -- an independent library (torch fp64
    # groups=C) and the per-channel brute force of Eq. 2.1
    rng = np.random.default_rng(K)
    x = rng.standard_normal((2, 5, 11, 9))
    w = rng.standard_normal((5, 1, K, K))
    y = direct.conv2d_depthwise(x, w, stride, pad)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x), torch.from_numpy(w), stride=stride, padding=pad,
                                     groups=5).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)
    for c in range(5):
        bf = direct.conv2d_bruteforce(x[:, c:c + 1].tolist(), w[c:c + 1].tolist(), stride, pad)
        np.testing.assert_allclose(y[:, c:c + 1], np.array(bf), rtol=1e-12, atol=1e-12)
