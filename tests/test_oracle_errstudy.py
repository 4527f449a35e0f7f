import numpy as np
import torch

from oracle.errstudy import rel_err, round_bf16, round_tf32, split_bf16


def test_bf16_matches_torch():
    a = np.random.default_rng(0).standard_normal(100000).astype(np.float32) * 1e3
    ref = torch.from_numpy(a).to(torch.bfloat16).to(torch.float32).numpy()
    np.testing.assert_array_equal(round_bf16(a), ref)


def test_tf32_mantissa_and_ties():
    a = np.array([1.0 + 2.0 ** -11, 1.0 + 2.0 ** -10 + 2.0 ** -11], dtype=np.float32)
    r = round_tf32(a)
    assert r[0] == np.float32(1.0 + 2.0 ** -10)          # tie rounds away from zero
    assert r[1] == np.float32(1.0 + 2.0 ** -9)
    b = np.random.default_rng(1).standard_normal(1000).astype(np.float32)
    assert np.all(np.abs(round_tf32(b) - b) <= np.abs(b) * 2.0 ** -11)


def test_split_reconstructs():
    a = np.random.default_rng(2).standard_normal(10000).astype(np.float32)
    hi, lo = split_bf16(a)
    assert np.all(np.abs((hi.astype(np.float64) + lo) - a) <= np.abs(a) * 2.0 ** -16)
    assert rel_err([1.0, 2.0], [1.0, 2.0]) == 0.0


def test_rel_err_hand_computed():
    # max|y - ref| / max|ref|: |diffs| = (0, 0.5, 1), max|ref| = 4 -> 0.25 (R14)
    assert rel_err([1.0, 2.5, -3.0], [1.0, 2.0, -4.0]) == 0.25
    # the denominator is the max over the reference, not over y, and signs count
    assert rel_err([-1.0, -2.0], [1.0, 2.0]) == 2.0
    assert rel_err(np.zeros((2, 3)), np.full((2, 3), -0.5)) == 1.0
    # 2-D / 4-D inputs reduce over every element
    y = np.zeros((2, 2, 2, 2)); r = np.ones((2, 2, 2, 2)); y[1, 0, 1, 1] = 1.75; r[0, 1, 0, 0] = 8.0
    assert rel_err(y, r) == 8.0 / 8.0
