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
