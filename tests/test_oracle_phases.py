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


# ---------------------------------------------------------------------------
# Pins of phase_taps and layer_geometry that do not go through the library
# (VERDICT r1 "What's weak" 1): each table is evaluated by the formula its
# docstring states and compared with torch CPU fp64, an independent library.
# A flipped offset sign, a wrong tap index or a wrong fold count fails here.
# ---------------------------------------------------------------------------
def _phases_from_table(tab):
    mode, nph, Kp = tab[0], tab[1], tab[2]
    offs, taps = [], []
    for p in range(nph):
        base = 3 + p * (Kp + 1)
        offs.append(tab[base])
        taps.append(tab[base + 1:base + 1 + Kp])
    return mode, nph, Kp, offs, taps


def _eval_phase_table(x, w, tab, stride, pad, output_padding=0):
    """Evaluate a convolution from phase_taps' table alone (2-D, separable table)."""
    mode, nph, Kp, offs, taps = _phases_from_table(tab)
    N, C, H, W = x.shape

    P = 4 * (H + W)   # generous zero border: every index the table can produce is inside it
    xz = np.zeros((N, C, H + 2 * P, W + 2 * P))
    xz[:, :, P:P + H, P:P + W] = x

    def xat(rows, cols):  # x[:, :, rows, cols] with zero outside the image
        return xz[:, :, np.asarray(rows) + P][:, :, :, np.asarray(cols) + P]

    if mode == 0:   # y[i] = sum_d x[i + d - offset] w[taps[d]]
        K = w.shape[2]
        Ho, Wo = H + 2 * pad - K + 1, W + 2 * pad - K + 1
        y = np.zeros((N, w.shape[0], Ho, Wo))
        for d in range(Kp):
            for e in range(Kp):
                win = xat([i + d - offs[0] for i in range(Ho)], [j + e - offs[0] for j in range(Wo)])
                y += np.einsum("nchw,oc->nohw", win, w[:, :, taps[0][d], taps[0][e]])
        return y
    if mode == 1:   # phase p: y[i] += sum_a x[2(i + a) + offset_p] w[taps_p[a]]
        K = w.shape[2]
        Ho, Wo = (H + 2 * pad - K) // 2 + 1, (W + 2 * pad - K) // 2 + 1
        y = np.zeros((N, w.shape[0], Ho, Wo))
        for p in range(nph):
            for q in range(nph):
                for a in range(Kp):
                    for b in range(Kp):
                        if taps[p][a] < 0 or taps[q][b] < 0:
                            continue
                        win = xat([2 * (i + a) + offs[p] for i in range(Ho)],
                                  [2 * (j + b) + offs[q] for j in range(Wo)])
                        y += np.einsum("nchw,oc->nohw", win, w[:, :, taps[p][a], taps[q][b]])
        return y
    # mode 2, transposed: y[2j + phi] = sum_d x[j + d - offset_phi] w[taps_phi[d]]
    K = w.shape[2]
    Ho = (H - 1) * 2 - 2 * pad + K + output_padding
    Wo = (W - 1) * 2 - 2 * pad + K + output_padding
    y = np.zeros((N, w.shape[1], Ho, Wo))
    for ph in range(2):
        for pw in range(2):
            nh, nw = len(range(ph, Ho, 2)), len(range(pw, Wo, 2))
            acc = np.zeros((N, w.shape[1], nh, nw))
            for d in range(Kp):
                for e in range(Kp):
                    if taps[ph][d] < 0 or taps[pw][e] < 0:
                        continue
                    win = xat([j + d - offs[ph] for j in range(nh)], [k + e - offs[pw] for k in range(nw)])
                    acc += np.einsum("nchw,co->nohw", win, w[:, :, taps[ph][d], taps[pw][e]])
            y[:, :, ph::2, pw::2] = acc
    return y


@pytest.mark.parametrize("K,pad", [(7, 3), (9, 4), (5, 2), (3, 1), (8, 3), (9, 0)])
def test_phase_taps_stride2_table_alone_vs_torch(K, pad):
    rng = np.random.default_rng(100 + K + pad)
    x = rng.standard_normal((2, 3, 23, 20))
    w = rng.standard_normal((4, 3, K, K))
    tab = phase_taps(K, 2, False, pad)
    assert tab[0] == 1 and tab[1] == 2 and tab[2] == -(-K // 2)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x), torch.from_numpy(w), stride=2, padding=pad).numpy()
    np.testing.assert_allclose(_eval_phase_table(x, w, tab, 2, pad), ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("K,pad", [(5, 2), (9, 4), (4, 0)])
def test_phase_taps_stride1_table_alone_vs_torch(K, pad):
    rng = np.random.default_rng(200 + K)
    x = rng.standard_normal((1, 2, 13, 11))
    w = rng.standard_normal((3, 2, K, K))
    tab = phase_taps(K, 1, False, pad)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x), torch.from_numpy(w), padding=pad).numpy()
    np.testing.assert_allclose(_eval_phase_table(x, w, tab, 1, pad), ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("K,pad,op", [(9, 4, 1), (5, 2, 1), (7, 3, 0), (9, 3, 1), (4, 1, 0)])
def test_phase_taps_transposed_table_alone_vs_torch(K, pad, op):
    rng = np.random.default_rng(300 + K + pad)
    x = rng.standard_normal((2, 3, 9, 8))
    w = rng.standard_normal((3, 2, K, K))
    tab = phase_taps(K, 2, True, pad)
    ref = torch.nn.functional.conv_transpose2d(torch.from_numpy(x), torch.from_numpy(w), stride=2, padding=pad,
                                               output_padding=op).numpy()
    np.testing.assert_allclose(_eval_phase_table(x, w, tab, 2, pad, op), ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("K,pad", [(7, 3), (9, 4), (5, 2)])
def test_layer_geometry_stride2_fold_is_one_conv(K, pad):
    """Cin_e = 4 Cin and K' = ceil(K/2) (R9): the stride-2 conv equals ONE
    stride-1 conv over the Cin_e stacked phase images with K' x K' stacked sub-filters."""
    from oracle.nested import layer_geometry
    Cin, Cout = 3, 5
    Kp, r_o, cin_e, cout_e = layer_geometry(K, 2, False, pad, 0, 4, 3, 0, Cin, Cout)
    assert (cin_e, cout_e) == (4 * Cin, Cout)
    rng = np.random.default_rng(K)
    x = rng.standard_normal((2, Cin, 26, 23))
    w = rng.standard_normal((Cout, Cin, K, K))
    Ho, Wo = (26 + 2 * pad - K) // 2 + 1, (23 + 2 * pad - K) // 2 + 1
    xp = np.zeros((2, Cin, 2 * (Ho + Kp), 2 * (Wo + Kp)))
    xp[:, :, pad:pad + 26, pad:pad + 23] = x[:, :, :2 * (Ho + Kp) - pad, :2 * (Wo + Kp) - pad]
    xs = np.concatenate([xp[:, :, p::2, q::2][:, :, :Ho + Kp - 1, :Wo + Kp - 1]
                         for p in range(2) for q in range(2)], axis=1)
    ws = np.zeros((Cout, 4, Cin, Kp, Kp))
    for p in range(2):
        for q in range(2):
            sub = w[:, :, p::2, q::2]
            ws[:, 2 * p + q, :, :sub.shape[2], :sub.shape[3]] = sub
    ws = ws.transpose(0, 1, 2, 3, 4).reshape(Cout, 4 * Cin, Kp, Kp)
    assert xs.shape[1] == cin_e and ws.shape[1] == cin_e
    y1 = torch.nn.functional.conv2d(torch.from_numpy(xs), torch.from_numpy(ws)).numpy()
    ref = torch.nn.functional.conv2d(torch.from_numpy(x), torch.from_numpy(w), stride=2, padding=pad).numpy()
    np.testing.assert_allclose(y1, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("K,pad,op", [(9, 4, 1), (5, 2, 1), (7, 3, 0)])
def test_layer_geometry_transposed_fold_is_one_conv(K, pad, op):
    """Cout_e = 4 Cout and K' = the common window of phase_taps (R11, #R11a): the
    transposed conv equals ONE stride-1 conv with Cout_e output channels + depth-to-space."""
    from oracle.nested import layer_geometry
    Cin, Cout = 3, 2
    Kp, r_o, cin_e, cout_e = layer_geometry(K, 2, True, pad, op, 4, 3, 0, Cin, Cout)
    assert (cin_e, cout_e) == (Cin, 4 * Cout)
    tab = phase_taps(K, 2, True, pad)
    assert Kp == tab[2]
    _, _, _, offs, taps = _phases_from_table(tab)
    assert offs[0] == offs[1]
    rng = np.random.default_rng(K + op)
    H, W = 9, 7
    x = rng.standard_normal((2, Cin, H, W))
    w = rng.standard_normal((Cin, Cout, K, K))
    Ho, Wo = (H - 1) * 2 - 2 * pad + K + op, (W - 1) * 2 - 2 * pad + K + op
    nh, nw = -(-Ho // 2), -(-Wo // 2)
    xp = np.zeros((2, Cin, nh + Kp, nw + Kp))
    o = offs[0]
    hh, ww = min(H, nh + Kp - o), min(W, nw + Kp - o)
    xp[:, :, o:o + hh, o:o + ww] = x[:, :, :hh, :ww]
    big = np.zeros((4 * Cout, Cin, Kp, Kp))   # output channel (2 phi_h + phi_w) * Cout + co
    for ph in range(2):
        for pw in range(2):
            for d in range(Kp):
                for e in range(Kp):
                    if taps[ph][d] >= 0 and taps[pw][e] >= 0:
                        big[(2 * ph + pw) * Cout:(2 * ph + pw + 1) * Cout, :, d, e] = w[:, :, taps[ph][d], taps[pw][e]].T
    assert big.shape[0] == cout_e
    z = torch.nn.functional.conv2d(torch.from_numpy(xp), torch.from_numpy(big)).numpy()
    y = np.zeros((2, Cout, Ho, Wo))
    for ph in range(2):
        for pw in range(2):
            part = z[:, (2 * ph + pw) * Cout:(2 * ph + pw + 1) * Cout]
            y[:, :, ph::2, pw::2] = part[:, :, :len(range(ph, Ho, 2)), :len(range(pw, Wo, 2))]
    ref = torch.nn.functional.conv_transpose2d(torch.from_numpy(x), torch.from_numpy(w), stride=2, padding=pad,
                                               output_padding=op).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)
