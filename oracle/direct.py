"""FP64 direct convolution by definition (Eq. 2.1).  TEST INFRASTRUCTURE ONLY.

Eq. 2.1 with its garbled indices read as (R1):
    y[n, o, i, j] = sum_{c, r, s} xpad[n, c, i*S + r, j*S + s] * w[o, c, r, s]
cross-correlation (no filter flip), zero padding ``pad`` on every side.

The transposed convolution (not in the paper; BASELINE config 5, R11)
is written from its own definition, the adjoint scatter of Eq. 2.1:
    y[n, o, i*S + r - pad, j*S + s - pad] += x[n, c, i, j] * w[c, o, r, s]
output size (H - 1) * S - 2 * pad + K + output_padding.

Pins (tests/test_oracle_direct.py): a scalar 7-deep loop on tiny inputs
(brute force), torch CPU fp64 conv2d / conv_transpose2d (an independent
library), the delta-filter and all-ones closed forms.
"""
from __future__ import annotations

import numpy as np


def out_size(H: int, K: int, stride: int, pad: int) -> int:
    return (H + 2 * pad - K) // stride + 1


def conv2d(x: np.ndarray, w: np.ndarray, stride: int = 1, pad: int = 0) -> np.ndarray:
    """y = Eq. 2.1 in float64.  x [N, C, H, W], w [O, C, K, K] -> y [N, O, Ho, Wo].

    One tap (r, s) at a time: the strided window of xpad for that tap is a
    [N, C, Ho, Wo] view, contracted with w[:, :, r, s] over C.  Same sum as
    Eq. 2.1, ordered tap by tap.
    """
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    N, C, H, W = x.shape
    O, C2, KH, KW = w.shape
    assert C == C2
    Ho, Wo = out_size(H, KH, stride, pad), out_size(W, KW, stride, pad)
    xp = np.zeros((N, C, H + 2 * pad, W + 2 * pad))
    xp[:, :, pad:pad + H, pad:pad + W] = x
    y = np.zeros((N, O, Ho, Wo))
    for r in range(KH):
        for s in range(KW):
            win = xp[:, :, r:r + stride * (Ho - 1) + 1:stride, s:s + stride * (Wo - 1) + 1:stride]
            # [N, C, Ho, Wo] x [O, C] -> [N, O, Ho, Wo]
            y += np.einsum("nchw,oc->nohw", win, w[:, :, r, s], optimize=True)
    return y


def conv2d_at(x: np.ndarray, w: np.ndarray, stride: int, pad: int, points) -> np.ndarray:
    """Eq. 2.1 evaluated only at the listed output points (n, o, i, j), float64.

    Used to check full-size GPU outputs on a sample the CPU can afford.
    """
    N, C, H, W = x.shape
    O, _, K, _ = w.shape
    out = np.empty(len(points))
    for t, (n, o, i, j) in enumerate(points):
        acc = 0.0
        h0, w0 = i * stride - pad, j * stride - pad
        hs, he = max(h0, 0), min(h0 + K, H)
        ws, we = max(w0, 0), min(w0 + K, W)
        if hs < he and ws < we:
            patch = np.asarray(x[n, :, hs:he, ws:we], dtype=np.float64)
            wt = np.asarray(w[o, :, hs - h0:he - h0, ws - w0:we - w0], dtype=np.float64)
            acc = float(np.sum(patch * wt))
        out[t] = acc
    return out


def conv_transpose2d(x: np.ndarray, w: np.ndarray, stride: int, pad: int,
                     output_padding: int = 0) -> np.ndarray:
    """Transposed convolution by its scatter definition, float64.

    x [N, C, H, W], w [C, O, K, K] (PyTorch layout) -> y [N, O, Ho, Wo] with
    Ho = (H - 1) * stride - 2 * pad + K + output_padding.
    """
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    N, C, H, W = x.shape
    C2, O, K, K2 = w.shape
    assert C == C2 and K == K2
    Ho = (H - 1) * stride - 2 * pad + K + output_padding
    Wo = (W - 1) * stride - 2 * pad + K + output_padding
    # full (uncropped) canvas: index u = i*stride + r, later shifted by -pad
    Hf = max((H - 1) * stride + K, Ho + pad)
    Wf = max((W - 1) * stride + K, Wo + pad)
    canvas = np.zeros((N, O, Hf, Wf))
    for r in range(K):
        for s in range(K):
            contrib = np.einsum("nchw,co->nohw", x, w[:, :, r, s], optimize=True)
            canvas[:, :, r:r + stride * (H - 1) + 1:stride, s:s + stride * (W - 1) + 1:stride] += contrib
    return canvas[:, :, pad:pad + Ho, pad:pad + Wo]


def conv_transpose2d_at(x: np.ndarray, w: np.ndarray, stride: int, pad: int, points) -> np.ndarray:
    """Transposed convolution at the listed output points (n, o, Y, X), float64."""
    N, C, H, W = x.shape
    _, O, K, _ = w.shape
    out = np.empty(len(points))
    for t, (n, o, Y, X) in enumerate(points):
        acc = 0.0
        for r in range(K):
            ui = Y + pad - r
            if ui < 0 or ui % stride:
                continue
            i = ui // stride
            if i >= H:
                continue
            for s in range(K):
                uj = X + pad - s
                if uj < 0 or uj % stride:
                    continue
                j = uj // stride
                if j >= W:
                    continue
                acc += float(np.dot(np.asarray(x[n, :, i, j], np.float64),
                                    np.asarray(w[:, o, r, s], np.float64)))
        out[t] = acc
    return out


def conv2d_depthwise(x: np.ndarray, w: np.ndarray, stride: int = 1, pad: int = 0) -> np.ndarray:
    """Depthwise (groups = C) Eq. 2.1 in float64: channel c of y sees only channel c of x and
    filter c -- y[n, c, i, j] = sum_{r, s} xpad[n, c, i*S + r, j*S + s] * w[c, 0, r, s]
    (Table I's PNASNet depthwise row).  x [N, C, H, W], w [C, 1, K, K]."""
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    N, C, H, W = x.shape
    C2, one, KH, KW = w.shape
    assert C == C2 and one == 1
    Ho, Wo = out_size(H, KH, stride, pad), out_size(W, KW, stride, pad)
    xp = np.zeros((N, C, H + 2 * pad, W + 2 * pad))
    xp[:, :, pad:pad + H, pad:pad + W] = x
    y = np.zeros((N, C, Ho, Wo))
    for r in range(KH):
        for s in range(KW):
            win = xp[:, :, r:r + stride * (Ho - 1) + 1:stride, s:s + stride * (Wo - 1) + 1:stride]
            y += win * w[None, :, 0, r, s, None, None]
    return y


def conv2d_bruteforce(x, w, stride: int = 1, pad: int = 0):
    """Eq. 2.1 as seven nested scalar loops (tiny inputs only)."""
    N, C, H, W = len(x), len(x[0]), len(x[0][0]), len(x[0][0][0])
    O, K = len(w), len(w[0][0])
    Ho, Wo = out_size(H, K, stride, pad), out_size(W, K, stride, pad)
    y = [[[[0.0] * Wo for _ in range(Ho)] for _ in range(O)] for _ in range(N)]
    for n in range(N):
        for o in range(O):
            for i in range(Ho):
                for j in range(Wo):
                    acc = 0.0
                    for c in range(C):
                        for r in range(K):
                            for s in range(K):
                                hh, ww = i * stride + r - pad, j * stride + s - pad
                                if 0 <= hh < H and 0 <= ww < W:
                                    acc += x[n][c][hh][ww] * w[o][c][r][s]
                    y[n][o][i][j] = acc
    return y
