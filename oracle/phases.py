"""Stride-Winograd phase decompositions.  TEST INFRASTRUCTURE ONLY.

Eq. 2.7: F(m, r; s) = p F(m, r'+1) + (s - p) F(m, r'), r = r' s + p:
a stride-s correlation is the sum of s stride-1 correlations of the input
phases x_t[i] = x[s*i + t] with the filter phases w_t[a] = w[s*a + t]; p of
them have r'+1 taps, s - p have r'.  With a single kernel the short phases run
on the long one "with zero padding" (R9).

The transposed convolution (BASELINE config 5; not in the paper) is split the
other way round (R11): output phase phi of a stride-2 transposed conv
is a stride-1 correlation of the (un-split) input with every other tap of the
flipped filter.

Both are pinned against the direct definitions in oracle.direct and against
torch CPU fp64 (tests/test_oracle_phases.py).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np

from . import direct
from .nested import nested_conv2d, phase_taps


def stride_phase_lengths(R: int, s: int) -> List[Tuple[int, int]]:
    """Eq. 2.7's split r = r' s + p -> [(p, r'+1), (s-p, r')] (zero counts dropped)."""
    rp, p = divmod(R, s)
    out = []
    if p:
        out.append((p, rp + 1))
    if s - p and rp:
        out.append((s - p, rp))
    return out


def _stride2_phase_operands(x: np.ndarray, w: np.ndarray, pad: int):
    """Phase images x_pq[u, v] = xpad[2u+p, 2v+q] and sub-filters w_pq[a, b] =
    w[2a+p, 2b+q] (zero-padded to Kp = ceil(K/2) taps), for p, q in {0, 1}."""
    N, C, H, W = x.shape
    O, _, K, _ = w.shape
    Kp = -(-K // 2)
    Ho = direct.out_size(H, K, 2, pad)
    Wo = direct.out_size(W, K, 2, pad)
    Hp, Wp = Ho + Kp - 1, Wo + Kp - 1          # phase-image extent the valid conv needs
    big = np.zeros((N, C, 2 * Hp + 2 + 2 * pad + H, 2 * Wp + 2 + 2 * pad + W), dtype=x.dtype)
    big[:, :, pad:pad + H, pad:pad + W] = x
    xs, ws = [], []
    for p in range(2):
        for q in range(2):
            xs.append(big[:, :, p:p + 2 * Hp:2, q:q + 2 * Wp:2])
            sub = np.zeros((O, w.shape[1], Kp, Kp), dtype=w.dtype)
            taps_h = [2 * a + p for a in range(Kp)]
            taps_w = [2 * b + q for b in range(Kp)]
            for a, th in enumerate(taps_h):
                for b, tw in enumerate(taps_w):
                    if th < K and tw < K:
                        sub[:, :, a, b] = w[:, :, th, tw]
            ws.append(sub)
    return xs, ws, Kp, Ho, Wo


def stride2_conv2d_direct_phases(x: np.ndarray, w: np.ndarray, pad: int) -> np.ndarray:
    """Stride-2 conv as the sum of four stride-1 phase correlations (float64 direct)."""
    xs, ws, Kp, Ho, Wo = _stride2_phase_operands(x, w, pad)
    y = 0
    for xp, wp in zip(xs, ws):
        y = y + direct.conv2d(xp, wp, 1, 0)[:, :, :Ho, :Wo]
    return y


def stride2_conv2d_nested(x, w, pad: int, m_o: int = 3, m_i: int = 3, r_o: int = 3,
                          counter=None, exact: bool = True):
    """Stride-2 conv = sum over the 4 phases of the nested stride-1 conv (Eq. 2.7)."""
    xs, ws, Kp, Ho, Wo = _stride2_phase_operands(np.asarray(x, dtype=object if exact else np.float64),
                                                 np.asarray(w, dtype=object if exact else np.float64), pad)
    y = None
    for xp, wp in zip(xs, ws):
        part = nested_conv2d(xp, wp, 0, m_o, m_i, r_o, 3, counter=counter, exact=exact)[:, :, :Ho, :Wo]
        y = part if y is None else y + part
    return y


def _transposed_phase_operands(x: np.ndarray, w: np.ndarray, pad: int, output_padding: int):
    """Per output phase (phi_h, phi_w): the stride-1 filter with taps from
    nested.phase_taps (flipped, every other tap) and the common input offset."""
    N, C, H, W = x.shape
    _, O, K, _ = w.shape
    tab = phase_taps(K, 2, True, pad)
    Kp = tab[2]
    offs = [tab[3], tab[3 + Kp + 1]]
    taps = [tab[4:4 + Kp], tab[4 + Kp + 1:4 + 2 * Kp + 1]]
    Ho = (H - 1) * 2 - 2 * pad + K + output_padding
    Wo = (W - 1) * 2 - 2 * pad + K + output_padding
    subs = {}
    for ph in range(2):
        for pw in range(2):
            sub = np.zeros((O, C, Kp, Kp), dtype=w.dtype)
            for d, th in enumerate(taps[ph]):
                for e, tw in enumerate(taps[pw]):
                    if th >= 0 and tw >= 0:
                        sub[:, :, d, e] = w[:, :, th, tw].T
            subs[(ph, pw)] = sub
    return subs, offs, Kp, Ho, Wo


def conv_transpose2d_phases(x, w, pad: int, output_padding: int, nested: bool = False,
                            m_o: int = 3, m_i: int = 3, exact: bool = False, counter=None):
    """Stride-2 transposed conv as 4 interleaved stride-1 correlations.

    Output phase (phi_h, phi_w) holds y[2j+phi_h, 2k+phi_w] = correlation of x
    zero-padded by the phase offset with the phase sub-filter.
    """
    x = np.asarray(x, dtype=object if exact else np.float64)
    w = np.asarray(w, dtype=object if exact else np.float64)
    subs, offs, Kp, Ho, Wo = _transposed_phase_operands(x, w, pad, output_padding)
    N, C, H, W = x.shape
    O = w.shape[1]
    y = np.zeros((N, O, Ho, Wo), dtype=x.dtype)
    for (ph, pw), sub in subs.items():
        nh, nw = -(-(Ho - ph) // 2), -(-(Wo - pw) // 2)
        assert offs[0] == offs[1]
        off = offs[0]
        # pad so that valid correlation output j reads x[j + d - off]
        padded = np.zeros((N, C, nh + Kp - 1, nw + Kp - 1), dtype=x.dtype)
        hh = min(H, nh + Kp - 1 - off)
        ww = min(W, nw + Kp - 1 - off)
        padded[:, :, off:off + hh, off:off + ww] = x[:, :, :hh, :ww]
        if nested:
            part = nested_conv2d(padded, sub, 0, m_o, m_i, 3, 3, counter=counter, exact=exact)
        else:
            part = direct.conv2d(padded, sub, 1, 0)
        y[:, :, ph::2, pw::2] = part[:, :, :nh, :nw]
    return y


def decompose(R: int, S: int, r: int):
    """Step 1 of the decomposition algorithm: while S > 1 apply the
    stride split (Eq. 2.7), while R > r nest (III.A).  Returns the expression tree
    ("sum", [...]) / ("nest", levels, leaf) / ("leaf", r)."""
    if S > 1:
        terms = []
        for count, length in stride_phase_lengths(R, S):
            for _ in range(count):
                terms.append(decompose(length, 1, r))
        return ("sum", terms)
    if R <= r:
        return ("leaf", r)
    levels, reach = 1, r
    while reach < R:
        levels += 1
        reach *= r
    return ("nest", levels, ("leaf", r))
