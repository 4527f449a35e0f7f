"""Literal OLA-Winograd evaluator with EWMM counter.  TEST INFRASTRUCTURE ONLY.

Eq. 2.3 and P:52-58: slice the length-R filter into ceil(R/r) blocks w'_b of
length r (last block zero-padded), slide each over the input with F(m, r) and
add the results at the same output positions:
    y[o : o+m] = sum_b F(m, r)(x[o + r*b : o + r*b + l], w'_b).
2-D: the same over block pairs (b_h, b_w) with the 2-D F(m x m, r x r) of
Eq. 2.2, input channels summed (Eq. 2.1).

Pins (tests/test_oracle_ola.py): Eq. 2.3's worked example (R = 4, F(2,2):
exactly the sub-vector pairs (x'_0, w'_0), (x'_1, w'_1) | (x'_1, w'_0),
(x'_2, w'_1), 12 multiplications, tests/golden/eq2_3_ola_f22.json); exact
equality with direct convolution; counter == closed form.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

from .cooktoom import generate_kernel


def ola_conv1d(x, w, m: int, r: int, counter=None, trace=None):
    """Valid 1-D correlation by OLA-Winograd (Eq. 2.3)."""
    k = generate_kernel(m, r)
    R = len(w)
    nb = -(-R // r)
    wz = list(w) + [0] * (nb * r - R)
    n_out = len(x) - R + 1
    xs = list(x) + [0] * (nb * r + k.l + m)
    y = [Fraction(0)] * n_out
    for o in range(0, n_out, m):
        acc = [Fraction(0)] * m
        for b in range(nb):
            xb = xs[o + r * b:o + r * b + k.l]
            wb = wz[r * b:r * b + r]
            if trace is not None:
                trace.append((o, b, o + r * b))
            bx = [sum(Fraction(k.BT[p][i]) * xb[i] for i in range(k.l)) for p in range(k.l)]
            gw = [sum(Fraction(k.G[p][i]) * wb[i] for i in range(r)) for p in range(k.l)]
            prod = [bx[p] * gw[p] for p in range(k.l)]
            if counter is not None:
                counter.mults += k.l
            for q in range(m):
                acc[q] += sum(k.AT[q][p] * prod[p] for p in range(k.l))
        for q in range(m):
            if o + q < n_out:
                y[o + q] = acc[q]
    return y


def ola_conv2d(x, w, pad: int, m: int, r: int = 3, counter=None, exact: bool = True):
    """Multichannel 2-D OLA-Winograd, stride 1, zero padding (Eq. 2.3 in 2-D)."""
    N, C, H, W = x.shape
    O, _, K, _ = w.shape
    k = generate_kernel(m, r)
    nb = -(-K // r)
    cast = (lambda v: Fraction(v)) if exact else float
    dt = object if exact else np.float64
    M = lambda mat: np.array([[cast(v) for v in row] for row in mat], dtype=dt)
    BT, G, AT = M(k.BT), M(k.G), M(k.AT)
    Ho, Wo = H + 2 * pad - K + 1, W + 2 * pad - K + 1
    wz = np.zeros((O, C, nb * r, nb * r), dtype=dt)
    if exact:
        wz[...] = Fraction(0)
    for o in range(O):
        for c in range(C):
            for i in range(K):
                for j in range(K):
                    wz[o, c, i, j] = cast(w[o, c, i, j])
    # U[bh, bw] = G w'_b G^T for every block pair
    U = {}
    for bh in range(nb):
        for bw in range(nb):
            blk = wz[:, :, r * bh:r * bh + r, r * bw:r * bw + r]
            U[(bh, bw)] = np.einsum("pi,ocij,qj->ocpq", G, blk, G) if not exact else \
                np.array([[G.dot(blk[o, c]).dot(G.T) for c in range(C)] for o in range(O)], dtype=object)
    ext = nb * r + k.l + m
    xp = np.zeros((N, C, H + 2 * pad + ext, W + 2 * pad + ext), dtype=dt)
    if exact:
        xp[...] = Fraction(0)
    for n in range(N):
        for c in range(C):
            for i in range(H):
                for j in range(W):
                    xp[n, c, pad + i, pad + j] = cast(x[n, c, i, j])
    y = np.zeros((N, O, Ho, Wo), dtype=dt)
    for n in range(N):
        for oh in range(0, Ho, m):
            for ow in range(0, Wo, m):
                acc = None
                for (bh, bw), Ub in U.items():
                    xb = xp[n, :, oh + r * bh:oh + r * bh + k.l, ow + r * bw:ow + r * bw + k.l]
                    V = np.array([BT.dot(xb[c]).dot(BT.T) for c in range(C)], dtype=dt)
                    Msum = sum(Ub[:, c] * V[c][None] for c in range(C))
                    if counter is not None:
                        counter.mults += O * C * k.l * k.l
                    acc = Msum if acc is None else acc + Msum
                Y = np.array([AT.dot(acc[o]).dot(AT.T) for o in range(O)], dtype=dt)
                hh, ww = min(m, Ho - oh), min(m, Wo - ow)
                y[n, :, oh:oh + hh, ow:ow + ww] = Y[:, :hh, :ww]
    return y
