"""Exact Cook-Toom construction of the Winograd kernel F(m, r).  TEST INFRASTRUCTURE ONLY.

Paper: y = A^T (B^T x (.) G w) for 1-D F(m, r), l = m + r - 1 (Eq. 2.2).
"These matrices are derived from a Vandermonde matrix"; the paper never
states the interpolation points (R2), so the reading used here is
the point order 0, 1, -1, 2, -2, 1/2, -1/2, 4, -4, 1/4, -1/4, ... with the last
point replaced by infinity for l >= 2.

Construction (polynomial-product view, written out step by step):
  linear convolution s = g * h of a length-r filter g and a length-m vector h is
  s = Interp . ((E_r g) (.) (E_m h)) where E_k[j] = [1, a_j, ..., a_j^(k-1)] is
  evaluation at point a_j (at infinity: the leading coefficient, [0,..,0,1]) and
  Interp = E_l^(-1).  Winograd's correlation F(m, r) is the transpose of that
  bilinear map in h, so
      A^T = E_m^T,   G = D^-1 E_r,   B^T = D Interp^T,
  where D is any invertible diagonal.  We take D = diag(f_j) with
  f_j = sgn(prod_{i!=j}(a_j - a_i)) * |prod ...| chosen so that B^T row j is
  sgn(f_j) * coeffs(prod_{i != j, finite} (x - a_i)) (integer for integer points)
  and G row j = a_j^k / |prod_{i != j} (a_j - a_i)|; the infinity row of B^T is
  coeffs(prod_i (x - a_i)) and of G is [0, .., 0, 1]  (R3: B and A
  integer, the fractions live in G).

Pins (tests/test_oracle_cooktoom.py): the exact identity A^T((B^T x)(.)(G w)) =
valid correlation on random rationals (brute force), for all m, r <= 6, l <= 9;
Lavin & Gray's published F(2,3) matrices (paper ref [1]) up to the sign of the
infinity row; F(1, r) degenerating to the native dot product.
"""
from __future__ import annotations

from fractions import Fraction
from typing import List, Optional, Sequence

INF = None  # the point at infinity


def make_points(l: int) -> List[Optional[Fraction]]:
    """l distinct interpolation points, last one infinity when l >= 2 (R2)."""
    if l < 1:
        raise ValueError("l must be >= 1")
    seq: List[Fraction] = [Fraction(0)]
    k = 0
    while len(seq) < l:
        # magnitudes 1, 2, 1/2, 4, 1/4, 8, ... each followed by its negative
        if k == 0:
            mag = Fraction(1)
        elif k % 2 == 1:
            mag = Fraction(2) ** ((k + 1) // 2)
        else:
            mag = Fraction(1, 2 ** (k // 2))
        seq.extend([mag, -mag])
        k += 1
    pts: List[Optional[Fraction]] = list(seq[:l])
    if l >= 2:
        pts[-1] = INF
    return pts


def _poly_from_roots(roots: Sequence[Fraction]) -> List[Fraction]:
    """Coefficients (constant term first) of prod (x - a)."""
    c = [Fraction(1)]
    for a in roots:
        nc = [Fraction(0)] * (len(c) + 1)
        for i, ci in enumerate(c):
            nc[i + 1] += ci
            nc[i] -= a * ci
        c = nc
    return c


class WinogradKernel:
    """The (A^T, G, B^T) triple of F(m, r) with exact Fraction entries."""

    def __init__(self, m: int, r: int, AT, G, BT, points):
        self.m, self.r, self.l = m, r, m + r - 1
        self.AT, self.G, self.BT, self.points = AT, G, BT, points

    def as_float(self):
        """Nearest IEEE-754 binary64 value of every entry (to_float_kernel)."""
        f = lambda M: [[float(v) for v in row] for row in M]
        return f(self.AT), f(self.G), f(self.BT)


def generate_kernel(m: int, r: int) -> WinogradKernel:
    if m < 1 or r < 1:
        raise ValueError("F(m, r) needs m >= 1 and r >= 1")
    l = m + r - 1
    pts = make_points(l)
    finite = [p for p in pts if p is not INF]
    if len(set(finite)) != len(finite):
        raise ValueError("coincident interpolation points")
    AT = [[Fraction(0)] * l for _ in range(m)]
    G = [[Fraction(0)] * r for _ in range(l)]
    BT = [[Fraction(0)] * l for _ in range(l)]
    for j, a in enumerate(pts):
        if a is INF:
            AT[m - 1][j] = Fraction(1)
            G[j][r - 1] = Fraction(1)
            coeffs = _poly_from_roots(finite)
            for i in range(l):
                BT[j][i] = coeffs[i] if i < len(coeffs) else Fraction(0)
            continue
        for i in range(m):
            AT[i][j] = a ** i
        others = [b for b in finite if b != a]
        f = Fraction(1)
        for b in others:
            f *= (a - b)
        sgn = 1 if f > 0 else -1
        for k in range(r):
            G[j][k] = (a ** k) / abs(f)
        coeffs = _poly_from_roots(others)
        for i in range(l):
            BT[j][i] = sgn * (coeffs[i] if i < len(coeffs) else Fraction(0))
    return WinogradKernel(m, r, AT, G, BT, pts)


def apply_1d(k: WinogradKernel, x: Sequence, w: Sequence) -> list:
    """y = A^T ((B^T x) (.) (G w)) in exact arithmetic (Eq. 2.2, 1-D form)."""
    bx = [sum(k.BT[p][i] * x[i] for i in range(k.l)) for p in range(k.l)]
    gw = [sum(k.G[p][i] * w[i] for i in range(k.r)) for p in range(k.l)]
    prod = [bx[p] * gw[p] for p in range(k.l)]
    return [sum(k.AT[o][p] * prod[p] for p in range(k.l)) for o in range(k.m)]


def correlate_valid_1d(x: Sequence, w: Sequence) -> list:
    """Brute-force valid cross-correlation y[i] = sum_k x[i+k] w[k] (Eq. 2.1, 1-D)."""
    n = len(x) - len(w) + 1
    return [sum(x[i + k] * w[k] for k in range(len(w))) for i in range(n)]


def verify_kernel(k: WinogradKernel, trials: int = 100, seed: int = 0) -> bool:
    """Exact identity A^T((B^T x)(.)(G w)) == valid correlation on random rationals."""
    import random

    rng = random.Random(seed)
    for _ in range(trials):
        x = [Fraction(rng.randint(-100, 100), rng.randint(1, 100)) for _ in range(k.l)]
        w = [Fraction(rng.randint(-100, 100), rng.randint(1, 100)) for _ in range(k.r)]
        if apply_1d(k, x, w) != correlate_valid_1d(x, w):
            return False
    return True


def kron(A, B):
    """Tensor (Kronecker) product of two Fraction matrices (Eq. 2.5)."""
    return [[a * b for a in ra for b in rb] for ra in A for rb in B]
