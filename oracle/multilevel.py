"""Nesting to any depth, per spatial axis, as one composite 1-D bilinear algorithm.
TEST INFRASTRUCTURE ONLY (oracle; imports nothing from the GPU package).

Section III.A of the paper nests one Winograd kernel inside another:
the filter of length R is reshaped into the "filter reordered matrix" (column
distance r_i), the inner kernel runs on every column, the outer kernel
runs across columns.  Applied to an inner algorithm that is itself nested, the
same step nests one level deeper: an outer F(m_o, r_o) over "super-taps" of
length R_i (the inner algorithm's reach) gives

    B^T_hat = (B_o^T (x) B_i^T) . Gather   Gather: entry (j, u) -> input R_i*j + u
    G_hat   = G_o (x) G_i                   filter tap k = R_i*k1 + k0
    A^T_hat = A_o^T (x) A_i^T               output q = t*m_i + s -> position R_i*t + pos_i[s]

with window L = R_i*(l_o - 1) + L_i ("L = r(l-1) + l" for two levels)
and reach R = R_i * r_o.  Positions produced twice keep the first t (the
redundant terms of P:112 are discarded).  For m >= r at every level the
distinct positions are contiguous from 0; their count O_d is the slice advance
(O_1 = m, O_j = (m - 1) r^(j-1) + O_(j-1) for the same kernel).
The two-level special case is oracle.nested.Axis/composite (R4 order);
tests/test_oracle_multilevel.py pins this module against it and against the
direct correlation (exact, brute force) for depths 1-4.

Used by the Fig. 7 sweep (oracle.fig7) and the decomposition planner
(oracle.planner) for nests deeper than the GPU's two levels (K > 9 at stride 1).
"""
from __future__ import annotations

from fractions import Fraction
from functools import lru_cache
from typing import List, Optional

from .cooktoom import generate_kernel, kron


class Algo1D:
    """A 1-D bilinear correlation algorithm y = A^T ((B^T x) (.) (G w)).

    BT: P x L, G: P x R, AT: M x P (Fraction lists); pos[q] = output position of
    nominal output q relative to the slice origin; L window, R reach."""

    def __init__(self, BT, G, AT, pos: List[int], L: int, R: int, name: str):
        self.BT, self.G, self.AT, self.pos, self.L, self.R, self.name = BT, G, AT, pos, L, R, name
        self.P = len(BT)
        self.M = len(AT)

    def distinct(self) -> List[int]:
        """Sorted distinct output positions."""
        return sorted(set(self.pos))

    def advance(self) -> Optional[int]:
        """Contiguous distinct outputs from 0 (the slice advance), or None if there are holes."""
        d = self.distinct()
        return len(d) if d == list(range(len(d))) else None


def leaf(m: int, r: int) -> Algo1D:
    """Plain Cook-Toom F(m, r)."""
    k = generate_kernel(m, r)
    return Algo1D(k.BT, k.G, k.AT, list(range(m)), m + r - 1, r, f"F({m},{r})")


def nest(m_o: int, r_o: int, inner: Algo1D) -> Algo1D:
    """Outer F(m_o, r_o) over the super-taps of `inner` (one more level of P:100-112)."""
    ko = generate_kernel(m_o, r_o)
    l_o = m_o + r_o - 1
    Ri, Li = inner.R, inner.L
    BT_k = kron(ko.BT, inner.BT)                        # (l_o*P_i) x (l_o*L_i)
    L = Ri * (l_o - 1) + Li
    gather = [Ri * j + u for j in range(l_o) for u in range(Li)]
    BT = [[Fraction(0)] * L for _ in range(len(BT_k))]
    for p in range(len(BT_k)):
        for q, c in enumerate(gather):
            if BT_k[p][q]:
                BT[p][c] += BT_k[p][q]
    G = kron(ko.G, inner.G)                             # column k1*R_i + k0
    AT = kron(ko.AT, inner.AT)                          # row t*M_i + s
    pos = [Ri * t + inner.pos[s] for t in range(m_o) for s in range(inner.M)]
    return Algo1D(BT, G, AT, pos, L, Ri * r_o, f"F({m_o},{r_o})(x){inner.name}")


@lru_cache(maxsize=None)
def levels(m: int, r: int, d: int) -> Algo1D:
    """The same kernel F(m, r) nested d deep (d = 1: the kernel itself); cached, treat as read-only."""
    a = leaf(m, r)
    for _ in range(d - 1):
        a = nest(m, r, a)
    return a


def depth_for(R: int, r: int) -> int:
    """d = ceil(log_r R): the fewest levels of an r-tap kernel that reach R taps."""
    d, reach = 1, r
    while reach < R:
        d += 1
        reach *= r
    return d


class Counter:
    def __init__(self):
        self.mults = 0


def conv1d(x, w, algo: Algo1D, counter: Optional[Counter] = None) -> List[Fraction]:
    """Valid 1-D correlation y[i] = sum_k x[i + k] w[k] with the composite algorithm,
    exact.  The filter is zero-padded at the end to the reach; slices advance by
    the contiguous distinct-output count; every slice costs P multiplications (EWMM)."""
    R = len(w)
    if R > algo.R:
        raise ValueError("filter longer than the algorithm's reach")
    adv = algo.advance()
    if adv is None:
        raise ValueError("output positions have holes (m < r): use oracle.nested coverage phases")
    n_out = len(x) - R + 1
    wz = [Fraction(v) for v in w] + [Fraction(0)] * (algo.R - R)
    U = [sum((g * wk for g, wk in zip(row, wz)), Fraction(0)) for row in algo.G]
    xs = [Fraction(v) for v in x] + [Fraction(0)] * (algo.L + adv)
    y: List[Optional[Fraction]] = [None] * n_out
    for o in range(0, n_out, adv):
        X = xs[o:o + algo.L]
        V = [sum((b * xv for b, xv in zip(row, X) if b), Fraction(0)) for row in algo.BT]
        Mx = [u * v for u, v in zip(U, V)]
        if counter is not None:
            counter.mults += len(Mx)
        for q, row in enumerate(algo.AT):
            p = o + algo.pos[q]
            if p < n_out and y[p] is None:
                y[p] = sum((a * m for a, m in zip(row, Mx) if a), Fraction(0))
    assert all(v is not None for v in y)
    return y
