"""The decomposition algorithm of section IV.B: expression tree, lengths, reverse Polish
order, execution.  TEST INFRASTRUCTURE ONLY (oracle; the library's planner in
csrc/decompose.cu is written independently and compared with this one).

P:126-134, four steps, here for a K-tap (R) stride-S axis and one base kernel F(m, r):
  step 1: "iteratively checks if the given F(M, R; S) has S > 1 or R > r.
      If yes, it decomposes the Winograd kernel with stride Winograd or nested Winograd
      algorithm, respectively."  Stride: Eq. 2.7, R = r' S + p -> p phases of
      r' + 1 taps and S - p of r' taps, summed (Sum); nesting: III.A (Nest, d =
      ceil(log_r R) levels of the same kernel, filter zero-padded at the end);
      R <= r: the kernel itself (Leaf, filter zero-padded to r taps).
  The tree is "read out in the reverse polish order": post-order tokens
      K<m>,<r>   NEST<d>   REP<n>   SUM<k>      (e.g. Eq. 4.1: "K2,2 NEST2 K2,2 REP2 SUM2").
  step 2: "M_2 = m. Then we compute backward": a Leaf outputs m, a Nest the
      distinct outputs O_d of d levels (m^2 for two levels when m = r), and a Sum
      needs equal-length terms -- "F(n.m, r) = n.F(m, r) can be used to adjust the output
      length": every term is wrapped in Repeat(n) to the least common multiple of the
      term lengths (R10a; SPEC S:318 makes the same choice).
  steps 3-4 (data marshaling, Fig. 6, missing): execute_plan splits input and filter into
      the S polyphase components (x_t[i] = x[S i + t], w_t[a] = w[S a + t]), runs every
      term on its phase and sums; Repeat runs its child n times on successive windows.

Phase -> term assignment (P:130 does not spell it out): term t handles
phase t, so the longer (r' + 1)-tap phases come first, as in Eq. 4.1 where the nested
term precedes the leaf.

Pins (tests/test_oracle_planner.py): Eq. 4.1's tree, lengths and RPN (tests/golden/
eq4_1_plan.json); execute_plan equals the direct strided correlation exactly for every
(R, S) in 1..12 x 1..3 and each Fig. 7 kernel (1-D) and for a 2-D sample; parse(to_rpn)
round trip; malformed streams are rejected; the library's nw_decompose emits the same
tokens and M for the whole grid.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from math import gcd
from typing import List, Optional, Union

from . import direct
from .multilevel import depth_for, leaf as ml_leaf, levels


# ----------------------------------------------------------------------------
# tree
# ----------------------------------------------------------------------------
@dataclass
class Leaf:
    m: int
    r: int
    taps: int                 # filter taps this leaf carries (<= r; zero-padded to r)
    M: int = 0


@dataclass
class Nest:
    m: int
    r: int
    levels: int
    taps: int                 # <= r ** levels
    M: int = 0


@dataclass
class Repeat:
    n: int
    child: "Node"
    M: int = 0


@dataclass
class Sum:
    terms: List["Node"]
    S: int                    # stride of the split (number of phases, incl. empty ones)
    M: int = 0


Node = Union[Leaf, Nest, Repeat, Sum]


def stride_phases(R: int, S: int) -> List[int]:
    """Taps of phase t = 0..S-1 of an R-tap filter at stride S: ceil((R - t) / S) (Eq. 2.7)."""
    return [max(0, -(-(R - t) // S)) for t in range(S)]


def decompose(R: int, S: int, m: int, r: int) -> Node:
    """Step 1."""
    if R < 1 or S < 1 or m < 1 or r < 1:
        raise ValueError("R, S, m, r must be >= 1")
    if m < r and R > r:
        raise ValueError("nesting needs m >= r (contiguous outputs); m < r leaves holes")
    if S > 1:
        terms = [decompose(t, 1, m, r) for t in stride_phases(R, S) if t > 0]
        return Sum(terms, S)
    if R > r:
        return Nest(m, r, depth_for(R, r), R)
    return Leaf(m, r, R)


def _lcm(a: int, b: int) -> int:
    return a * b // gcd(a, b)


def resolve_lengths(p: Node) -> Node:
    """Step 2: fill M bottom-up; wrap Sum terms in Repeat to their lcm."""
    if isinstance(p, Leaf):
        p.M = p.m
    elif isinstance(p, Nest):
        p.M = levels(p.m, p.r, p.levels).advance()
    elif isinstance(p, Repeat):
        resolve_lengths(p.child)
        p.M = p.n * p.child.M
    elif isinstance(p, Sum):
        for t in p.terms:
            resolve_lengths(t)
        L = 1
        for t in p.terms:
            L = _lcm(L, t.M)
        p.terms = [t if t.M == L else Repeat(L // t.M, t, L) for t in p.terms]
        p.M = L
    return p


def plan(R: int, S: int, m: int, r: int) -> Node:
    return resolve_lengths(decompose(R, S, m, r))


# ----------------------------------------------------------------------------
# reverse Polish order
# ----------------------------------------------------------------------------
def to_rpn(p: Node) -> List[str]:
    if isinstance(p, Leaf):
        return [f"K{p.m},{p.r}"]
    if isinstance(p, Nest):
        return [f"K{p.m},{p.r}", f"NEST{p.levels}"]
    if isinstance(p, Repeat):
        return to_rpn(p.child) + [f"REP{p.n}"]
    out: List[str] = []
    for t in p.terms:
        out += to_rpn(t)
    return out + [f"SUM{len(p.terms)}"]


def rpn_text(p: Node) -> str:
    return " ".join(to_rpn(p))


def parse_rpn(tokens) -> Node:
    """Stack evaluation of the token stream (structure only: tap counts are not in the RPN)."""
    if isinstance(tokens, str):
        tokens = tokens.split()
    st: List[Node] = []
    for tok in tokens:
        if tok.startswith("K"):
            m, r = (int(v) for v in tok[1:].split(","))
            st.append(Leaf(m, r, r))
        elif tok.startswith("NEST"):
            if not st or not isinstance(st[-1], Leaf):
                raise ValueError("NEST needs a kernel operand")
            k = st.pop()
            st.append(Nest(k.m, k.r, int(tok[4:]), k.r ** int(tok[4:])))
        elif tok.startswith("REP"):
            if not st:
                raise ValueError("stack underflow at " + tok)
            st.append(Repeat(int(tok[3:]), st.pop()))
        elif tok.startswith("SUM"):
            k = int(tok[3:])
            if len(st) < k:
                raise ValueError("stack underflow at " + tok)
            terms = st[-k:]
            del st[-k:]
            st.append(Sum(terms, k))
        else:
            raise ValueError("bad token " + tok)
    if len(st) != 1:
        raise ValueError("malformed stream: %d operands left" % len(st))
    return st[0]


def shape(p: Node):
    """Structural signature (kind, kernel, levels / n / arity) for round-trip comparisons."""
    if isinstance(p, Leaf):
        return ("K", p.m, p.r)
    if isinstance(p, Nest):
        return ("NEST", p.m, p.r, p.levels)
    if isinstance(p, Repeat):
        return ("REP", p.n, shape(p.child))
    return ("SUM", tuple(shape(t) for t in p.terms))


# ----------------------------------------------------------------------------
# execution (steps 3-4): exact, with an EWMM counter
# ----------------------------------------------------------------------------
class Counter:
    def __init__(self):
        self.mults = 0


def _algo(p: Node):
    return ml_leaf(p.m, p.r) if isinstance(p, Leaf) else levels(p.m, p.r, p.levels)


def _slice1(p: Node, xs: List[Fraction], w: List[Fraction], o: int, cnt: Optional[Counter]) -> List[Fraction]:
    """One slice of a Leaf / Nest at output origin o: its M outputs."""
    a = _algo(p)
    wz = list(w) + [Fraction(0)] * (a.R - len(w))
    U = [sum((g * v for g, v in zip(row, wz)), Fraction(0)) for row in a.G]
    X = xs[o:o + a.L]
    V = [sum((b * v for b, v in zip(row, X) if b), Fraction(0)) for row in a.BT]
    Mx = [u * v for u, v in zip(U, V)]
    if cnt is not None:
        cnt.mults += len(Mx)
    out: List[Optional[Fraction]] = [None] * p.M
    for q, row in enumerate(a.AT):
        pos = a.pos[q]
        if pos < p.M and out[pos] is None:
            out[pos] = sum((c * v for c, v in zip(row, Mx) if c), Fraction(0))
    return out


def _eval1(p: Node, xs, w, o: int, cnt) -> List[Fraction]:
    """Outputs o .. o + p.M - 1 of the correlation of xs with w (stride of p's level)."""
    if isinstance(p, (Leaf, Nest)):
        return _slice1(p, xs, w, o, cnt)
    if isinstance(p, Repeat):
        out = []
        for j in range(p.n):
            out += _eval1(p.child, xs, w, o + j * p.child.M, cnt)
        return out
    S = p.S
    acc = [Fraction(0)] * p.M
    ts = [t for t in range(S) if len(w[t::S]) > 0]
    for t, term in zip(ts, p.terms):
        part = _eval1(term, xs[t::S], w[t::S], o, cnt)
        acc = [a + b for a, b in zip(acc, part)]
    return acc


def execute_plan(p: Node, x, w, S: int, cnt: Optional[Counter] = None) -> List[Fraction]:
    """y[i] = sum_k x[S i + k] w[k] (valid, stride S) by the plan, in tiles of p.M outputs."""
    R = len(w)
    n_out = (len(x) - R) // S + 1
    xs = [Fraction(v) for v in x] + [Fraction(0)] * (S * (p.M + 64 * R + 64))
    ws = [Fraction(v) for v in w]
    y: List[Fraction] = []
    for o in range(0, n_out, p.M):
        y += _eval1(p, xs, ws, o, cnt)
    return y[:n_out]


def _slice2(ph: Node, pw: Node, X, W, oh: int, ow: int, cnt):
    ah, aw = _algo(ph), _algo(pw)
    Wz = [[Fraction(0)] * aw.R for _ in range(ah.R)]
    for i, row in enumerate(W):
        for j, v in enumerate(row):
            Wz[i][j] = v
    GW = [[sum((g * Wz[k][j] for k, g in enumerate(grow) if g), Fraction(0)) for j in range(aw.R)] for grow in ah.G]
    U = [[sum((gw * g for gw, g in zip(GW[i], grow) if g), Fraction(0)) for grow in aw.G] for i in range(ah.P)]
    Xs = [row[ow:ow + aw.L] for row in X[oh:oh + ah.L]]
    BX = [[sum((b * Xs[k][j] for k, b in enumerate(brow) if b), Fraction(0)) for j in range(aw.L)] for brow in ah.BT]
    V = [[sum((bx * b for bx, b in zip(BX[i], brow) if b), Fraction(0)) for brow in aw.BT] for i in range(ah.P)]
    Mx = [[U[i][j] * V[i][j] for j in range(aw.P)] for i in range(ah.P)]
    if cnt is not None:
        cnt.mults += ah.P * aw.P
    AM = [[sum((a * Mx[k][j] for k, a in enumerate(arow) if a), Fraction(0)) for j in range(aw.P)] for arow in ah.AT]
    Y = [[sum((am * a for am, a in zip(AM[i], arow) if a), Fraction(0)) for arow in aw.AT] for i in range(ah.M)]
    out = [[None] * pw.M for _ in range(ph.M)]
    for qi in range(ah.M):
        for qj in range(aw.M):
            i, j = ah.pos[qi], aw.pos[qj]
            if i < ph.M and j < pw.M and out[i][j] is None:
                out[i][j] = Y[qi][qj]
    return out


def _eval2(ph: Node, pw: Node, X, W, oh: int, ow: int, cnt):
    """A ph.M x pw.M output block: the same tree runs on both axes (separable, R7)."""
    if isinstance(ph, Repeat):
        rows = []
        for j in range(ph.n):
            rows += _eval2(ph.child, pw, X, W, oh + j * ph.child.M, ow, cnt)
        return rows
    if isinstance(pw, Repeat):
        parts = [_eval2(ph, pw.child, X, W, oh, ow + j * pw.child.M, cnt) for j in range(pw.n)]
        return [sum((p[i] for p in parts), []) for i in range(ph.M)]
    if isinstance(ph, Sum):
        S = ph.S
        acc = [[Fraction(0)] * pw.M for _ in range(ph.M)]
        ts = [t for t in range(S) if len(W[t::S]) > 0]
        for th, termh in zip(ts, ph.terms):
            for tw, termw in zip(ts, pw.terms):
                Xp = [row[tw::S] for row in X[th::S]]
                Wp = [row[tw::S] for row in W[th::S]]
                part = _eval2(termh, termw, Xp, Wp, oh, ow, cnt)
                acc = [[a + b for a, b in zip(ra, rb)] for ra, rb in zip(acc, part)]
        return acc
    return _slice2(ph, pw, X, W, oh, ow, cnt)


def execute_plan2d(p: Node, x, w, S: int, cnt: Optional[Counter] = None):
    """2-D valid correlation at stride S (square filter, the plan on both axes)."""
    H, Wd = len(x), len(x[0])
    R = len(w)
    Ho, Wo = (H - R) // S + 1, (Wd - R) // S + 1
    ext = S * (p.M + 64 * R + 64)
    X = [[Fraction(v) for v in row] + [Fraction(0)] * ext for row in x] + \
        [[Fraction(0)] * (Wd + ext) for _ in range(ext)]
    Wf = [[Fraction(v) for v in row] for row in w]
    y = [[None] * Wo for _ in range(Ho)]
    for oh in range(0, Ho, p.M):
        for ow in range(0, Wo, p.M):
            blk = _eval2(p, p, X, Wf, oh, ow, cnt)
            for i in range(p.M):
                for j in range(p.M):
                    if oh + i < Ho and ow + j < Wo:
                        y[oh + i][ow + j] = blk[i][j]
    return y
