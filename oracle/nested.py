"""Literal nested-Winograd evaluator, composite matrices and plan tables.
TEST INFRASTRUCTURE ONLY.

Follows P:98-114 (section III.A) step by step, per spatial axis:
  step 1, nested filter transform: reshape the length-R filter
      into the "filter reordered matrix" W[k0][k1] = w[r_i*k1 + k0] (column
      distance r_i, "zero-pad at the end of the filter" for taps >= R), then
      U = G_i W G_o^T  (the 2-D Winograd filter transform of Eq. 2.6).
  step 2, nested input transform: the outer slide cuts a slice of
      length L = r_i*(l_o - 1) + l_i at origin o; the inner slide (window l_i,
      stride r_i) cuts its "reordered columns" X[s][j] = x[o + r_i*j + s],
      then V = B_i^T X B_o.
  step 3: EWMM M = U (.) V, counted; output reordered matrix
      Y = A_i^T M A_o; Y[s][t] is the output at o + r_i*t + s; redundant terms
      (m != r) are discarded.
2-D (P:114 is truncated; R7): the same procedure applied separably
to both spatial axes, i.e. the rank-4 reordered tensors X[s_h][j_h][s_w][j_w]
transformed by a mode product on each axis, input channels summed in the
transform domain (Eq. 2.1's channel sum; R4 fixes the index order).

The paper's own example uses F(2,2) at both levels (Fig. 3); the build uses
3-tap tiles (r_i = 3, BASELINE north_star) with F(m_o, r_o) outer and
F(m_i, 3) inner.  This module is general in (m_o, r_o, m_i, r_i).

Slice advance and coverage (R5, #R6): the distinct outputs of one
slice are the positions r_i*t + s.  When m_i >= r_i they are contiguous,
0 .. r_i*(m_o-1) + m_i - 1, the slice advances by that count and a position
produced twice keeps the smallest t.  When m_i < r_i they leave holes; the
slice is then repeated at shifts 0, m_i, 2*m_i, ... (< r_i) -- "coverage
phases" -- each keeping the residues it adds, and the tile advances r_i*m_o.

Pins (tests/test_oracle_nested.py): exact equality with direct convolution
(oracle.direct) on integer inputs for K = 3..9 and several (m_o, m_i);
Fig. 3's worked example (R = 4, F(2,2): window L = 7, 9 multiplications,
4 outputs); the l^n / m^n count law; composite-matrix form equals the
literal mode-product form; counter equals the closed forms in oracle.counts.
"""
from __future__ import annotations

from fractions import Fraction
from math import gcd
from typing import List, Tuple

import numpy as np

from .cooktoom import generate_kernel, kron


# ----------------------------------------------------------------------------
# per-axis geometry
# ----------------------------------------------------------------------------
class Axis:
    """One spatial axis of a nested F(m_o, r_o) (x) F(m_i, r_i) algorithm."""

    def __init__(self, m_o: int, r_o: int, m_i: int, r_i: int = 3):
        self.m_o, self.r_o, self.m_i, self.r_i = m_o, r_o, m_i, r_i
        self.ko = generate_kernel(m_o, r_o)
        self.ki = generate_kernel(m_i, r_i)
        self.l_o, self.l_i = self.ko.l, self.ki.l
        self.P = self.l_o * self.l_i                       # transform points per axis
        self.L = r_i * (self.l_o - 1) + self.l_i           # slice window
        self.M = m_o * m_i                                 # nominal outputs per slice
        self.reach = r_i * r_o                             # longest filter handled
        # coverage phases and tile advance (R5/#R6)
        if m_i >= r_i:
            self.shifts = [0]
            self.adv = r_i * (m_o - 1) + m_i
        else:
            self.shifts = list(range(0, r_i, m_i))
            self.adv = r_i * m_o

    def positions(self) -> List[int]:
        """Output position r_i*t + s of nominal output q = t*m_i + s."""
        return [self.r_i * t + s for t in range(self.m_o) for s in range(self.m_i)]

    def keep(self, phase: int) -> List[bool]:
        """Which nominal outputs of coverage phase ``phase`` are written."""
        sh = self.shifts[phase]
        out = []
        for t in range(self.m_o):
            for s in range(self.m_i):
                if self.m_i >= self.r_i:
                    out.append(s < self.r_i or t == self.m_o - 1)
                else:
                    out.append(sh + s < self.r_i)
        return out


# ----------------------------------------------------------------------------
# exact mode products on numpy object arrays
# ----------------------------------------------------------------------------
def _mat(M) -> np.ndarray:
    return np.array([[v for v in row] for row in M], dtype=object)


def mode_product(t: np.ndarray, M, axis: int) -> np.ndarray:
    """Multiply every mode-``axis`` fibre of t by matrix M (rows x t.shape[axis])."""
    Mo = _mat(M) if not isinstance(M, np.ndarray) else M
    r = np.tensordot(Mo, t, axes=([1], [axis]))       # new axis first
    return np.moveaxis(r, 0, axis)


class Counter:
    def __init__(self):
        self.mults = 0


def _zero_like(dtype):
    return Fraction(0) if dtype == "exact" else 0.0


# ----------------------------------------------------------------------------
# 1-D literal procedure (Fig. 3 example)
# ----------------------------------------------------------------------------
def nested_conv1d(x, w, m_o: int, m_i: int, r_o: int | None = None, r_i: int = 2,
                  counter: Counter | None = None, trace: list | None = None):
    """Valid 1-D correlation of x with w by the literal nested procedure.

    Defaults reproduce the paper's own example (F(2,2) at both levels).
    """
    R = len(w)
    if r_o is None:
        r_o = r_i
    ax = Axis(m_o, r_o, m_i, r_i)
    if R > ax.reach:
        raise ValueError("filter longer than r_i*r_o")
    n_out = len(x) - R + 1
    # step 1: filter reordered matrix (column distance r_i, zero-padded end)
    W = np.array([[Fraction(w[r_i * k1 + k0]) if r_i * k1 + k0 < R else Fraction(0)
                   for k1 in range(r_o)] for k0 in range(r_i)], dtype=object)
    U = _mat(ax.ki.G).dot(W).dot(_mat(ax.ko.G).T)
    y: List = [None] * n_out
    xs = list(x) + [0] * (ax.L + ax.adv)               # zero tail for ragged end
    for o in range(0, n_out, ax.adv):
        for ph, sh in enumerate(ax.shifts):
            org = o + sh
            # step 2: input reordered matrix, columns = inner-slide windows
            X = np.array([[Fraction(xs[org + r_i * j + s]) for j in range(ax.l_o)]
                          for s in range(ax.l_i)], dtype=object)
            if trace is not None:
                trace.append(("slice", org, X.copy()))
            V = _mat(ax.ki.BT).dot(X).dot(_mat(ax.ko.BT).T)
            # step 3: EWMM, output reordered matrix, scatter + discard
            Mx = U * V
            if counter is not None:
                counter.mults += Mx.size
            Y = _mat(ax.ki.AT).dot(Mx).dot(_mat(ax.ko.AT).T)   # [s][t]
            keep = ax.keep(ph)
            for t in range(m_o):
                for s in range(m_i):
                    q = t * m_i + s
                    pos = org + r_i * t + s
                    if keep[q] and pos < n_out and y[pos] is None:
                        y[pos] = Y[s][t]
    return y


# ----------------------------------------------------------------------------
# 2-D literal procedure, multichannel, stride 1, zero padding
# ----------------------------------------------------------------------------
def nested_conv2d(x, w, pad: int, m_o: int, m_i: int, r_o: int = 3, r_i: int = 3,
                  counter: Counter | None = None, exact: bool = True) -> np.ndarray:
    """y[n, o] = sum_c x[n, c] (*) w[o, c]  (Eq. 2.1, stride 1) via nested Winograd.

    x [N, C, H, W] and w [O, C, K, K] are integer/Fraction (exact=True) or float
    arrays.  Returns an object array (exact) or float64 array.  Each slice is
    transformed with mode products (B_i^T, B_o^T on each axis), the EWMM is
    counted, channels are summed in the transform domain, and the inverse
    transform A_i^T, A_o^T is scattered with the keep rule.
    """
    N, C, H, W_ = x.shape
    O, C2, K, K2 = w.shape
    assert C == C2 and K == K2
    ax = Axis(m_o, r_o, m_i, r_i)
    if K > ax.reach:
        raise ValueError("filter larger than r_i*r_o taps")
    Ho, Wo = H + 2 * pad - K + 1, W_ + 2 * pad - K + 1
    cast = (lambda v: Fraction(v)) if exact else (lambda v: float(v))
    dt = object if exact else np.float64

    def M(mat):
        return np.array([[cast(v) for v in row] for row in mat], dtype=dt)

    Gi, Go, BiT, BoT, AiT, AoT = (M(ax.ki.G), M(ax.ko.G), M(ax.ki.BT), M(ax.ko.BT),
                                  M(ax.ki.AT), M(ax.ko.AT))
    # step 1: rank-4 filter reordered tensor Wr[o, c, k0h, k1h, k0w, k1w]
    Wr = np.zeros((O, C, r_i, r_o, r_i, r_o), dtype=dt)
    if exact:
        Wr[...] = Fraction(0)
    for k1h in range(r_o):
        for k0h in range(r_i):
            kh = r_i * k1h + k0h
            if kh >= K:
                continue
            for k1w in range(r_o):
                for k0w in range(r_i):
                    kw = r_i * k1w + k0w
                    if kw >= K:
                        continue
                    for o in range(O):
                        for c in range(C):
                            Wr[o, c, k0h, k1h, k0w, k1w] = cast(w[o, c, kh, kw])
    U = Wr
    for a, Gm in ((2, Gi), (3, Go), (4, Gi), (5, Go)):
        U = mode_product(U, Gm, a)
    # padded input with a zero tail wide enough for the last slice window
    tail = ax.L + ax.adv
    xp = np.zeros((N, C, H + 2 * pad + tail, W_ + 2 * pad + tail), dtype=dt)
    if exact:
        xp[...] = Fraction(0)
    for n in range(N):
        for c in range(C):
            for i in range(H):
                for j in range(W_):
                    xp[n, c, pad + i, pad + j] = cast(x[n, c, i, j])
    y = np.zeros((N, O, Ho, Wo), dtype=dt)
    done = np.zeros((Ho, Wo), dtype=bool)
    idx_h = lambda org: [[org + r_i * j + s for j in range(ax.l_o)] for s in range(ax.l_i)]
    for n in range(N):
        done[...] = False
        for oh in range(0, Ho, ax.adv):
            for ow in range(0, Wo, ax.adv):
                for ph_h, sh_h in enumerate(ax.shifts):
                    for ph_w, sh_w in enumerate(ax.shifts):
                        orgh, orgw = oh + sh_h, ow + sh_w
                        # step 2: rank-4 input reordered tensor X[c, s_h, j_h, s_w, j_w]
                        ih = np.array(idx_h(orgh))
                        iw = np.array(idx_h(orgw))
                        X = xp[n][:, ih[:, :, None, None], iw[None, None, :, :]]
                        V = X
                        for a, Bm in ((1, BiT), (2, BoT), (3, BiT), (4, BoT)):
                            V = mode_product(V, Bm, a)
                        # step 3: EWMM + transform-domain channel sum
                        Msum = np.einsum("ocabde,cabde->oabde", U, V) if not exact else \
                            sum(U[:, c] * V[c][None] for c in range(C))
                        if counter is not None:
                            counter.mults += O * C * V[0].size
                        Y = Msum
                        for a, Am in ((1, AiT), (2, AoT), (3, AiT), (4, AoT)):
                            Y = mode_product(Y, Am, a)             # [o, s_h, t_h, s_w, t_w]
                        kh_, kw_ = ax.keep(ph_h), ax.keep(ph_w)
                        for th in range(m_o):
                            for s_h in range(m_i):
                                qh = th * m_i + s_h
                                ph_pos = orgh + r_i * th + s_h
                                if not kh_[qh] or ph_pos >= Ho:
                                    continue
                                for tw in range(m_o):
                                    for s_w in range(m_i):
                                        qw = tw * m_i + s_w
                                        pw_pos = orgw + r_i * tw + s_w
                                        if not kw_[qw] or pw_pos >= Wo:
                                            continue
                                        if done[ph_pos, pw_pos]:
                                            continue
                                        done[ph_pos, pw_pos] = True
                                        y[n, :, ph_pos, pw_pos] = Y[:, s_h, th, s_w, tw]
        assert done.all(), "coverage hole"
    return y


# ----------------------------------------------------------------------------
# composite per-axis matrices (the whole two-level algorithm as one F(.,.))
# ----------------------------------------------------------------------------
def composite(ax: Axis) -> Tuple[list, list, list, list]:
    """B^T_hat (P x L), G_hat (P x r_i*r_o), A^T_hat (M x P) and the gather list.

    Point index p = p_o*l_i + p_i, filter tap k = r_i*k1 + k0, nominal output
    q = t*m_i + s  (R4).  B^T_hat = (B_o^T (x) B_i^T) . Gather where
    Gather sends reordered-column entry (j, s) to slice input r_i*j + s;
    G_hat = G_o (x) G_i; A^T_hat = A_o^T (x) A_i^T.
    """
    BT_k = kron(ax.ko.BT, ax.ki.BT)            # P x (l_o*l_i)
    gather = [ax.r_i * j + s for j in range(ax.l_o) for s in range(ax.l_i)]
    BT = [[Fraction(0)] * ax.L for _ in range(ax.P)]
    for p in range(ax.P):
        for q, c in enumerate(gather):
            BT[p][c] += BT_k[p][q]
    G = kron(ax.ko.G, ax.ki.G)                 # P x (r_o*r_i), column k1*r_i + k0
    AT = kron(ax.ko.AT, ax.ki.AT)              # (m_o*m_i) x P
    return BT, G, AT, gather


# ----------------------------------------------------------------------------
# plan tables, written independently of the library (compared bit-exactly)
# ----------------------------------------------------------------------------
TABLE_BT, TABLE_G, TABLE_AT, TABLE_GATHER, TABLE_SCATTER, TABLE_ORIGINS, \
    TABLE_PHASE_TAPS, TABLE_DIMS = range(8)


def _frac_pairs(M) -> List[int]:
    out = []
    for row in M:
        for v in row:
            v = Fraction(v)
            g = gcd(v.numerator, v.denominator)
            out += [v.numerator // g, v.denominator // g]
    return out


def layer_geometry(K: int, stride: int, transposed: bool, pad: int, output_padding: int,
                   m_o: int, m_i: int, outer_taps: int, Cin: int, Cout: int):
    """Per-axis effective filter length, phase split and channel folding.

    stride 1: K' = K.  stride 2 forward (Eq. 2.7, R9): the
    s^2 input phases are stride-1 correlations with sub-filters w[2a+p] padded
    to K' = ceil(K/2) ("replace F(m,r') by F(m,r'+1) with zero padding"),
    summed -> folded into the contraction (Cin_e = 4 Cin).  Transposed stride 2
    (R11): 4 output phases, each a stride-1 correlation with flipped
    sub-sampled taps -> folded into the output channels (Cout_e = 4 Cout).
    outer_taps = 3 is the paper's fixed 3x3 tile grid; 0 = mixed ceil(K'/3)
    (R8).
    """
    if stride == 1:
        Kp = K
    elif not transposed:
        Kp = -(-K // 2)
    else:
        Kp = phase_taps(K, stride, True, pad)[2]
    r_o = outer_taps if outer_taps else max(1, -(-Kp // 3))
    cin_e = Cin * (4 if (stride == 2 and not transposed) else 1)
    cout_e = Cout * (4 if (stride == 2 and transposed) else 1)
    return Kp, r_o, cin_e, cout_e


def phase_taps(K: int, stride: int, transposed: bool, pad: int):
    """[mode, nphase, Kp, (offset, taps[Kp]) per phase] (see DESIGN.md tables).

    mode 0, stride 1:   y[i] = sum_d x[i + d - offset] w[taps[d]].
    mode 1, stride 2:   phase p: y[i] += sum_a x[2(i + a) + offset_p] w[taps_p[a]].
    mode 2, transposed: y[2j + phi] = sum_d x[j + d - offset_phi] w[taps_phi[d]].
    taps = -1 marks a zero tap.
    """
    if stride == 1:
        return [0, 1, K, pad] + list(range(K))
    Kp = -(-K // 2)
    out = [2 if transposed else 1, 2, Kp]
    if not transposed:
        for p in range(2):
            taps = [2 * a + p if 2 * a + p < K else -1 for a in range(Kp)]
            out += [p - pad] + taps
        return out
    # transposed: y[2j+phi] = sum_a x[j + c_phi - a] w[2a + rho], rho = (phi+pad)%2
    offs, tapl = [], []
    for phi in range(2):
        rho = (phi + pad) % 2
        c_phi = (phi + pad - rho) // 2
        offs.append(Kp - 1 - c_phi)
        tapl.append([2 * (Kp - 1 - d) + rho if 2 * (Kp - 1 - d) + rho < K else -1
                     for d in range(Kp)])
    # one common input window for both phases: shift the smaller-offset phase's
    # taps right (leading zero taps) so every phase reads x[j + d - max(offs)]
    omax, omin = max(offs), min(offs)
    Kq = Kp + omax - omin
    out[2] = Kq
    for phi in range(2):
        lead = omax - offs[phi]
        taps = [-1] * lead + tapl[phi]
        taps += [-1] * (Kq - len(taps))
        out += [omax] + taps
    return out


def plan_tables(K: int, stride: int, m_o: int, m_i: int, Cin: int, Cout: int,
                transposed: bool = False, pad: int = 0, outer_taps: int = 3) -> dict:
    """All integer tables of a plan, keyed by table id (compared with nw_plan_tables)."""
    Kp, r_o, cin_e, cout_e = layer_geometry(K, stride, transposed, pad, 0, m_o, m_i,
                                           outer_taps, Cin, Cout)
    ax = Axis(m_o, r_o, m_i, 3)
    if Kp > ax.reach:
        raise ValueError("filter larger than reach")
    BT, G, AT, gather = composite(ax)
    scatter = []
    pos = ax.positions()
    for ph, sh in enumerate(ax.shifts):
        kp = ax.keep(ph)
        for q in range(ax.M):
            scatter += [sh + pos[q], int(kp[q])]
    taps = phase_taps(K, stride, transposed, pad)
    dims = [K, stride, int(transposed), m_o, r_o, m_i, ax.l_o, ax.l_i, ax.P, ax.L, ax.M,
            ax.P * ax.P, Cin, Cout, cin_e, cout_e, taps[2], len(ax.shifts), ax.adv]
    return {
        TABLE_BT: _frac_pairs(BT),
        TABLE_G: _frac_pairs(G),
        TABLE_AT: _frac_pairs(AT),
        TABLE_GATHER: gather,
        TABLE_SCATTER: scatter,
        TABLE_ORIGINS: [ax.adv, len(ax.shifts)] + ax.shifts,
        TABLE_PHASE_TAPS: taps,
        TABLE_DIMS: dims,
    }


def composite_conv2d(x, w, pad: int, tables: dict, exact: bool = True) -> np.ndarray:
    """Stride-1 conv evaluated from the plan tables alone (composite form).

    Per slice at output origin (a_h*adv + shift_h, a_w*adv + shift_w):
    V = B^T_hat X B_hat on the L x L input window, U = G_hat W G_hat^T on the
    zero-padded r_i*r_o square filter, M = sum_c U (.) V, Y = A^T_hat M A_hat,
    then the scatter/keep table places Y.  Equal to nested_conv2d because
    B^T_hat = (B_o^T (x) B_i^T) . Gather etc. (Eq. 2.5 -> 2.6).
    """
    dims = tables[TABLE_DIMS]
    P_a, L, M_a = dims[8], dims[9], dims[10]
    r_o = dims[4]
    R = 3 * r_o

    def F(flat, rows, cols):
        vals = [Fraction(flat[2 * i], flat[2 * i + 1]) for i in range(rows * cols)]
        if not exact:
            vals = [float(v) for v in vals]
        return np.array(vals, dtype=object if exact else np.float64).reshape(rows, cols)

    BT, G, AT = F(tables[TABLE_BT], P_a, L), F(tables[TABLE_G], P_a, R), F(tables[TABLE_AT], M_a, P_a)
    adv, nph = tables[TABLE_ORIGINS][0], tables[TABLE_ORIGINS][1]
    shifts = tables[TABLE_ORIGINS][2:2 + nph]
    sc = tables[TABLE_SCATTER]
    N, C, H, W_ = x.shape
    O, _, K, _ = w.shape
    Ho, Wo = H + 2 * pad - K + 1, W_ + 2 * pad - K + 1
    dt = object if exact else np.float64
    cast = Fraction if exact else float
    wz = np.zeros((O, C, R, R), dtype=dt)
    if exact:
        wz[...] = Fraction(0)
    wz[:, :, :K, :K] = np.vectorize(cast, otypes=[dt])(w)
    U = np.array([[G.dot(wz[o, c]).dot(G.T) for c in range(C)] for o in range(O)], dtype=dt)
    ext = L + adv
    xp = np.zeros((N, C, H + 2 * pad + ext, W_ + 2 * pad + ext), dtype=dt)
    if exact:
        xp[...] = Fraction(0)
    xp[:, :, pad:pad + H, pad:pad + W_] = np.vectorize(cast, otypes=[dt])(x)
    y = np.zeros((N, O, Ho, Wo), dtype=dt)
    for n in range(N):
        for a_h in range(0, Ho, adv):
            for a_w in range(0, Wo, adv):
                for ph in range(nph):
                    for pw in range(nph):
                        oh, ow = a_h + shifts[ph], a_w + shifts[pw]
                        X = xp[n, :, oh:oh + L, ow:ow + L]
                        V = np.array([BT.dot(X[c]).dot(BT.T) for c in range(C)], dtype=dt)
                        Msum = sum(U[:, c] * V[c][None] for c in range(C))
                        Y = np.array([AT.dot(Msum[o]).dot(AT.T) for o in range(O)], dtype=dt)
                        for qh in range(M_a):
                            posh, kh = sc[2 * (ph * M_a + qh)], sc[2 * (ph * M_a + qh) + 1]
                            if not kh or a_h + posh >= Ho:
                                continue
                            for qw in range(M_a):
                                posw, kw = sc[2 * (pw * M_a + qw)], sc[2 * (pw * M_a + qw) + 1]
                                if not kw or a_w + posw >= Wo:
                                    continue
                                y[n, :, a_h + posh, a_w + posw] = Y[:, qh, qw]
    return y
