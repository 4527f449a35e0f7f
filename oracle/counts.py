"""Closed-form EWMM multiplication counts.  TEST INFRASTRUCTURE ONLY.

P:110: an n-dimensional nested Winograd "consumes l^n multiplications and
produce[s] m^n outputs for each input vector slice"; transform arithmetic is
additions / constant multiplications and is not counted (Winograd's
convention).  Per spatial axis (exact Fractions):

  native (Eq. 2.1)            R
  direct Winograd F(m, R)     (m + R - 1) / m
  OLA-Winograd F(m, r)        ceil(R/r) * l / m                     (Eq. 2.3)
  nested F(m_o,r_o)(x)F(m_i,r_i)  n_phases * l_o * l_i / advance    (P:110 + DESIGN.md#R5/#R6)

2-D counts are the squares; a whole layer multiplies the per-slice count by the
number of slices and by Cin * Cout.

Pins (tests/test_oracle_counts.py): Eq. 2.3 / P:58 (12 vs 9 multiplications
for R = 4 with F(2,2)); Table I's measured GOPs ratios 1.43 (5x5) and 3.29
(9x9) within 3% of the analytic 1.44 and 3.24; agreement with the
instrumented counters of oracle.nested / oracle.ola (exact integers); the
qualitative claims of P:148.  The "+2.2%" of P:148 for F(6,3) on 5x5 is
**parity unpinned** (figure 7 is missing; this module gives +30.6% for the
same kernel at both levels and 0% with a mixed outer kernel, R17).
"""
from __future__ import annotations

from fractions import Fraction

from .nested import Axis


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def native_per_axis(R: int) -> Fraction:
    return Fraction(R)


def direct_winograd_per_axis(R: int, m: int) -> Fraction:
    return Fraction(m + R - 1, m)


def ola_per_axis(R: int, m: int, r: int) -> Fraction:
    return Fraction(ceil_div(R, r) * (m + r - 1), m)


def nested_per_axis(m_o: int, r_o: int, m_i: int, r_i: int) -> Fraction:
    ax = Axis(m_o, r_o, m_i, r_i)
    return Fraction(len(ax.shifts) * ax.P, ax.adv)


def nested_same_kernel_per_axis(R: int, m: int, r: int) -> Fraction:
    """SPEC-style d-level nesting with the same F(m, r) at every level, d = ceil(log_r R),
    distinct outputs O_d (O_1 = m, O_j = (m-1) r^(j-1) + O_(j-1)), valid for m >= r."""
    d, reach = 1, r
    while reach < R:
        d += 1
        reach *= r
    if m < r and d > 1:
        # holes: use the coverage-phase construction of oracle.nested (2 levels)
        assert d == 2
        return nested_per_axis(m, r, m, r)
    O = m
    for j in range(2, d + 1):
        O = (m - 1) * r ** (j - 1) + O
    return Fraction((m + r - 1) ** d, O)


def per_output_2d(per_axis: Fraction) -> Fraction:
    return per_axis * per_axis


def layer_ewmm_nested(N: int, Ho: int, Wo: int, cin_e: int, cout_e: int,
                      m_o: int, r_o: int, m_i: int, r_i: int = 3) -> int:
    """EWMM multiplications of one nested layer: slices * P * Cin_e * Cout_e."""
    ax = Axis(m_o, r_o, m_i, r_i)
    tiles = ceil_div(Ho, ax.adv) * ceil_div(Wo, ax.adv)
    slices = N * tiles * len(ax.shifts) ** 2
    return slices * ax.P * ax.P * cin_e * cout_e


def layer_ewmm_ola(N: int, Ho: int, Wo: int, cin: int, cout: int, K: int, m: int, r: int = 3) -> int:
    tiles = ceil_div(Ho, m) * ceil_div(Wo, m)
    nb = ceil_div(K, r)
    return N * tiles * nb * nb * (m + r - 1) ** 2 * cin * cout


def direct_flops(N: int, Ho: int, Wo: int, cin: int, cout: int, K: int) -> int:
    """Direct-equivalent FLOPs 2 * MACs of Eq. 2.1 (the paper's GOPs numerator
    counts #mult + #add of native convolution)."""
    return 2 * N * Ho * Wo * cin * cout * K * K
