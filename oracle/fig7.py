"""Fig. 7 sweep: multiplication complexity of nested, OLA- and direct Winograd.
TEST INFRASTRUCTURE ONLY (oracle; no GPU code).

Section V.A: "We simulated 2D convolutions with different filter
sizes ranging from 3x3 to 12x12 with four different Winograd kernels -- F(2,2),
F(3,3), F(4,4) and F(6,3)", comparing the nested Winograd, the OLA-Winograd and
the "direct Winograd, which directly uses F(m, r) with a varying r".  The figure
itself is missing from the text, so its values are not available; this
module recomputes the table from the counting conventions written out in
oracle.counts (EWMM multiplications only, transforms are additions and constant
multiplications):

  direct Winograd F(m, R)   (m + R - 1)^2 multiplications per m^2 outputs
  OLA F(m, r)               ceil(R/r)^2 blocks x (m + r - 1)^2 per m^2 outputs (Eq. 2.3)
  nested F(m, r)^(x)d       l^(2d) per O_d^2 outputs, d = ceil(log_r R) levels of the same
                            kernel, O_d the contiguous distinct outputs (oracle.multilevel)

(R23 states the direct-Winograd reading: F(m, R) with the sweep
kernel's m; the paper's restriction "not using the Winograd kernel larger than
the nested Winograd" bounds its tile to the nested composite, which every cell
here satisfies, see fig7_rows' `direct_l_le_nested` column.)

Pins (tests/test_oracle_fig7.py): every cell's per-tile count equals the
instrumented counter of an exact evaluation (oracle.multilevel.conv1d squared,
oracle.nested / oracle.ola counters) where one exists; R <= r degenerates to one
value for all three methods; the paper's qualitative claims of P:146-148
(nested <= OLA for F(2,2) and F(3,3), the gap grows with R, direct Winograd is
the cheapest of the three for F(6,3) on 5x5).  The "+2.2%" cell stays parity
unpinned (R17).
"""
from __future__ import annotations

import csv
import io
from fractions import Fraction
from math import ceil
from typing import Dict, List

from .multilevel import depth_for, levels

KERNELS = [(2, 2), (3, 3), (4, 4), (6, 3)]
SIDES = list(range(3, 13))
METHODS = ["nested", "ola", "direct"]
CSV_FIELDS = ["method", "filter_side", "kernel_m", "kernel_r", "dims", "levels", "mults_per_tile",
              "outputs_per_tile", "mults_per_output", "mults_per_output_float", "direct_l_le_nested"]


def cell(method: str, R: int, m: int, r: int) -> Dict:
    """One 2-D cell: per-tile multiplications and outputs (exact)."""
    if method == "direct":
        l = m + R - 1
        per_tile, outs, d = l * l, m * m, 1
    elif method == "ola":
        nb = ceil(R / r)
        l = m + r - 1
        per_tile, outs, d = nb * nb * l * l, m * m, 1
    elif method == "nested":
        d = depth_for(R, r)
        a = levels(m, r, d)
        adv = a.advance()
        per_tile, outs = a.P * a.P, adv * adv
    else:
        raise ValueError(method)
    nested_L = levels(m, r, depth_for(R, r)).P
    return {"method": method, "filter_side": R, "kernel_m": m, "kernel_r": r, "dims": 2, "levels": d,
            "mults_per_tile": per_tile, "outputs_per_tile": outs,
            "mults_per_output": Fraction(per_tile, outs),
            "direct_l_le_nested": (m + R - 1) <= nested_L}


def sweep() -> List[Dict]:
    """The full 10 x 4 x 3 table of section V.A."""
    return [cell(meth, R, m, r) for (m, r) in KERNELS for R in SIDES for meth in METHODS]


def to_csv(rows: List[Dict]) -> str:
    out = io.StringIO()
    w = csv.writer(out, lineterminator="\n")
    w.writerow(CSV_FIELDS)
    for c in rows:
        mpo = c["mults_per_output"]
        w.writerow([c["method"], c["filter_side"], c["kernel_m"], c["kernel_r"], c["dims"], c["levels"],
                    c["mults_per_tile"], c["outputs_per_tile"], f"{mpo.numerator}/{mpo.denominator}",
                    f"{float(mpo):.6f}", int(c["direct_l_le_nested"])])
    return out.getvalue()


if __name__ == "__main__":
    print(to_csv(sweep()), end="")
