"""Operand-rounding emulation for error prediction.  TEST INFRASTRUCTURE ONLY.

The paper fixes no floating-point format for its GPU-free method (Table II is
16-bit fixed point on an FPGA); BASELINE's tolerances gate the build
(R12).  These helpers emulate the tensor-core operand formats on the
CPU so predicted errors can be compared with measured ones:
  bf16 (round to nearest even), tf32 (round to nearest, ties away: cvt.rna),
  and the split v = hi + lo with hi = bf16(v), lo = bf16(v - hi).
Informative only, not a pass gate.  Pins: bf16 rounding equals torch's
float32 -> bfloat16 cast bit for bit; hi + lo reproduces v to 2^-16 relative.
"""
from __future__ import annotations

import numpy as np


def round_bf16(a) -> np.ndarray:
    """float32 -> nearest bfloat16 (RNE), returned as float32."""
    u = np.asarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def round_tf32(a) -> np.ndarray:
    """float32 -> tf32 (10-bit mantissa), round to nearest, ties away from zero."""
    u = np.asarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x1000) >> 13) << 13
    return r.astype(np.uint32).view(np.float32)


def split_bf16(a):
    """v -> (hi, lo) with hi = bf16(v), lo = bf16(v - hi) (R12)."""
    a = np.asarray(a, dtype=np.float32)
    hi = round_bf16(a)
    lo = round_bf16(a - hi)
    return hi, lo


def rel_err(y, ref) -> float:
    """BASELINE metric: max |y - y_ref| / max |y_ref| (R14)."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(y - ref)) / np.max(np.abs(ref)))
