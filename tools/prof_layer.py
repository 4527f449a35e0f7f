#!/usr/bin/env python
"""Run one BASELINE layer through nw_conv_forward a few times (for ncu captures).

    python tools/prof_layer.py c2k9 [--math bf16x3|fp32|bf16] [--path nested|ola|direct] [--iters 4]

Exits 0 after a synchronising check that the output is finite; prints the
CUDA-event time of the last iteration (never a bench value when run under ncu).
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2102_13272_b200 as nw  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("layer")
    ap.add_argument("--math", default="bf16x3", choices=["bf16x3", "fp32", "bf16"])
    ap.add_argument("--path", default="nested", choices=["nested", "ola", "direct"])
    ap.add_argument("--iters", type=int, default=4)
    a = ap.parse_args()
    l = synth.CONFIGS[a.layer]
    math = {"bf16x3": nw.MATH_BF16X3, "fp32": nw.MATH_FP32_SIMT, "bf16": nw.MATH_BF16}[a.math]
    t = synth.make_inputs(l)
    w, x = t["w"].cuda(), t["x"].cuda()
    slopes = torch.full((l.Cout,), synth.PRELU_SLOPE, device="cuda") if l.prelu else None
    conv = nw.NestedConv2d(w, l.stride, l.pad, l.m_o, l.m_i, math, transposed=l.transposed, outer_taps=l.r_o,
                           output_padding=l.output_padding, prelu_slopes=slopes, depthwise=l.depthwise)
    y = torch.empty(conv.out_shape(x.shape), dtype=x.dtype, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(a.iters):
        e0.record()
        conv(x, y, path=a.path)
        e1.record()
    torch.cuda.synchronize()
    assert torch.isfinite(y).all().item()
    print(f"{a.layer} {a.path} {a.math}: {e0.elapsed_time(e1):.4f} ms (last iteration)")


if __name__ == "__main__":
    main()
