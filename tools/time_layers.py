#!/usr/bin/env python
"""Time nw_conv_forward per layer without per-kernel profiling events (CUDA events around
R back-to-back calls), e.g. to compare launch settings: python tools/time_layers.py c2k5 c2k7 c2k9"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2102_13272_b200 as nw  # noqa: E402
import synth  # noqa: E402

tot = 0.0
for name in sys.argv[1:]:
    l = synth.CONFIGS[name]
    t = synth.make_inputs(l)
    conv = nw.NestedConv2d(t["w"].cuda(), l.stride, l.pad, l.m_o, l.m_i, nw.MATH_BF16X3, transposed=l.transposed,
                           outer_taps=l.r_o, output_padding=l.output_padding)
    x = t["x"].cuda()
    y = torch.empty(conv.out_shape(x.shape), dtype=x.dtype, device="cuda")
    for _ in range(3):
        conv(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 20
    e0.record()
    for _ in range(R):
        conv(x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    tot += ms
    print(f"{name}: {ms:.4f} ms  {l.direct_flops() / ms / 1e9:.1f} TFLOP/s")
    if os.environ.get("KERNELS"):
        from paper_2102_13272_b200 import _lib
        _lib.profile_begin()
        for _ in range(5):
            conv(x, y)
        torch.cuda.synchronize()
        prof = _lib.profile_end()
        print("   ", {k: round(v[1] / v[0], 4) for k, v in prof.items()})
print(f"total {tot:.4f} ms")
