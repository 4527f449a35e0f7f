#!/usr/bin/env python
"""Time one BASELINE layer with another nesting (e.g. outer F(5,2) for C2 K=5):
    python tools/time_plan.py c2k5 5 0      # layer, m_outer, outer_taps (0 = ceil(K'/3))"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2102_13272_b200 as nw  # noqa: E402
import synth  # noqa: E402

name, m_o, r_o = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
l = synth.CONFIGS[name].with_(m_o=m_o, r_o=r_o)
t = synth.make_inputs(l)
conv = nw.NestedConv2d(t["w"].cuda(), l.stride, l.pad, l.m_o, l.m_i, nw.MATH_BF16X3, transposed=l.transposed,
                       outer_taps=l.r_o, output_padding=l.output_padding)
x = t["x"].cuda()
y = torch.empty(conv.out_shape(x.shape), dtype=x.dtype, device="cuda")
for _ in range(3):
    conv(x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    conv(x, y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"{name} F({m_o},{r_o or 'mixed'}): {ms:.4f} ms  {l.direct_flops() / ms / 1e9:.1f} TFLOP/s  info {conv.info['points']} pts")
from paper_2102_13272_b200 import _lib  # noqa: E402
_lib.profile_begin()
for _ in range(5):
    conv(x, y)
torch.cuda.synchronize()
prof = _lib.profile_end()
print("   ", {k: round(v[1] / v[0], 4) for k, v in prof.items()})
