#!/usr/bin/env python
"""Streamed-pipeline experiment: time layers and hash their outputs under the current NW_STREAM*
environment (compare the hashes across runs: the streamed path must be bit-identical).
python tools/stream_exp.py c2k9 c2k5"""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2102_13272_b200 as nw  # noqa: E402
import synth  # noqa: E402

tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("NW_"))
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
    h = hashlib.sha1(y.view(torch.int16 if y.dtype == torch.bfloat16 else torch.int32).cpu().numpy().tobytes()).hexdigest()[:12]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 20
    e0.record()
    for _ in range(R):
        conv(x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    h2 = hashlib.sha1(y.view(torch.int16 if y.dtype == torch.bfloat16 else torch.int32).cpu().numpy().tobytes()).hexdigest()[:12]
    from paper_2102_13272_b200 import _lib
    _lib.profile_begin()
    for _ in range(5):
        conv(x, y)
    torch.cuda.synchronize()
    prof = _lib.profile_end()
    ks = {k: round(v[1] / v[0], 4) for k, v in prof.items()}
    print(f"{name} [{tag}]: {ms:.4f} ms {l.direct_flops() / ms / 1e9:.1f} TFLOP/s hash {h} {'' if h == h2 else 'UNSTABLE ' + h2} {ks}",
          flush=True)
