"""Helper for tests/test_gpu_env_variants.py: run one layer through the C ABI in a fresh
process (environment tunables are read once per process) and save y to argv[2].

usage: python tests/_variant_run.py <json layer spec> <out.npy> [host]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2102_13272_b200 import MATH_BF16X3, MATH_FP32_SIMT, NestedConv2d  # noqa: E402

spec = json.loads(sys.argv[1])
base = synth.CONFIGS[spec.pop("config")]
math = {"bf16x3": MATH_BF16X3, "fp32": MATH_FP32_SIMT}[spec.pop("math", "bf16x3")]
extra = {k: spec.pop(k) for k in ("m_o", "r_o", "dtype", "xdist") if k in spec}
layer = synth.small(base, **spec) if spec else base
if extra:
    layer = layer.with_(**extra)
t = synth.make_inputs(layer)
slopes = torch.full((layer.Cout,), synth.PRELU_SLOPE, device="cuda") if layer.prelu else None
conv = NestedConv2d(t["w"].cuda(), layer.stride, layer.pad, layer.m_o, layer.m_i, math, outer_taps=layer.r_o,
                    transposed=layer.transposed, output_padding=layer.output_padding, prelu_slopes=slopes)
if len(sys.argv) > 3 and sys.argv[3] == "host":
    # the bench's e2e entry point: pinned host x -> device -> forward -> host y (nw_conv_forward_host)
    N, H, W = layer.N, layer.H, layer.W
    hx = t["x"].pin_memory()
    hy = torch.empty(conv.out_shape(hx.shape), dtype=hx.dtype).pin_memory()
    nbytes = conv.plan.workspace_size(N, H, W, "host")
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    conv.plan.forward_host(hx, conv.U, hy, N, H, W, ws, nbytes)
    torch.cuda.synchronize()
    y = hy
else:
    y = conv(t["x"].cuda())
    torch.cuda.synchronize()
np.save(sys.argv[2], y.float().cpu().numpy())
