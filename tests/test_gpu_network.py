"""The FSRCNN-s-shaped network of BASELINE configs[4] run as a chain through the C ABI (conv1 5x5
and the 9x9 stride-2 deconv on the nested path, the 1x1 / 3x3 layers on the direct path, PReLU
fused into every store but the last) against the FP64 oracle chain, at a reduced image size."""
import numpy as np
import pytest
import torch

import synth
from oracle import direct
from oracle.errstudy import rel_err
from test_gpu_nested import TOL, _math

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("math", ["fp32", "bf16x3"])
def test_fsrcnn_chain(math):
    from paper_2102_13272_b200 import NestedConv2d
    layers = [synth.small(synth.CONFIGS[n], N=2, H=27, W=34) for n in synth.C5_NET]
    x0 = synth.make_inputs(layers[0])["x"]
    xg, xr = x0.cuda(), x0.double().numpy()
    for l in layers:
        w = synth.make_inputs(l, x=False)["w"]
        slopes = torch.full((l.Cout,), synth.PRELU_SLOPE, device="cuda") if l.prelu else None
        conv = NestedConv2d(w.cuda(), l.stride, l.pad, l.m_o, l.m_i, _math(math), transposed=l.transposed,
                            outer_taps=l.r_o, output_padding=l.output_padding, prelu_slopes=slopes)
        xg = conv(xg, path="direct" if l.K <= 3 else "nested")
        w64 = w.double().numpy()
        xr = (direct.conv_transpose2d(xr, w64, l.stride, l.pad, l.output_padding) if l.transposed
              else direct.conv2d(xr, w64, l.stride, l.pad))
        if l.prelu:
            xr = np.where(xr >= 0, xr, synth.PRELU_SLOPE * xr)
    y = xg.cpu().numpy()
    assert y.shape == (2, 1, 54, 68)
    # five layers compound the per-layer rounding; the per-layer gate applies to the chain
    assert rel_err(y, xr) <= TOL[math]
