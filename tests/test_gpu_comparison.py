"""GPU parity of the comparison paths through the C ABI against the FP64 oracle.

nw_conv_ola     OLA-Winograd (Eq. 2.3): single-level F(3,3) per 3x3 filter block, blocks summed
nw_conv_direct  native convolution (Eq. 2.1) as an implicit GEMM
Both run in the plan's math mode; the gates are the nested path's (BASELINE north_star):
1e-4 for FP32 SIMT, 5e-3 for the bf16x3 tensor-core mode.
"""
import numpy as np
import pytest
import torch

import synth
from oracle.errstudy import rel_err
from test_gpu_nested import SMALL, TOL, _math, _ref, check_parity

pytestmark = pytest.mark.gpu


def _run(layer, math, path):
    from paper_2102_13272_b200 import NestedConv2d
    t = synth.make_inputs(layer)
    x, w = t["x"].cuda(), t["w"].cuda()
    slopes = torch.full((layer.Cout,), synth.PRELU_SLOPE, device="cuda") if layer.prelu else None
    conv = NestedConv2d(w, layer.stride, layer.pad, layer.m_o, layer.m_i, _math(math), outer_taps=layer.r_o,
                        transposed=layer.transposed, output_padding=layer.output_padding,
                        prelu_slopes=slopes)
    y = conv(x, path=path)
    torch.cuda.synchronize()
    return t, y.float().cpu().numpy()


@pytest.mark.parametrize("path", ["ola", "direct"])
@pytest.mark.parametrize("math", ["fp32", "bf16x3"])
@pytest.mark.parametrize("name", list(SMALL))
def test_comparison_path_parity(name, math, path):
    layer = SMALL[name]
    t, y = _run(layer, math, path)
    ref = _ref(layer, t)
    check_parity(y, ref, math, layer.dtype)


@pytest.mark.parametrize("N,H,W", [(1, 1, 1), (2, 10, 37), (1, 64, 5)])
def test_comparison_edges(N, H, W):
    layer = synth.small(synth.CONFIGS["c2k9"], N=N, H=H, W=W, Cin=16, Cout=32)
    for path in ("ola", "direct"):
        t, y = _run(layer, "bf16x3", path)
        assert rel_err(y, _ref(layer, t)) <= TOL["bf16x3"], path


def test_three_paths_agree():
    # nested, OLA and direct compute the same convolution (Eq. 2.1); in FP32 they agree to rounding
    layer = SMALL["c2k7"]
    ys = [_run(layer, "fp32", p)[1] for p in ("nested", "ola", "direct")]
    scale = np.abs(ys[2]).max()
    assert np.abs(ys[0] - ys[2]).max() / scale < 5e-5   # nested FP32 rounding grows with the outer tile (R20)
    assert np.abs(ys[1] - ys[2]).max() / scale < 1e-5
