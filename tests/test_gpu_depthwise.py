"""GPU parity of the depthwise path (Table I's PNASNet depthwise 7x7 row; SURVEY 8(f)
rank 2) against the FP64 depthwise oracle: nested transforms with the per-channel
transform-domain product (csrc/depthwise.cu), and the OLA / direct comparison paths with
their per-channel block / tap sums.  Same gates as every layer (BASELINE tolerances)."""
import numpy as np
import pytest
import torch

import synth
from oracle import direct
from test_gpu_nested import _math, check_parity

pytestmark = pytest.mark.gpu


def _run(layer, math, path="nested"):
    from paper_2102_13272_b200 import NestedConv2d
    t = synth.make_inputs(layer)
    conv = NestedConv2d(t["w"].cuda(), 1, layer.pad, layer.m_o, layer.m_i, _math(math), outer_taps=layer.r_o,
                        depthwise=True)
    y = conv(t["x"].cuda(), path=path)
    torch.cuda.synchronize()
    ref = direct.conv2d_depthwise(t["x"].double().numpy(), t["w"].double().numpy(), 1, layer.pad)
    return y.float().cpu().numpy(), ref, conv


SMALL = synth.small(synth.CONFIGS["t1_pnas_dw7"], N=2, H=37, W=41)


@pytest.mark.parametrize("math", ["fp32", "bf16x3"])
@pytest.mark.parametrize("path", ["nested", "ola", "direct"])
def test_depthwise_parity(math, path):
    y, ref, _ = _run(SMALL, math, path)
    check_parity(y, ref, math, SMALL.dtype)


@pytest.mark.parametrize("shape", [dict(N=1, H=1, W=1), dict(N=3, H=12, W=12), dict(N=2, H=83, W=83, Cin=16, Cout=16),
                                   dict(N=1, H=25, W=64, Cin=130, Cout=130)])
def test_depthwise_edges_and_channel_counts(shape):
    # single pixel, one exact tile, the full image size with a channel count at the 16-granule,
    # and more channels than one 128-channel tile row... (130 -> cin_pad 144)
    layer = synth.small(synth.CONFIGS["t1_pnas_dw7"], **shape)
    y, ref, _ = _run(layer, "bf16x3")
    check_parity(y, ref, "bf16x3", layer.dtype)


@pytest.mark.parametrize("K,m_o,r_o", [(5, 4, 0), (9, 3, 3), (3, 4, 3)])
def test_depthwise_other_filters(K, m_o, r_o):
    layer = synth.small(synth.CONFIGS["t1_pnas_dw7"], N=2, H=30, W=27).with_(K=K, pad=K // 2, m_o=m_o, r_o=r_o)
    y, ref, _ = _run(layer, "bf16x3")
    check_parity(y, ref, "bf16x3", layer.dtype)


def test_depthwise_full_size():
    layer = synth.CONFIGS["t1_pnas_dw7"]
    for math in ("bf16x3", "fp32"):
        y, ref, conv = _run(layer, math)
        check_parity(y, ref, math, layer.dtype)
    assert conv.plan.count_mults(layer.N, layer.H, layer.W) == 8 * 7 * 7 * 900 * 54
