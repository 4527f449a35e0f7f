"""GPU parity over geometries beyond the five BASELINE configs: filter sizes 3..9 (and 11..17 at
stride 2, K <= 9 per phase), stride 1 / 2, transposed stride 2 with output_padding 0 / 1, odd
pads, non-square images, every nested kernel built (m_o = 3, 4, 5 with inner F(3,3); F(2,3) (x) F(2,3)
with coverage phases), in FP32 and bf16x3, against the FP64 oracle (Eq. 2.1 / its transposed form)."""
import numpy as np
import pytest
import torch

import synth
from oracle import direct
from oracle.errstudy import rel_err
from test_gpu_nested import TOL, _math

pytestmark = pytest.mark.gpu

GEOMS = [
    # K, stride, pad, transposed, output_padding, m_o, m_i
    (3, 1, 1, False, 0, 3, 3),
    (4, 1, 1, False, 0, 3, 3),
    (6, 1, 2, False, 0, 4, 3),
    (8, 1, 4, False, 0, 5, 3),
    (5, 1, 0, False, 0, 3, 3),
    (9, 1, 1, False, 0, 4, 3),
    (5, 2, 2, False, 0, 3, 3),
    (7, 2, 1, False, 0, 4, 3),
    (11, 2, 5, False, 0, 3, 3),
    (17, 2, 8, False, 0, 4, 3),
    (3, 2, 1, True, 1, 3, 3),
    (5, 2, 2, True, 1, 4, 3),
    (7, 2, 3, True, 0, 3, 3),
    (9, 2, 4, True, 0, 4, 3),
    (7, 1, 3, False, 0, 2, 2),
]


def _case(K, stride, pad, transposed, op, m_o, m_i, seed):
    layer = synth.Layer(f"g{K}_{stride}_{pad}_{int(transposed)}", 2, 6, 5, 23, 17, K, stride, pad,
                        transposed=transposed, output_padding=op, m_o=m_o, m_i=m_i,
                        xdist="unif11", wdist="unif11", seed=seed)
    return layer


@pytest.mark.parametrize("math", ["fp32", "bf16x3"])
@pytest.mark.parametrize("K,stride,pad,tr,op,m_o,m_i", GEOMS)
def test_geometry(K, stride, pad, tr, op, m_o, m_i, math):
    from paper_2102_13272_b200 import NestedConv2d
    layer = _case(K, stride, pad, tr, op, m_o, m_i, seed=100 + K)
    t = synth.make_inputs(layer)
    conv = NestedConv2d(t["w"].cuda(), stride, pad, m_o, m_i, _math(math), transposed=tr, output_padding=op)
    y = conv(t["x"].cuda()).cpu().numpy()
    x64, w64 = t["x"].double().numpy(), t["w"].double().numpy()
    ref = direct.conv_transpose2d(x64, w64, stride, pad, op) if tr else direct.conv2d(x64, w64, stride, pad)
    assert y.shape == ref.shape
    assert np.isfinite(y).all()
    assert rel_err(y, ref) <= TOL[math]
