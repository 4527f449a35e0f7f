"""GPU parity of the single-kernel path for layers with at most four contraction outputs
(fused_smallout.cuh): BASELINE config 5's 9x9 stride-2 deconvolution (Cout_e = 4 output
phases) and Table I's SRCNN 5x5 1 <- 32, against the FP64 oracle; plus ragged slice counts,
P_a = 25 and 30 plans, Cout_e = 1..4, bf16 storage and the FP32 math mode."""
import pytest
import torch

import synth
from test_gpu_nested import _math, _ref, _run, check_parity

pytestmark = pytest.mark.gpu

# x rows are 16-byte multiples (the kernel loads its windows by TMA); tile rows with fewer
# tiles than a chunk, with more, and ragged last chunks
CASES = {
    "c5_deconv": synth.small(synth.CONFIGS["c5_deconv"], N=2, H=27, W=44),            # F(4,2)(x)F(3,3), 4 phases
    "c5_deconv_wide": synth.small(synth.CONFIGS["c5_deconv"], N=1, H=13, W=200),
    "c5_deconv_tiny": synth.small(synth.CONFIGS["c5_deconv"], N=1, H=5, W=4),
    "srcnn5b": synth.small(synth.CONFIGS["t1_srcnn5b"], N=2, H=37, W=160),            # 32 -> 1, 14 tiles a row
    "k9_cout3": synth.small(synth.CONFIGS["c2k9"], N=2, H=31, W=132, Cin=48, Cout=3),  # F(4,3)(x)F(3,3): P_a 30
    "k7_cout2_m3": synth.small(synth.CONFIGS["c2k7"], N=3, H=26, W=36, Cin=20, Cout=2).with_(m_o=3),
    "k5_cout4_bf16": synth.small(synth.CONFIGS["c2k5"], N=2, H=40, W=24, Cin=64, Cout=4).with_(dtype="bf16"),
    "k9_cout1_cin2": synth.small(synth.CONFIGS["c2k9"], N=1, H=50, W=52, Cin=2, Cout=1),
}


@pytest.mark.parametrize("math", ["bf16x3", "fp32"])
@pytest.mark.parametrize("name", list(CASES))
def test_fused_small_output_parity(name, math):
    layer = CASES[name]
    from paper_2102_13272_b200 import NestedConv2d
    t = synth.make_inputs(layer)
    conv = NestedConv2d(t["w"].cuda(), layer.stride, layer.pad, layer.m_o, layer.m_i, _math(math),
                        outer_taps=layer.r_o, transposed=layer.transposed, output_padding=layer.output_padding)
    assert conv.info["single_kernel"] == 1, conv.info
    y = conv(t["x"].cuda())
    torch.cuda.synchronize()
    check_parity(y.float().cpu().numpy(), _ref(layer, t), math, layer.dtype)


def test_unaligned_rows_take_the_three_kernel_path():
    # W * 4 bytes not a multiple of 16: no TMA windows, the regular pipeline runs (same gate)
    layer = synth.small(synth.CONFIGS["c5_deconv"], N=1, H=19, W=23)
    t, y = _run(layer, "bf16x3")
    check_parity(y, _ref(layer, t), "bf16x3", layer.dtype)

# the full-size C5 deconvolution runs this kernel in test_gpu_fullsize.py::test_full_size_full_tensor
