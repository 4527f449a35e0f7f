"""GPU parity of the nested-Winograd path (through the C ABI) against the FP64 oracle.

Metric (BASELINE north_star, R14): max|y - y_ref| / max|y_ref| with
y_ref = oracle.direct in float64 from the stored (cast) x and w.
Tolerances: 1e-4 for the FP32 CUDA-core path, 5e-3 for the tensor-core path.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import direct
from oracle.errstudy import rel_err
from oracle.phases import conv_transpose2d_phases

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "bf16x3": 5e-3}


def bf16_half_ulp(v):
    """Largest rounding error of a round-to-nearest bf16 store of a value of magnitude v:
    half the bf16 spacing 2^(floor(log2 v) - 7), i.e. 2^(floor(log2 v) - 8) (8 significant bits)."""
    v = np.maximum(np.abs(np.asarray(v, dtype=np.float64)), np.finfo(np.float64).tiny)
    return np.ldexp(1.0, (np.floor(np.log2(v)) - 8).astype(np.int64))


def check_parity(y, ref, math, dtype):
    """BASELINE gate on the stored output (R14, #R22).

    fp32 storage: max|y - ref| / max|ref| <= TOL[math].
    bf16 storage: the tensor-core gate (5e-3) applies to the stored output as is; the FP32
    CUDA-core path must be within 1e-4 BEFORE the store, so elementwise
    |y - ref| <= delta + half_ulp_bf16(|ref| + delta), delta = 1e-4 * max|ref| (the exact
    bound of one round-to-nearest bf16 store of a value within delta of ref).
    Returns rel_err for reporting."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert y.shape == ref.shape and np.isfinite(y).all()
    err = rel_err(y, ref)
    if dtype == "f32" or math != "fp32":
        assert err <= TOL[math], err
        return err
    delta = TOL[math] * np.abs(ref).max()
    bound = delta + bf16_half_ulp(np.abs(ref) + delta)
    bad = np.abs(y - ref) > bound
    assert not bad.any(), (int(bad.sum()), float(np.abs(y - ref)[bad].max()), err)
    return err


def _math(name):
    from paper_2102_13272_b200 import MATH_BF16, MATH_BF16X3, MATH_FP32_SIMT
    return {"fp32": MATH_FP32_SIMT, "bf16x3": MATH_BF16X3, "bf16": MATH_BF16}[name]


def _run(layer, math, prelu=False):
    from paper_2102_13272_b200 import NestedConv2d
    t = synth.make_inputs(layer)
    x, w = t["x"].cuda(), t["w"].cuda()
    slopes = None
    if layer.prelu or prelu:
        slopes = torch.full((layer.Cout,), synth.PRELU_SLOPE, device="cuda")
    conv = NestedConv2d(w, layer.stride, layer.pad, layer.m_o, layer.m_i, _math(math), outer_taps=layer.r_o,
                        transposed=layer.transposed, output_padding=layer.output_padding,
                        prelu_slopes=slopes)
    y = conv(x)
    torch.cuda.synchronize()
    return t, y.float().cpu().numpy()


def _ref(layer, t):
    x = t["x"].double().numpy()
    w = t["w"].double().numpy()
    if layer.transposed:
        y = direct.conv_transpose2d(x, w, layer.stride, layer.pad, layer.output_padding)
    else:
        y = direct.conv2d(x, w, layer.stride, layer.pad)
    if layer.prelu:
        y = np.where(y >= 0, y, synth.PRELU_SLOPE * y)
    return y


SMALL = {
    "c1": synth.CONFIGS["c1"],
    "c2k5": synth.small(synth.CONFIGS["c2k5"], N=2, H=40, W=31),
    "c2k7": synth.small(synth.CONFIGS["c2k7"], N=2, H=40, W=31),
    "c2k9": synth.small(synth.CONFIGS["c2k9"], N=2, H=40, W=31),
    "c3": synth.small(synth.CONFIGS["c3"], N=1, H=29, W=36, Cin=64, Cout=48),
    "c4a": synth.small(synth.CONFIGS["c4a"], N=2, H=45, W=38),
    "c4b": synth.small(synth.CONFIGS["c4b"], N=1, H=40, W=36, Cin=32, Cout=32),
    "c5_conv1": synth.small(synth.CONFIGS["c5_conv1"], N=1, H=30, W=41),
    "c5_deconv": synth.small(synth.CONFIGS["c5_deconv"], N=1, H=19, W=23),
}


@pytest.mark.parametrize("name", list(SMALL))
def test_fp32_simt_parity(name):
    layer = SMALL[name]
    t, y = _run(layer, "fp32")
    ref = _ref(layer, t)
    check_parity(y, ref, "fp32", layer.dtype)


def test_mixed_outer_kernel_fp32():
    layer = synth.small(synth.CONFIGS["c2k5"], N=1, H=33, W=20, Cin=16, Cout=16)
    from paper_2102_13272_b200 import NestedConv2d
    t = synth.make_inputs(layer)
    conv = NestedConv2d(t["w"].cuda(), 1, 2, 3, 3, _math("fp32"), outer_taps=0)
    assert conv.info["r_outer"] == 2 and conv.info["points"] == 400
    y = conv(t["x"].cuda()).cpu().numpy()
    assert rel_err(y, _ref(layer, t)) <= TOL["fp32"]


def test_deterministic_and_no_nan():
    layer = SMALL["c2k9"]
    _, y1 = _run(layer, "fp32")
    _, y2 = _run(layer, "fp32")
    assert np.array_equal(y1, y2)
    assert np.isfinite(y1).all()


@pytest.mark.parametrize("name", list(SMALL))
def test_bf16x3_tensor_core_parity(name):
    layer = SMALL[name]
    t, y = _run(layer, "bf16x3")
    ref = _ref(layer, t)
    assert y.shape == ref.shape
    err = rel_err(y, ref)
    assert err <= TOL["bf16x3"], err


def test_bf16x3_matches_fp32_closely():
    # both paths compute the same nested algorithm; bf16x3 differs only by the
    # split-operand rounding (R12), far below the 5e-3 gate
    layer = SMALL["c2k9"]
    _, y32 = _run(layer, "fp32")
    _, y3 = _run(layer, "bf16x3")
    assert rel_err(y3, y32) < 2e-3


def test_plain_bf16_runs_finite():
    from paper_2102_13272_b200 import MATH_BF16, NestedConv2d
    layer = SMALL["c2k5"]
    t = synth.make_inputs(layer)
    conv = NestedConv2d(t["w"].cuda(), 1, layer.pad, 3, 3, MATH_BF16)
    y = conv(t["x"].cuda()).cpu().numpy()
    err = rel_err(y, _ref(layer, t))
    assert np.isfinite(y).all() and err < 0.5, err   # speed-ceiling mode, not gated (R12)


@pytest.mark.parametrize("N,H,W", [(1, 9, 9), (1, 1, 1), (3, 10, 100), (2, 128, 17)])
def test_edge_shapes_bf16x3(N, H, W):
    # single tile, degenerate 1x1 input, wide / tall ragged grids
    layer = synth.small(synth.CONFIGS["c2k9"], N=N, H=H, W=W, Cin=16, Cout=32)
    t, y = _run(layer, "bf16x3")
    assert rel_err(y, _ref(layer, t)) <= TOL["bf16x3"]


@pytest.mark.parametrize("m_o,r_o", [(3, 3), (4, 3), (5, 3), (4, 0), (5, 0)])
@pytest.mark.parametrize("name", ["c2k5", "c2k7", "c2k9", "c3", "c4a", "c4b", "c5_conv1", "c5_deconv"])
@pytest.mark.parametrize("math", ["fp32", "bf16x3"])
def test_larger_outer_tile(m_o, r_o, name, math):
    # F(m_o, r_o) (x) F(3,3): (3 m_o) x (3 m_o) outputs per slice; r_o = 0 picks ceil(K'/3) taps
    # (F(m_o, 2) for filters of <= 6 taps per phase); same gates (R8, #R20)
    layer = SMALL[name].with_(m_o=m_o, r_o=r_o)
    t, y = _run(layer, math)
    check_parity(y, _ref(layer, t), math, layer.dtype)


@pytest.mark.parametrize("name", ["t1_srcnn9", "t1_srcnn5a", "t1_srcnn5b"])
@pytest.mark.parametrize("path", ["nested", "ola"])
def test_table1_shapes(name, path):
    # Table I layer shapes at a reduced image size, bf16x3
    from paper_2102_13272_b200 import NestedConv2d
    layer = synth.small(synth.CONFIGS[name], N=2, H=37, W=30)
    t = synth.make_inputs(layer)
    conv = NestedConv2d(t["w"].cuda(), 1, layer.pad, layer.m_o, layer.m_i, _math("bf16x3"), outer_taps=layer.r_o)
    y = conv(t["x"].cuda(), path=path).cpu().numpy()
    assert rel_err(y, _ref(layer, t)) <= TOL["bf16x3"]


@pytest.mark.parametrize("Cout,N,H,W", [(256, 1, 40, 30), (144, 3, 37, 41), (208, 2, 50, 26)])
def test_wide_output_cta_pairs(Cout, N, H, W):
    # Cout_pad > 128: the contraction runs as CTA pairs that multicast the shared B (U) tile;
    # odd 128-slice block counts leave one CTA of the last pair without a block
    layer = synth.small(synth.CONFIGS["c3"], N=N, H=H, W=W, Cin=64, Cout=Cout)
    t, y = _run(layer, "bf16x3")
    check_parity(y, _ref(layer, t), "bf16x3", layer.dtype)


@pytest.mark.parametrize("math", ["fp32", "bf16x3"])
def test_stride2_full_channel_pitch(math):
    # stride 2 with 64 source channels: 4 x 64 = 256 phase-major contraction channels, the
    # compile-time channel pitch of the V stores (C4b's layout) -- every output checked
    layer = synth.small(synth.CONFIGS["c4b"], N=1, H=40, W=37, Cin=64, Cout=32)
    t, y = _run(layer, math)
    assert rel_err(y, _ref(layer, t)) <= TOL[math]


def test_output_buffer_is_validated():
    # the C ABI writes through y's raw pointer: a wrong shape, dtype, device or layout is refused
    from paper_2102_13272_b200 import NestedConv2d
    layer = synth.small(synth.CONFIGS["c2k9"], N=1, H=20, W=20, Cin=16, Cout=16)
    t = synth.make_inputs(layer)
    conv = NestedConv2d(t["w"].cuda(), 1, layer.pad, 4, 3, _math("bf16x3"), outer_taps=3)
    x = t["x"].cuda()
    shp = conv.out_shape(x.shape)
    for bad in (torch.empty((1, 16, 20, 19), device="cuda"),
                torch.empty(shp, dtype=torch.bfloat16, device="cuda"),
                torch.empty(shp),
                torch.empty((shp[0], shp[1], shp[3], shp[2]), device="cuda").transpose(2, 3)):
        with pytest.raises(ValueError):
            conv(x, bad)
    with pytest.raises(ValueError):
        conv(t["x"])   # host x
    y = torch.empty(shp, device="cuda")
    assert conv(x, y) is y


# the persistent TMA-fed input transform (input_transform_tma.cuh) runs for bf16 x whose rows
# are 16-byte multiples; these shapes take it, with more tasks than CTA slots (in-loop TMA
# refills), every 16-byte phase of the window start and ragged tile edges
TMA_SHAPES = {
    "c2k9": synth.small(synth.CONFIGS["c2k9"], N=8, H=61, W=64).with_(dtype="bf16"),
    "c2k5": synth.small(synth.CONFIGS["c2k5"], N=4, H=50, W=72).with_(dtype="bf16"),
    "c2k7": synth.small(synth.CONFIGS["c2k7"], N=3, H=47, W=88).with_(dtype="bf16"),
    "c3": synth.small(synth.CONFIGS["c3"], N=3, H=40, W=48, Cin=64, Cout=64),
    "c5_deconv": synth.small(synth.CONFIGS["c5_deconv"], N=2, H=30, W=40).with_(dtype="bf16"),
    "c2k9_m3": synth.small(synth.CONFIGS["c2k9"], N=4, H=45, W=64).with_(m_o=3, dtype="bf16"),
}


@pytest.mark.parametrize("math", ["bf16x3"])
@pytest.mark.parametrize("name", list(TMA_SHAPES))
def test_tma_input_transform_shapes(name, math):
    layer = TMA_SHAPES[name]
    t, y = _run(layer, math)
    check_parity(y, _ref(layer, t), math, layer.dtype)
