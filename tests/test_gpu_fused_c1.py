"""GPU parity of the single-input-channel fused kernel (fused_small.cuh) against the
FP64 oracle.  Every nested stride-1 layer with Cin = 1 runs through it (e.g. FSRCNN-s conv1,
Table I SRCNN 9x9 conv1); the cases below add ragged slice counts, more 32-slice chunks than
SMs (persistent loop), output-channel counts that are not a multiple of the per-pass group,
bf16 storage, PReLU and the plain-bf16 math mode.  Tolerances as tests/test_gpu_nested.py.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import direct
from oracle.errstudy import rel_err
from test_gpu_nested import check_parity

pytestmark = pytest.mark.gpu

# plain bf16 is the speed-ceiling mode: finite and bounded, not gated (R12)
TOL = {"fp32": 1e-4, "bf16x3": 5e-3, "bf16": 0.5}


def _math(name):
    import paper_2102_13272_b200 as nw
    return {"fp32": nw.MATH_FP32_SIMT, "bf16x3": nw.MATH_BF16X3, "bf16": nw.MATH_BF16}[name]


def _check(layer, math, prelu=False):
    from paper_2102_13272_b200 import NestedConv2d
    t = synth.make_inputs(layer)
    x, w = t["x"].cuda(), t["w"].cuda()
    slope = 0.25
    slopes = torch.full((layer.Cout,), slope, device="cuda") if prelu else None
    conv = NestedConv2d(w, layer.stride, layer.pad, layer.m_o, layer.m_i, _math(math), outer_taps=layer.r_o,
                        prelu_slopes=slopes)
    y = conv(x)
    torch.cuda.synchronize()
    y = y.float().cpu().numpy()
    ref = direct.conv2d(t["x"].double().numpy(), t["w"].double().numpy(), layer.stride, layer.pad)
    if prelu:
        ref = np.where(ref >= 0, ref, slope * ref)
    if math == "bf16":
        assert np.isfinite(y).all() and rel_err(y, ref) <= TOL[math]
    else:
        check_parity(y, ref, math, layer.dtype)


BASE = synth.CONFIGS["c5_conv1"]


@pytest.mark.parametrize("K,m_o,r_o", [(5, 4, 0), (5, 4, 3), (7, 3, 3), (9, 4, 3), (9, 5, 3), (3, 2, 3)])
@pytest.mark.parametrize("math", ["fp32", "bf16x3"])
def test_kernels_and_outer_tiles(K, m_o, r_o, math):
    layer = synth.small(BASE, N=2, H=37, W=29, Cout=32).with_(K=K, pad=K // 2, m_o=m_o, r_o=r_o)
    _check(layer, math)


@pytest.mark.parametrize("N,H,W,Cout", [(1, 1, 1, 32), (1, 12, 12, 1), (3, 50, 7, 13), (5, 131, 97, 6),
                                        (8, 300, 300, 4)])
def test_ragged_and_persistent(N, H, W, Cout):
    # one slice / one channel / ragged grids / > 148 chunks of 32 slices per CTA loop
    layer = synth.small(BASE, N=N, H=H, W=W, Cout=Cout)
    _check(layer, "bf16x3")


def test_prelu_bf16_storage_and_plain_bf16():
    layer = synth.small(BASE, N=2, H=45, W=33, Cout=32)
    _check(layer, "bf16x3", prelu=True)
    _check(layer.with_(dtype="bf16"), "bf16x3", prelu=True)
    _check(layer, "bf16")


def test_three_kernel_path_still_matches(tmp_path):
    # NW_FUSED_C1=0 (read once per process) routes the same layer through input transform,
    # contraction and output transform; both must agree with each other and the oracle
    import os
    import subprocess
    import sys
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import synth\n"
        "from paper_2102_13272_b200 import NestedConv2d, MATH_BF16X3\n"
        "l = synth.small(synth.CONFIGS['c5_conv1'], N=2, H=45, W=33)\n"
        "t = synth.make_inputs(l)\n"
        "y = NestedConv2d(t['w'].cuda(), 1, l.pad, l.m_o, l.m_i, MATH_BF16X3, outer_taps=l.r_o)(t['x'].cuda())\n"
        "np.save(%r, y.float().cpu().numpy())\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for flag in ("0", "1"):
        out = str(tmp_path / f"y{flag}.npy")
        env = dict(os.environ, NW_FUSED_C1=flag)
        r = subprocess.run([sys.executable, "-c", code % (root, os.path.join(root, "tests"), out)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[flag] = np.load(out)
    l = synth.small(BASE, N=2, H=45, W=33)
    t = synth.make_inputs(l)
    ref = direct.conv2d(t["x"].double().numpy(), t["w"].double().numpy(), 1, l.pad)
    for flag, y in outs.items():
        assert rel_err(y, ref) <= TOL["bf16x3"], flag
    assert rel_err(outs["0"], outs["1"]) <= TOL["bf16x3"]
