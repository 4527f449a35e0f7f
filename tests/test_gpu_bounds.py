"""Out-of-bounds write checks (compute-sanitizer is not available on the GPU pool): every path writes
only inside y and inside the workspace size the library reports.  y and the workspace are carved out of
larger buffers whose guard regions hold a byte pattern that must survive the call."""
import pytest
import torch

import synth
from test_gpu_nested import _math

pytestmark = pytest.mark.gpu

GUARD = 1 << 16  # bytes on each side


def _guarded(nbytes, device="cuda"):
    buf = torch.full((nbytes + 2 * GUARD,), 0xA5, dtype=torch.uint8, device=device)
    return buf, buf[GUARD:GUARD + nbytes]


def _intact(buf, nbytes):
    return bool((buf[:GUARD] == 0xA5).all().item() and (buf[GUARD + nbytes:] == 0xA5).all().item())


CASES = [
    ("c2k9", dict(N=2, H=29, W=31, Cin=32, Cout=32)),
    ("c3", dict(N=1, H=20, W=19, Cin=64, Cout=64)),
    ("c4a", dict(N=2, H=21, W=17)),
    ("c4b", dict(N=1, H=22, W=23, Cin=8, Cout=16)),
    ("c5_conv1", dict(N=1, H=19, W=25)),
    ("c5_deconv", dict(N=1, H=11, W=13)),
    ("c1", None),
]


@pytest.mark.parametrize("path", ["nested", "ola", "direct"])
@pytest.mark.parametrize("math", ["bf16x3", "fp32"])
@pytest.mark.parametrize("name,kw", CASES)
def test_writes_stay_in_bounds(name, kw, math, path):
    from paper_2102_13272_b200 import NestedConv2d
    layer = synth.small(synth.CONFIGS[name], **kw) if kw else synth.CONFIGS[name]
    t = synth.make_inputs(layer)
    slopes = torch.full((layer.Cout,), synth.PRELU_SLOPE, device="cuda") if layer.prelu else None
    conv = NestedConv2d(t["w"].cuda(), layer.stride, layer.pad, layer.m_o, layer.m_i, _math(math), outer_taps=layer.r_o,
                        transposed=layer.transposed, output_padding=layer.output_padding, prelu_slopes=slopes)
    x = t["x"].cuda()
    N, _, H, W = x.shape
    shape = conv.out_shape(x.shape)
    es = x.element_size()
    ny = es * shape[0] * shape[1] * shape[2] * shape[3]
    ybuf, yv = _guarded(ny)
    y = yv.view(x.dtype).view(shape)
    nws = conv.plan.workspace_size(N, H, W, path)
    wbuf, ws = _guarded(nws)
    if path == "nested":
        conv.plan.forward(x, conv.U, y, N, H, W, ws, nws)
    elif path == "ola":
        conv.plan.ola(x, conv.w, y, N, H, W, ws, nws)
    else:
        conv.plan.direct(x, conv.w, y, N, H, W, ws, nws)
    torch.cuda.synchronize()
    assert _intact(ybuf, ny), "write outside y"
    assert _intact(wbuf, nws), "write outside the workspace"
    assert torch.isfinite(y).all().item()
