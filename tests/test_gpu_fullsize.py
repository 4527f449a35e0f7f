"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Every configuration runs once through the C ABI at its full shape (same NestedConv2d
setup and batch as bench.py); the FP64 oracle is evaluated only at sampled outputs
(oracle.direct.conv2d_at / conv_transpose2d_at): every corner and edge of the first and
last image and channel plus random interior points.  Metric (R14) with the
denominator taken over the sampled reference values (stricter than the full max).
Also checks the host-buffer entry point (nw_conv_forward_host, pipelined copies)
against the device entry point bit for bit.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import direct
from test_gpu_nested import TOL, _math

pytestmark = pytest.mark.gpu

FULL = ["c1", "c2k5", "c2k7", "c2k9", "c3", "c4a", "c4b", "c5_conv1", "c5_deconv"]


def _points(layer, n_random=1500, seed=0):
    rng = np.random.default_rng(seed)
    Ho, Wo = layer.Ho, layer.Wo
    pts = set()
    for n in (0, layer.N - 1):
        for o in (0, layer.Cout - 1):
            for i in (0, 1, Ho // 2, Ho - 2, Ho - 1):
                for j in (0, 1, Wo // 2, Wo - 2, Wo - 1):
                    pts.add((n, o, max(i, 0), max(j, 0)))
    for _ in range(n_random):
        pts.add((int(rng.integers(layer.N)), int(rng.integers(layer.Cout)), int(rng.integers(Ho)),
                 int(rng.integers(Wo))))
    return sorted(pts)


@pytest.mark.parametrize("name", FULL)
def test_full_size_sampled(name):
    from paper_2102_13272_b200 import NestedConv2d
    layer = synth.CONFIGS[name]
    t = synth.make_inputs(layer)
    slopes = torch.full((layer.Cout,), synth.PRELU_SLOPE, device="cuda") if layer.prelu else None
    conv = NestedConv2d(t["w"].cuda(), layer.stride, layer.pad, layer.m_o, layer.m_i, _math("bf16x3"), outer_taps=layer.r_o,
                        transposed=layer.transposed, output_padding=layer.output_padding, prelu_slopes=slopes)
    y = conv(t["x"].cuda())
    torch.cuda.synchronize()
    assert tuple(y.shape) == (layer.N, layer.Cout, layer.Ho, layer.Wo)
    pts = _points(layer)
    idx = tuple(torch.tensor(c, device="cuda") for c in zip(*pts))
    got = y[idx].float().cpu().numpy().astype(np.float64)
    x64, w64 = t["x"].double().numpy(), t["w"].double().numpy()
    if layer.transposed:
        ref = direct.conv_transpose2d_at(x64, w64, layer.stride, layer.pad, pts)
    else:
        ref = direct.conv2d_at(x64, w64, layer.stride, layer.pad, pts)
    if layer.prelu:
        ref = np.where(ref >= 0, ref, synth.PRELU_SLOPE * ref)
    tol = TOL["bf16x3"]
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert np.isfinite(got).all() and err <= tol, err
    assert torch.isfinite(y).all().item()


@pytest.mark.parametrize("N", [1, 5])
def test_host_entry_point_matches_device(N):
    from paper_2102_13272_b200 import NestedConv2d
    layer = synth.small(synth.CONFIGS["c2k9"], N=N, H=40, W=33, Cin=32, Cout=32)
    t = synth.make_inputs(layer)
    conv = NestedConv2d(t["w"].cuda(), 1, layer.pad, 3, 3, _math("bf16x3"))
    y_dev = conv(t["x"].cuda()).cpu()
    hx = t["x"].pin_memory()
    hy = torch.empty(y_dev.shape, dtype=y_dev.dtype).pin_memory()
    nbytes = conv.plan.workspace_size(N, layer.H, layer.W, "host")
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    conv.plan.forward_host(hx, conv.U, hy, N, layer.H, layer.W, ws, nbytes)
    torch.cuda.synchronize()
    assert torch.equal(hy, y_dev)


# ---------------------------------------------------------------------------
# Full-tensor parity at the full BASELINE sizes (every output, both math modes).
# The FP64 oracle (oracle.direct, einsum per tap) runs on all host cores: C2
# ~5 s per layer, C3 ~40 s on a 16-core host.  One reference per layer serves
# both math modes.
# ---------------------------------------------------------------------------
FULL_TENSOR = ["c2k5", "c2k7", "c2k9", "c3", "c4a", "c4b", "c5_conv1", "c5_deconv"]


@pytest.mark.parametrize("name", FULL_TENSOR)
def test_full_size_full_tensor(name):
    from paper_2102_13272_b200 import NestedConv2d
    from test_gpu_nested import _ref, check_parity
    layer = synth.CONFIGS[name]
    t = synth.make_inputs(layer)
    ref = _ref(layer, t)
    x, w = t["x"].cuda(), t["w"].cuda()
    slopes = torch.full((layer.Cout,), synth.PRELU_SLOPE, device="cuda") if layer.prelu else None
    errs = {}
    for math in ("bf16x3", "fp32"):
        conv = NestedConv2d(w, layer.stride, layer.pad, layer.m_o, layer.m_i, _math(math), outer_taps=layer.r_o,
                            transposed=layer.transposed, output_padding=layer.output_padding, prelu_slopes=slopes)
        y = conv(x)
        torch.cuda.synchronize()
        errs[math] = check_parity(y.float().cpu().numpy(), ref, math, layer.dtype)
        del conv, y
        torch.cuda.empty_cache()
    print(name, {k: f"{v:.3e}" for k, v in errs.items()})
