"""Seeded synthetic inputs for the BASELINE configs (shared by tests, bench and smoke).

Holds no arithmetic of the method: only shapes, seeds and value distributions
(BASELINE.json `configs`).  Every tensor is drawn on
the CPU with torch.Generator(seed) in float64 and cast once (round to nearest
even) to its storage dtype, x first then w, so the oracle and the GPU path see
identical bits.  No public dataset is used: the paper's SR images / trained
SRCNN, FSRCNN and PNASNet weights are not available; these distributions stand
in for them.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Dict, List, Optional

import torch


@dataclass(frozen=True)
class Layer:
    name: str
    N: int
    Cin: int
    Cout: int
    H: int
    W: int
    K: int
    stride: int = 1
    pad: int = 0
    transposed: bool = False
    output_padding: int = 0
    m_o: int = 3
    m_i: int = 3
    r_o: int = 3                # outer kernel taps: 3 = the paper's fixed 3x3 tile grid, 0 = ceil(K'/3) (R8)
    dtype: str = "f32"          # storage dtype of x, w, y
    xdist: str = "normal"       # normal | relu_normal | unif01 | unif11
    wdist: str = "he"           # he | unif11
    seed: int = 0
    prelu: bool = False
    depthwise: bool = False     # groups = Cin = Cout: w [C][1][K][K] (Table I's PNASNet row)

    @property
    def Ho(self) -> int:
        if self.transposed:
            return (self.H - 1) * self.stride - 2 * self.pad + self.K + self.output_padding
        return (self.H + 2 * self.pad - self.K) // self.stride + 1

    @property
    def Wo(self) -> int:
        if self.transposed:
            return (self.W - 1) * self.stride - 2 * self.pad + self.K + self.output_padding
        return (self.W + 2 * self.pad - self.K) // self.stride + 1

    def direct_flops(self) -> int:
        """2 * MACs of the native convolution (Eq. 2.1; GOPs convention of P:164)."""
        if self.depthwise:
            return 2 * self.N * self.Ho * self.Wo * self.Cout * self.K * self.K
        if self.transposed:
            return 2 * self.N * self.H * self.W * self.Cin * self.Cout * self.K * self.K
        return 2 * self.N * self.Ho * self.Wo * self.Cin * self.Cout * self.K * self.K

    def with_(self, **kw) -> "Layer":
        return replace(self, **kw)


CONFIGS: Dict[str, Layer] = {
    # configs[0]: parity config, F(2,3)(x)F(2,3) with coverage phases
    "c1": Layer("c1", 1, 16, 16, 32, 32, 5, 1, 2, m_o=2, m_i=2, xdist="unif11", wdist="unif11", seed=1),
    # configs[1]: filter-size sweep (the bench workload)
    # (nesting F(4,3) (x) F(3,3) for configs[1..4]: 12x12-output slices; the fastest outer
    #  kernel that meets the 5e-3 gate with margin -- DESIGN.md#R20)
    "c2k5": Layer("c2k5", 32, 64, 64, 128, 128, 5, 1, 2, m_o=4, r_o=0, seed=21),
    "c2k7": Layer("c2k7", 32, 64, 64, 128, 128, 7, 1, 3, m_o=4, seed=22),
    "c2k9": Layer("c2k9", 32, 64, 64, 128, 128, 9, 1, 4, m_o=4, seed=23),
    # configs[2]: large-filter bf16 layer
    "c3": Layer("c3", 64, 256, 256, 64, 64, 9, 1, 4, m_o=4, dtype="bf16", xdist="relu_normal", seed=3),
    # configs[3]: strided large filters (stride-Winograd phases)
    "c4a": Layer("c4a", 256, 3, 64, 224, 224, 7, 2, 3, m_o=4, r_o=0, xdist="unif01", seed=41),
    "c4b": Layer("c4b", 256, 64, 64, 112, 112, 9, 2, 4, m_o=4, r_o=0, xdist="unif01", seed=42),
    # configs[4]: FSRCNN-s shaped network, nested layers first and last
    "c5_conv1": Layer("c5_conv1", 16, 1, 32, 540, 960, 5, 1, 2, m_o=4, r_o=0, xdist="unif01", seed=5,
                      prelu=True),
    "c5_conv2": Layer("c5_conv2", 16, 32, 5, 540, 960, 1, 1, 0, seed=51, prelu=True),
    "c5_conv3": Layer("c5_conv3", 16, 5, 5, 540, 960, 3, 1, 1, seed=52, prelu=True),
    "c5_conv4": Layer("c5_conv4", 16, 5, 32, 540, 960, 1, 1, 0, seed=53, prelu=True),
    "c5_deconv": Layer("c5_deconv", 16, 32, 1, 540, 960, 9, 2, 4, transposed=True, output_padding=1,
                       m_o=4, r_o=0, seed=54),
}

# Table I of the paper (ZCU102): the conv2d layer shapes (Cout, Cin, H, W), measured
# there as nested vs OLA-Winograd GOPs.  Weights / images of SRCNN are not available: the
# synthetic stand-ins use BASELINE configs[1]'s distributions; batch 8 (the paper runs one image).
# The depthwise PNASNet 7x7 row ((54, 54, 83, 83)) runs the depthwise path (groups = 54,
# same padding; the paper gives no padding: 3 keeps 83 x 83), He-normal over the 49 taps.
CONFIGS.update({
    "t1_srcnn9": Layer("t1_srcnn9", 8, 1, 64, 256, 256, 9, 1, 4, m_o=4, seed=61),
    "t1_pnas_dw7": Layer("t1_pnas_dw7", 8, 54, 54, 83, 83, 7, 1, 3, m_o=4, seed=64, depthwise=True),
    "t1_srcnn5a": Layer("t1_srcnn5a", 8, 64, 32, 256, 256, 5, 1, 2, m_o=4, r_o=0, seed=62),
    "t1_srcnn5b": Layer("t1_srcnn5b", 8, 32, 1, 256, 256, 5, 1, 2, m_o=4, r_o=0, seed=63),
})
TABLE1 = ["t1_srcnn9", "t1_pnas_dw7", "t1_srcnn5a", "t1_srcnn5b"]
TABLE1_PAPER_SPEEDUP = {"t1_srcnn9": 3.29, "t1_pnas_dw7": 1.41, "t1_srcnn5a": 1.43,
                        "t1_srcnn5b": 1.43}

C2_SWEEP = ["c2k5", "c2k7", "c2k9"]
C5_NET = ["c5_conv1", "c5_conv2", "c5_conv3", "c5_conv4", "c5_deconv"]
PRELU_SLOPE = 0.25


def _draw(gen: torch.Generator, shape, dist: str, fan_in: int) -> torch.Tensor:
    if dist == "normal":
        return torch.randn(shape, generator=gen, dtype=torch.float64)
    if dist == "relu_normal":
        return torch.relu(torch.randn(shape, generator=gen, dtype=torch.float64))
    if dist == "unif01":
        return torch.rand(shape, generator=gen, dtype=torch.float64)
    if dist == "unif11":
        return torch.rand(shape, generator=gen, dtype=torch.float64) * 2 - 1
    if dist == "he":
        return torch.randn(shape, generator=gen, dtype=torch.float64) * math.sqrt(2.0 / fan_in)
    raise ValueError(dist)


def storage_dtype(layer: Layer) -> torch.dtype:
    return torch.bfloat16 if layer.dtype == "bf16" else torch.float32


def make_inputs(layer: Layer, x: bool = True) -> Dict[str, torch.Tensor]:
    """{'x': [N, Cin, H, W], 'w': [Cout, Cin, K, K] (transposed: [Cin, Cout, K, K])}
    on the CPU in the storage dtype."""
    gen = torch.Generator().manual_seed(layer.seed)
    out = {}
    dt = storage_dtype(layer)
    if x:
        out["x"] = _draw(gen, (layer.N, layer.Cin, layer.H, layer.W), layer.xdist, 1).to(dt)
    else:
        # keep the draw order (x first, then w) even when x is not materialised
        gen = torch.Generator().manual_seed(layer.seed)
        _draw(gen, (layer.N, layer.Cin, layer.H, layer.W), layer.xdist, 1)
    if layer.depthwise:   # one K x K filter per channel: fan-in K^2
        out["w"] = _draw(gen, (layer.Cout, 1, layer.K, layer.K), layer.wdist, layer.K * layer.K).to(dt)
        return out
    wshape = ((layer.Cin, layer.Cout, layer.K, layer.K) if layer.transposed
              else (layer.Cout, layer.Cin, layer.K, layer.K))
    out["w"] = _draw(gen, wshape, layer.wdist, layer.Cin * layer.K * layer.K).to(dt)
    return out


def small(layer: Layer, N: int = 1, H: Optional[int] = None, W: Optional[int] = None,
          Cin: Optional[int] = None, Cout: Optional[int] = None) -> Layer:
    """Same distributions and filter geometry at a size the oracle finishes in seconds."""
    return layer.with_(name=layer.name + "_small", N=N, H=H or layer.H, W=W or layer.W,
                       Cin=Cin or layer.Cin, Cout=Cout or layer.Cout)
