"""Thin torch-facing wrappers over the C ABI (device memory via torch, compute in libnw.so).

``NestedConv2d`` owns a plan, the transformed filter U and a workspace, and
calls ``nw_conv_forward`` / ``nw_conv_ola`` / ``nw_conv_direct``.  torch is used
only to allocate device buffers and to name the current stream.
"""
from __future__ import annotations

from typing import Optional

import torch

from . import _lib
from ._lib import DTYPE_BF16, DTYPE_F32, MATH_BF16, MATH_BF16X3, MATH_FP32_SIMT, Plan  # noqa: F401

_DT = {torch.float32: DTYPE_F32, torch.bfloat16: DTYPE_BF16}


class NestedConv2d:
    """One convolution layer: y = conv(x, w) by nested Winograd (or a comparison path)."""

    def __init__(self, w: torch.Tensor, stride: int = 1, pad: Optional[int] = None, m_outer: int = 3,
                 m_inner: int = 3, math: int = MATH_BF16X3, transposed: bool = False,
                 output_padding: int = 0, outer_taps: int = 3, prelu_slopes: Optional[torch.Tensor] = None,
                 transform: bool = True, depthwise: bool = False):
        """transform=False allocates U without computing it: a multi-GPU run transforms the
        filter on rank 0 only and broadcasts U (dist.broadcast_filter) into the other ranks'.
        depthwise=True: w is [C][1][K][K] (groups = C, Table I's PNASNet row), Cin = Cout = C."""
        if not w.is_cuda:
            raise ValueError("w must be a CUDA tensor")
        if w.dtype not in _DT:
            raise ValueError(f"unsupported dtype {w.dtype}")
        K = w.shape[-1]
        Cin, Cout = (w.shape[0], w.shape[1]) if transposed else (w.shape[1], w.shape[0])
        if depthwise:
            if w.shape[1] != 1:
                raise ValueError("depthwise filters are [C][1][K][K]")
            Cin = Cout = w.shape[0]
        self.w = w.contiguous()
        self.dtype = w.dtype
        self.prelu_slopes = prelu_slopes
        self.plan = Plan(K, stride, m_outer, m_inner, Cin, Cout, math=math, dtype=_DT[w.dtype],
                         transposed=transposed, output_padding=output_padding, outer_taps=outer_taps,
                         pad=pad, prelu_slopes=prelu_slopes, depthwise=depthwise)
        self.info = self.plan.info()
        self.Cin, self.Cout = Cin, Cout
        self.U = torch.empty(self.info["filter_bytes"], dtype=torch.uint8, device=w.device)
        self._ws = {}
        if transform:
            self.transform_filter()

    def transform_filter(self, stream=None) -> None:
        self.plan.transform_filter(self.w, self.U, stream)

    def workspace(self, N: int, H: int, W: int, path: str = "nested") -> torch.Tensor:
        key = (N, H, W, path)
        if key not in self._ws:
            nbytes = self.plan.workspace_size(N, H, W, path)
            self._ws[key] = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.w.device)
        return self._ws[key]

    def out_shape(self, x_shape):
        N, _, H, W = x_shape
        Ho, Wo = self.plan.output_size(H, W)
        return (N, self.Cout, Ho, Wo)

    def __call__(self, x: torch.Tensor, y: Optional[torch.Tensor] = None, path: str = "nested",
                 stream=None) -> torch.Tensor:
        if x.dtype != self.dtype or not x.is_cuda:
            raise ValueError("x must be a CUDA tensor with the filter's dtype")
        if x.device != self.w.device:
            raise ValueError(f"x is on {x.device}, the plan's filter on {self.w.device}")
        if x.dim() != 4:
            raise ValueError("x must be NCHW")
        x = x.contiguous()
        N, C, H, W = x.shape
        if C != self.Cin:
            raise ValueError("channel mismatch")
        if y is None:
            y = torch.empty(self.out_shape(x.shape), dtype=self.dtype, device=x.device)
        else:  # the C ABI writes through a raw pointer: shape, dtype, device and layout must match
            if tuple(y.shape) != self.out_shape(x.shape):
                raise ValueError(f"y has shape {tuple(y.shape)}, expected {self.out_shape(x.shape)}")
            if y.dtype != self.dtype or y.device != x.device:
                raise ValueError("y must have the filter's dtype and x's device")
            if not y.is_contiguous():
                raise ValueError("y must be contiguous (NCHW)")
        ws = self.workspace(N, H, W, path)
        if path == "nested":
            self.plan.forward(x, self.U, y, N, H, W, ws, ws.numel(), stream)
        elif path == "ola":
            self.plan.ola(x, self.w, y, N, H, W, ws, ws.numel(), stream)
        elif path == "direct":
            self.plan.direct(x, self.w, y, N, H, W, ws, ws.numel(), stream)
        else:
            raise ValueError(path)
        return y


def nested_conv2d(x: torch.Tensor, w: torch.Tensor, stride: int = 1, pad: Optional[int] = None,
                  m_outer: int = 3, m_inner: int = 3, math: int = MATH_BF16X3, **kw) -> torch.Tensor:
    """Functional form: plan + filter transform + forward in one call."""
    return NestedConv2d(w, stride, pad, m_outer, m_inner, math, **kw)(x)
