"""B200-native nested Winograd convolution (arXiv 2102.13272).

The compute lives in ``libnw.so`` (C ABI, include/nw.h, CUDA for sm_100a);
this package is the thin Python binding (``_lib``), torch-facing wrappers
(``conv``) and the multi-GPU launch helpers (``dist``).
"""
from ._lib import (DTYPE_BF16, DTYPE_F32, MATH_BF16, MATH_BF16X3, MATH_FP32_SIMT, NWError, Plan,  # noqa: F401
                   launch_count, load)
from .conv import NestedConv2d, nested_conv2d  # noqa: F401
