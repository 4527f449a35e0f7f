"""The CUDA path must be the one that runs: fail loudly, never fall back."""
import os

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_native_library_loaded_and_launching():
    import paper_2102_13272_b200 as nw
    lib = nw.load()
    assert os.path.exists(nw._lib.LIB_PATH)
    maps = open("/proc/self/maps").read()
    assert "libnw.so" in maps
    before = nw.launch_count()
    w = torch.randn(8, 8, 5, 5, device="cuda")
    x = torch.randn(1, 8, 20, 20, device="cuda")
    nw.nested_conv2d(x, w, 1, 2, math=nw.MATH_FP32_SIMT)
    torch.cuda.synchronize()
    assert nw.launch_count() >= before + 4
