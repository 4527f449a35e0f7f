"""C3 at full size with fp32 storage (the bf16 inputs are exact in fp32): the FP32 CUDA-core
path's error before any bf16 store, per BASELINE metric, plus where the worst element sits."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from oracle import direct
from paper_2102_13272_b200 import NestedConv2d, MATH_FP32_SIMT, MATH_BF16X3
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
N = int(sys.argv[2]) if len(sys.argv) > 2 else None
l = synth.CONFIGS[name]
if N: l = l.with_(N=N)
t = synth.make_inputs(l)
x32, w32 = t["x"].float(), t["w"].float()
ref = direct.conv2d(x32.double().numpy(), w32.double().numpy(), 1, l.pad)
M = np.abs(ref).max()
for mo in (4, 3):
  for math, nm in ((MATH_FP32_SIMT, "fp32"), (MATH_BF16X3, "bf16x3")):
    conv = NestedConv2d(w32.cuda(), 1, l.pad, mo, 3, math, outer_taps=3)
    y = conv(x32.cuda()).cpu().double().numpy()
    d = np.abs(y - ref)
    i = np.unravel_index(d.argmax(), d.shape)
    print(f"{name} N={l.N} F({mo},3)(x)F(3,3) {nm}: rel_err {d.max()/M:.3e}  mean {d.mean()/M:.2e}  worst at {i} ref {ref[i]:.4f} max|ref| {M:.3f}", flush=True)
