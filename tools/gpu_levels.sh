#!/bin/bash
# Per-layer and per-kernel times of the contraction's fusion levels:
#   NW_FUSE_AI=1 (inner output level along w) vs 2 (both axes, default) on the 64-channel layers,
#   NW_FUSE_WIDE=0 (plain contraction) vs 1 (128-channel level 1, default) on C3.
# bash tools/gpu_levels.sh   (after a parity run of the nested tests)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nested.py tests/test_gpu_geometries.py -m gpu -q -x > gpurun_out/levels_pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/levels_pt.log
for f in 1 2; do
  echo "== NW_FUSE_AI=$f"
  NW_FUSE_AI=$f KERNELS=1 timeout 600 python tools/time_layers.py c2k5 c2k7 c2k9 c4a c4b 2>&1 | tail -12
done
for f in 0 1; do
  echo "== NW_FUSE_WIDE=$f"
  NW_FUSE_WIDE=$f KERNELS=1 timeout 600 python tools/time_layers.py c3 2>&1 | tail -3
done
