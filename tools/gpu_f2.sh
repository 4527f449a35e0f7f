#!/bin/bash
# fused level 2 (M'') check: parity subset, then per-layer and per-kernel times for NW_FUSE_AI=1 vs 2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nested.py tests/test_gpu_geometries.py -m gpu -q -x > gpurun_out/f2_pt.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/f2_pt.log
for f in 1 2; do
  echo "== NW_FUSE_AI=$f"
  NW_FUSE_AI=$f KERNELS=1 timeout 600 python tools/time_layers.py c2k5 c2k7 c2k9 c4a c4b 2>&1 | tail -12
done
