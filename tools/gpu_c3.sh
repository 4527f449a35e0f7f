#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nested.py tests/test_gpu_network.py -m gpu -q -x > gpurun_out/c3_pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/c3_pt.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "c3" > gpurun_out/c3_pt2.log 2>&1; echo "pytest fullsize rc=$?"; tail -3 gpurun_out/c3_pt2.log
for f in 0 1; do
  echo "== NW_FUSE_WIDE=$f"
  NW_FUSE_WIDE=$f KERNELS=1 timeout 600 python tools/time_layers.py c3 2>&1 | tail -3
done
