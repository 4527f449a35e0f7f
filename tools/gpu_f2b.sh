#!/bin/bash
for e in "NW_FUSE_AI=2" "NW_FUSE_AI=2 NW_CLUSTER=1"; do
  echo "== $e"
  env $e KERNELS=1 timeout 600 python tools/time_layers.py c2k5 c2k9 c4a c4b 2>&1 | tail -9
done
bash tools/gpu_ncu.sh f2c "c2k9 contraction" "c4a contraction"
