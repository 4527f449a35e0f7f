# usage: bash tools/gpu_t.sh layer...  -- per-layer / per-kernel times only (no tests)
KERNELS=1 timeout 300 python tools/time_layers.py "$@" 2>&1 | tail -20
