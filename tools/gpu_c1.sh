# usage: bash tools/gpu_c1.sh <tag>  -- fused single-channel kernel: parity, then per-layer times on / off
TAG=${1:-c1}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused_c1.py -x -q > gpurun_out/pt_fc1_$TAG.log 2>&1; echo "fused tests rc=$?"; tail -5 gpurun_out/pt_fc1_$TAG.log
for F in 1 0; do
  echo "NW_FUSED_C1=$F"; NW_FUSED_C1=$F KERNELS=1 timeout 300 python tools/time_layers.py c5_conv1 t1_srcnn9 c2k9 c3 2>&1 | tail -12
done
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pt_all_$TAG.log 2>&1; echo "all gpu tests rc=$?"; tail -5 gpurun_out/pt_all_$TAG.log
