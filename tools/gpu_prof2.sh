# usage: bash tools/gpu_prof2.sh <tag> -- full bench (cpu baseline), launch list, ncu --set full of the
# three kernels on c2k9 and c3, and dram bytes (lightweight ncu metrics) of every C2 / C3 layer
TAG=${1:-r1p}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks_$TAG.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
kill $SMI
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-compare > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-compare > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launches rc=$?"
for LAYER in c2k5 c2k7 c2k9 c3 c5_conv1; do
  timeout 300 python tools/prof_layer.py $LAYER --iters 2 > gpurun_out/prof_plain_${TAG}_$LAYER.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/dram_${TAG}_$LAYER.csv python tools/prof_layer.py $LAYER --iters 2 > /dev/null 2>&1; echo "dram $LAYER rc=$?"
done
for LAYER in c2k9 c3; do
for K in input_transform contraction output_transform; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_${LAYER}_$K python tools/prof_layer.py $LAYER > gpurun_out/ncu_${K}_${TAG}_$LAYER.log 2>&1; echo "ncu $LAYER $K rc=$?"
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_c1 -s 1 -c 1 \
  -o gpurun_out/prof_${TAG}_c5conv1_fused_c1 python tools/prof_layer.py c5_conv1 > gpurun_out/ncu_fused_${TAG}.log 2>&1; echo "ncu c5_conv1 fused_c1 rc=$?"
du -sh gpurun_out
