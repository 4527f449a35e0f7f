TAG=${1:-wl2}
mkdir -p gpurun_out
for WL in c3 c4 c5 table1 c5net c1; do
  timeout 900 python bench.py --workload $WL --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}_$WL.json 2> gpurun_out/bench_${TAG}_$WL.err; echo "bench $WL rc=$?"
done
