#!/bin/bash
# round-2 final evidence: default bench line with clocks, every workload with compare legs,
# launch list of the default bench
TAG=${1:-r2z2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks_$TAG.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
for wl in c3 c4 c5 table1; do timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${TAG}_$wl.json 2>> gpurun_out/bench_$TAG.err; echo "bench $wl rc=$?"; done
kill $SMI
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-compare > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-compare > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launches rc=$?"
for L in c2k9 c3; do
  for K in contraction input_transform output_transform; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_${L}_$K python tools/prof_layer.py $L > gpurun_out/ncu_${K}_${TAG}_$L.log 2>&1; echo "ncu $L $K rc=$?"
  done
done
for r in gpurun_out/prof_${TAG}_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  ncu -i $r --page raw --csv > gpurun_out/$b.raw.csv 2>/dev/null
  case "$b" in *contraction) ;; *) rm -f $r;; esac
done
du -sh gpurun_out
