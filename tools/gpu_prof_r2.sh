#!/bin/bash
# round 2 evidence: default bench line with clocks, launch list, ncu --set full of the round's new / changed kernels
TAG=${1:-r2a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks_$TAG.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
for wl in c3 c4 c5 table1; do timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_${TAG}_$wl.json 2>> gpurun_out/bench_$TAG.err; done
kill $SMI
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-compare > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-compare > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launches rc=$?"
for L in c3 c2k9 t1_pnas_dw7; do
  timeout 300 python tools/prof_layer.py $L > gpurun_out/prof_plain_${TAG}_$L.log 2>&1 || continue
  for K in input_transform contraction output_transform depthwise; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_${L}_$K python tools/prof_layer.py $L > gpurun_out/ncu_${K}_${TAG}_$L.log 2>&1; echo "ncu $L $K rc=$?"
  done
done
# keep gpurun_out under the 64 MiB copy-back limit: export every report's raw metrics and
# per-instruction source view as CSV, keep the .ncu-rep only for the kernels named in KEEP
KEEP=${KEEP:-"prof_${TAG}_c3_input_transform prof_${TAG}_c2k9_contraction"}
for r in gpurun_out/prof_${TAG}_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  ncu -i $r --page raw --csv > gpurun_out/$b.raw.csv 2>/dev/null
  ncu -i $r --page source --csv > gpurun_out/$b.source.csv 2>/dev/null
  case " $KEEP " in *" $b "*) ;; *) rm -f $r;; esac
done
du -sh gpurun_out; ls gpurun_out | grep $TAG
