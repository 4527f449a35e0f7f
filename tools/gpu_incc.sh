TAG=${1:-incc}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_$TAG.log
for CC in 32 64; do for WL in c2 c3; do
  NW_IN_CC=$CC timeout 600 python bench.py --workload $WL --steps 10 --warmup 3 --no-cpu --no-e2e --no-compare > gpurun_out/bench_${TAG}_${WL}_$CC.json 2>&1; echo "bench $WL cc=$CC rc=$?"
  python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/bench_${TAG}_${WL}_$CC.json') if l.startswith('{')][-1])
print('  value', d['value'], 'ms/step', d['ms_per_step'], {k:round(v['ms_total']/v['launches'],3) for k,v in d['kernel_ms'].items()})
PY
done; done
