TAG=${1:-c4}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_$TAG.log; grep -E "^FAILED" gpurun_out/pt_$TAG.log | head
for WL in c4 c5 c2; do
  timeout 600 python bench.py --workload $WL --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_${TAG}_$WL.json 2>&1; echo "bench $WL rc=$?"
  python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/bench_${TAG}_$WL.json') if l.startswith('{')][-1])
print('  value', d['value'], 'ms', d['ms_per_step'], [(p['layer'], p['ms'], p['tflops_direct_equiv']) for p in d['per_layer']], d['compare'], {k:round(v['ms_total']/v['launches'],3) for k,v in d['kernel_ms'].items()})
PY
done
