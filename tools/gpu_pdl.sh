TAG=${1:-pdl}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_$TAG.log; grep -E "^FAILED" gpurun_out/pt_$TAG.log | head
for P in 0 1; do for WL in c2 c3; do
  NW_PDL=$P timeout 600 python bench.py --workload $WL --steps 10 --warmup 3 --no-cpu --no-compare > gpurun_out/bench_${TAG}_${WL}_$P.json 2>&1; echo "bench $WL pdl=$P rc=$?"
  python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/bench_${TAG}_${WL}_$P.json') if l.startswith('{')][-1])
print('  value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], [(p['layer'], p['ms']) for p in d['per_layer']], {k:round(v['ms_total']/v['launches'],3) for k,v in d['kernel_ms'].items()})
PY
done; done
