TAG=${1:-mo}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pt_$TAG.log
for MO in 3 4 5; do
for WL in c2 c3; do
  timeout 600 python bench.py --workload $WL --m-outer $MO --steps 5 --warmup 3 --no-cpu --no-e2e --no-compare > gpurun_out/bench_${TAG}_${WL}_m$MO.json 2> gpurun_out/bench_${TAG}_${WL}_m$MO.err; echo "bench $WL m_o=$MO rc=$?"
  python - <<PY
import json
try:
    d=json.loads([l for l in open('gpurun_out/bench_${TAG}_${WL}_m$MO.json') if l.startswith('{')][-1])
    print('  value', d['value'], 'ms/step', d['ms_per_step'], {k:round(v['ms_total']/v['launches'],3) for k,v in d['kernel_ms'].items()})
except Exception as e: print('  no bench line', e); print(open('gpurun_out/bench_${TAG}_${WL}_m$MO.err').read()[-2000:])
PY
done; done
