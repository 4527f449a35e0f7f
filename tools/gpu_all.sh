# usage: bash tools/gpu_all.sh <tag>  -- full GPU test suite, smoke, and a bench line per workload
TAG=${1:-all}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pt_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_$TAG.log
for WL in c2 c1 c3 c4 c5; do
  timeout 600 python bench.py --workload $WL --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}_$WL.json 2> gpurun_out/bench_${TAG}_$WL.err; echo "bench $WL rc=$?"
  python - <<PY
import json
try:
    d=json.loads([l for l in open('gpurun_out/bench_${TAG}_$WL.json') if l.startswith('{')][-1])
    print('  value', d['value'], 'ms/step', d['ms_per_step'], 'e2e', d['e2e'] and d['e2e']['value'], 'roof', d['roofline'] and (d['roofline']['kernel'], d['roofline']['frac']))
    print('  per_layer', [(p['layer'], p['ms'], p['tflops_direct_equiv']) for p in d['per_layer']]); print('  compare', d['compare'])
except Exception as e: print('  no bench line', e); print(open('gpurun_out/bench_${TAG}_$WL.err').read()[-2000:])
PY
done
