TAG=${1:-wl}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_$TAG.log; grep -E "^FAILED" gpurun_out/pt_$TAG.log | head
for CFG in "c1 0" "c3 0" "c4 0" "c4 4" "c5 0" "c5 4"; do
  set -- $CFG
  MO=""; [ "$2" != "0" ] && MO="--m-outer $2"
  timeout 600 python bench.py --workload $1 $MO --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}_$1_$2.json 2>&1; echo "bench $1 m=$2 rc=$?"
  python - <<PY
import json
try:
    d=json.loads([l for l in open('gpurun_out/bench_${TAG}_$1_$2.json') if l.startswith('{')][-1])
    print('  value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], [(p['layer'], p['ms'], p['tflops_direct_equiv']) for p in d['per_layer']], d['compare'], {k:round(v['ms_total']/v['launches'],3) for k,v in d['kernel_ms'].items()})
except Exception as e: print(' fail', e, open('gpurun_out/bench_${TAG}_$1_$2.json').read()[-800:])
PY
done
