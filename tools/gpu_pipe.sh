TAG=${1:-pipe}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_$TAG.log
for CFG in "1 0" "2 0" "4 0" "4 120" "4 96" "8 96" "8 120"; do
  set -- $CFG
  NW_PIPE_CHUNKS=$1 NW_GEMM_CTAS=$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-compare > gpurun_out/bench_${TAG}_$1_$2.json 2>&1; echo "bench chunks=$1 ctas=$2 rc=$?"
  python - <<PY
import json
try:
    d=json.loads([l for l in open('gpurun_out/bench_${TAG}_$1_$2.json') if l.startswith('{')][-1])
    print('  value', d['value'], 'ms/step', d['ms_per_step'], [p['ms'] for p in d['per_layer']])
except Exception as e: print('  no bench line', e); print(open('gpurun_out/bench_${TAG}_$1_$2.json').read()[-1500:])
PY
done
