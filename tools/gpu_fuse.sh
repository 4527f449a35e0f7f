TAG=${1:-fuse}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_$TAG.log; grep -E "^FAILED|Error" gpurun_out/pt_$TAG.log | head -5
for F in 1; do for WL in c2 table1 c5 c4; do
  NW_FUSE_AI=$F timeout 600 python bench.py --workload $WL --steps 10 --warmup 3 --no-cpu --no-e2e --no-compare > gpurun_out/bench_${TAG}_${WL}_$F.json 2>&1; echo "bench $WL fuse=$F rc=$?"
  python - <<PY
import json
try:
    d=json.loads([l for l in open('gpurun_out/bench_${TAG}_${WL}_$F.json') if l.startswith('{')][-1])
    print('  value', d['value'], 'ms/step', d['ms_per_step'], {k:round(v['ms_total']/v['launches'],3) for k,v in d['kernel_ms'].items()})
except Exception as e: print(' fail', e); print(open('gpurun_out/bench_${TAG}_${WL}_$F.json').read()[-1500:])
PY
done; done
