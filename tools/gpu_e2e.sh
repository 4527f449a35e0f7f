TAG=${1:-e2e}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_$TAG.log
for HC in 4 8; do
  NW_HOST_CHUNKS=$HC timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-compare > gpurun_out/bench_${TAG}_$HC.json 2>&1; echo "bench host_chunks=$HC rc=$?"
  python - <<PY
import json
d=json.loads([l for l in open('gpurun_out/bench_${TAG}_$HC.json') if l.startswith('{')][-1])
print('  value', d['value'], 'e2e', d['e2e'], 'roof', d['roofline'])
PY
done
