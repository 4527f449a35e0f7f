# usage: bash tools/gpu_iter.sh <tag> [layer] [kernel-regex ...]
#   GPU parity tests, a quick bench line, and (optionally) ncu --set full of the named kernels on one layer.
TAG=${1:-it}; LAYER=${2:-c2k9}; shift 2 || true
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pt_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - <<PY
import json
try:
    d=json.loads([l for l in open('gpurun_out/bench_$TAG.json') if l.startswith('{')][-1])
    print('value', d['value'], 'ms/step', d['ms_per_step'], 'e2e', d['e2e'] and d['e2e']['value'])
    print('kernels', d['kernel_ms']); print('roof', d['roofline']); print('per_layer', d['per_layer']); print('compare', d['compare'])
except Exception as e: print('no bench line', e); print(open('gpurun_out/bench_$TAG.err').read()[-3000:])
PY
if [ $# -gt 0 ]; then
  timeout 300 python tools/prof_layer.py $LAYER > gpurun_out/prof_plain_$TAG.log 2>&1 && \
  for K in "$@"; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_${LAYER}_$K python tools/prof_layer.py $LAYER > gpurun_out/ncu_${K}_$TAG.log 2>&1; echo "ncu $K rc=$?"
  done
fi
