#!/bin/bash
# comparison paths + plain contraction check: parity tests, then bench lines with compare legs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_comparison.py tests/test_gpu_nested.py tests/test_gpu_math_modes.py -m gpu -q -x > gpurun_out/cmp_pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/cmp_pt.log
for wl in c2 c3; do
timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/cmp_$wl.json 2>gpurun_out/cmp_$wl.err; echo "bench $wl rc=$?"
python - <<PY
import json
d=json.load(open('gpurun_out/cmp_$wl.json'))
print(d['value'], d['ms_per_step'], [(p['layer'],p['ms']) for p in d['per_layer']])
for k,v in d['compare'].items(): print(' ',k, v['ms_per_step'], v.get('roofline_frac'), [round(q.get('ms',0),3) for q in v['per_layer']])
PY
done
