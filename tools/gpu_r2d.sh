#!/bin/bash
# round 2: TMA input transform after the 16-byte box-start fix
python -m pytest tests/test_gpu_env_variants.py -q -p no:cacheprovider -k "INPUT_TMA" > gpurun_out/r2d_tests.log 2>&1
python -m pytest tests/test_gpu_nested.py -q -p no:cacheprovider -k "tma_input" >> gpurun_out/r2d_tests.log 2>&1
for wl in c2 c3; do
  python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu --no-compare --no-e2e > gpurun_out/r2d_bench_$wl.json 2> gpurun_out/r2d_bench_$wl.err
  NW_INPUT_TMA=0 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu --no-compare --no-e2e > gpurun_out/r2d_bench_${wl}_old.json 2>> gpurun_out/r2d_bench_$wl.err
done
grep -E "passed|failed" gpurun_out/r2d_tests.log
for f in gpurun_out/r2d_bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], {k:(v['launches'],round(v['ms_total']/v['launches'],4)) for k,v in d['kernel_ms'].items()}, [ (p['layer'],p['ms']) for p in d['per_layer']])"; done
