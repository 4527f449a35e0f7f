#!/bin/bash
# round 2: TMA input transform -- bit-identity vs the first-round kernel, full-size parity, timing
set -x
python -m pytest tests/test_gpu_env_variants.py -q -p no:cacheprovider -k "INPUT_TMA" > gpurun_out/r2c_tests.log 2>&1
python -m pytest "tests/test_gpu_fullsize.py" -q -p no:cacheprovider -k "full_tensor and (c3 or c2k9)" -s >> gpurun_out/r2c_tests.log 2>&1
for wl in c2 c3; do
  python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu --no-compare --no-e2e > gpurun_out/r2c_bench_$wl.json 2> gpurun_out/r2c_bench_$wl.err
  NW_INPUT_TMA=0 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu --no-compare --no-e2e > gpurun_out/r2c_bench_${wl}_old.json 2>> gpurun_out/r2c_bench_$wl.err
done
tail -5 gpurun_out/r2c_tests.log
for f in gpurun_out/r2c_bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], {k:(v['launches'],v['ms_total']) for k,v in d['kernel_ms'].items()})"; done
