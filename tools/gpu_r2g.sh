#!/bin/bash
python -m pytest tests/test_gpu_env_variants.py tests/test_gpu_nested.py -q -p no:cacheprovider -k "INPUT_TMA or tma_input" > gpurun_out/r2g_tests.log 2>&1
python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu --no-compare --no-e2e > gpurun_out/r2g_bench_c3.json 2> gpurun_out/r2g_bench_c3.err
tail -3 gpurun_out/r2g_tests.log
python -c "
import json; d=json.load(open('gpurun_out/r2g_bench_c3.json')); print(d['value'], d['ms_per_step'], {k:(v['launches'],round(v['ms_total']/v['launches'],4)) for k,v in d['kernel_ms'].items()}, d['roofline_step'])"
