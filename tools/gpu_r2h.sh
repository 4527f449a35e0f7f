#!/bin/bash
python -m pytest tests/test_gpu_depthwise.py -q -p no:cacheprovider > gpurun_out/r2h_tests.log 2>&1
tail -3 gpurun_out/r2h_tests.log
python bench.py --workload table1 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2h_bench_table1.json 2> gpurun_out/r2h_bench_table1.err
python -c "
import json; d=json.load(open('gpurun_out/r2h_bench_table1.json')); print(d['value'], d['ms_per_step'], [(p['layer'],p['ms']) for p in d['per_layer']]); print({k:[(l['layer'],l.get('ms'),l.get('nested_speedup')) for l in v.get('per_layer',[])] for k,v in d['compare'].items()})" || tail -20 gpurun_out/r2h_bench_table1.err
