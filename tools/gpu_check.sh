#!/bin/bash
# GPU test suite + default bench line (quick check of a build): bash tools/gpu_check.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/check_pt.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/check_pt.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/check_bench.json 2> gpurun_out/check_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/check_bench.json'));print(d['value'],d['ms_per_step'],d.get('graph'),d['roofline']['frac'],d['roofline']['avg_launch_ms']); print([(p['layer'],p['ms']) for p in d['per_layer']]); print(d['e2e'])"
