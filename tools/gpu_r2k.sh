#!/bin/bash
# TMA input transform: 16 vs 32 channels per task, bf16 (C3) and fp32 (C2, NW_ITMA_F32=1) vs first-round kernel
NW_ITMA_CC=32 python -m pytest tests/test_gpu_env_variants.py tests/test_gpu_nested.py -q -p no:cacheprovider -k "INPUT_TMA or tma_input" > gpurun_out/r2k_tests.log 2>&1
NW_ITMA_F32=1 NW_ITMA_CC=32 python -m pytest tests/test_gpu_nested.py -q -p no:cacheprovider -k "bf16x3_tensor_core_parity or tma_input" >> gpurun_out/r2k_tests.log 2>&1
grep -E "passed|failed" gpurun_out/r2k_tests.log
for wl in c2 c3; do
  for v in "NW_ITMA_CC=16" "NW_ITMA_CC=32" "NW_ITMA_F32=1 NW_ITMA_CC=16" "NW_ITMA_F32=1 NW_ITMA_CC=32" "NW_INPUT_TMA=0"; do
    env $v python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu --no-compare --no-e2e > /tmp/b.json 2>/dev/null
    python -c "
import json; d=json.load(open('/tmp/b.json')); print('$wl', '$v', d['ms_per_step'], round(d['kernel_ms']['input_transform']['ms_total']/d['kernel_ms']['input_transform']['launches'],4))"
  done
done
