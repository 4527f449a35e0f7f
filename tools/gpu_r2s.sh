#!/bin/bash
# round-2 re-entry check: GPU tests, smoke, C2 bench line, and the in-launch L2 bandwidth study
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2s_smi.txt 2>&1
timeout 300 ./tools/l2_bw2.bin > gpurun_out/r2s_l2.txt 2>&1; echo "l2 rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2s_pt.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2s_pt.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r2s_bench.json
