mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -x -q -k "fp32_simt or lib_loaded or mixed or determin" > gpurun_out/pt_fp32.log 2>&1; echo "fp32 rc=$?"
tail -5 gpurun_out/pt_fp32.log
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pt_all.log 2>&1; echo "all rc=$?"
tail -30 gpurun_out/pt_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_c2.log
