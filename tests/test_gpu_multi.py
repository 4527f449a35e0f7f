"""bench.py --gpus 2 end to end over NCCL (needs >= 2 GPUs on the box; skipped otherwise).
The run re-executes itself under torch.distributed.run, transforms U on rank 0 only,
broadcasts it, times both ranks (max over ranks) and checks every rank's outputs against
rank 0's recomputation bit for bit."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_bench_two_ranks_nccl():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3", "--no-cpu", "--no-compare", "--no-e2e"],
                       capture_output=True, text=True, timeout=900, env={**os.environ, "NCCL_DEBUG": "INFO"})
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    out = json.loads(line)
    assert out["n_gpus"] == 2
    assert out["multi_gpu"]["bit_identical_to_1_rank"] is True
    assert "NCCL" in r.stdout + r.stderr


def test_bench_two_ranks_one_gpu_orchestration():
    # the same multi-rank path (re-exec under torchrun, U on rank 0 + broadcast, max-over-ranks
    # timing, bit-identity check against rank 0's recomputation) on a 1-GPU box: both ranks share
    # cuda:0 over gloo (NCCL refuses two ranks on one device).  The ranks' kernels are independent;
    # the timing is contended and not a measurement.
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3", "--no-cpu", "--no-compare", "--no-e2e", "--workload", "c1"],
                       capture_output=True, text=True, timeout=900, env={**os.environ, "NW_BENCH_BACKEND": "gloo"})
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert out["n_gpus"] == 2
    assert out["multi_gpu"]["bit_identical_to_1_rank"] is True
    assert out["multi_gpu"]["u_broadcast_bytes"] > 0
