"""Off-default code paths selected by environment tunables (include/nw.h), each run in a
fresh process (the library reads them once) and compared with the default path.

Tunables that only change scheduling (chunking, CTA pairs, K-block width, unit size,
launch mode, channels per CTA) must give BIT-IDENTICAL outputs: every output is the
same sequence of fp32 operations.  Tunables that change the arithmetic (NW_FUSE_AI=0 / 1:
the inner output level leaves the contraction epilogue / is applied along w only; NW_FUSED_C1=0: the three-kernel
pipeline instead of the single fused kernel) are checked against the FP64 oracle with the
BASELINE gate.  Also the bench's end-to-end configuration: nw_conv_forward_host at N = 32
with NW_HOST_CHUNKS=4 (chunk schedule 1,2,4,8,8,4,2,1... with a short tail) bit for bit
against the device entry point.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import synth
from test_gpu_nested import _ref, check_parity

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(spec, env=None, host=False, tmp=None):
    out = os.path.join(str(tmp), f"y_{abs(hash((json.dumps(spec, sort_keys=True), json.dumps(env), host)))}.npy")
    e = dict(os.environ)
    e.update(env or {})
    cmd = [sys.executable, os.path.join(HERE, "_variant_run.py"), json.dumps(spec), out] + (["host"] if host else [])
    r = subprocess.run(cmd, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


C2 = {"config": "c2k9", "N": 3, "H": 47, "W": 53, "Cin": 64, "Cout": 64}
C3 = {"config": "c3", "N": 2, "H": 40, "W": 37, "Cin": 64, "Cout": 256}
C4B = {"config": "c4b", "N": 3, "H": 45, "W": 40, "Cin": 16, "Cout": 32}

BITWISE = [
    (C2, {"NW_PIPE_CHUNKS": "2"}),
    (C2, {"NW_PIPE_CHUNKS": "3"}),            # N = 3 over 3 chunks; with N = 5 below a short tail
    ({**C2, "N": 5}, {"NW_PIPE_CHUNKS": "3"}),
    (C2, {"NW_PDL": "1"}),
    (C2, {"NW_KBK": "64"}),
    (C2, {"NW_IN_CC": "16"}),
    (C2, {"NW_IN_CC": "64"}),
    (C3, {"NW_CLUSTER": "1"}),
    (C2, {"NW_CLUSTER": "1"}),                # level-2 fused contraction without CTA pairs (no A multicast)
    (C4B, {"NW_CLUSTER": "1"}),
    ({**C2, "N": 7, "H": 50, "W": 45}, {"NW_PIPE_CHUNKS": "2", "NW_GEMM_CTAS": "3"}),   # odd grid cap: pairs + a spare CTA slot
    (C3, {"NW_GEMM_G": "1"}),
    (C3, {"NW_PDL": "1"}),
    (C4B, {"NW_KBK": "64"}),
    (C4B, {"NW_PIPE_CHUNKS": "2"}),
    (C3, {"NW_PIPE_CHUNKS": "2", "NW_GEMM_CTAS": "1"}),   # grid cap below a CTA pair: unpaired launch
    # persistent TMA-fed input transform (bf16 x) vs the first-round kernel: same fp32 operation
    # sequence.  The TMA path needs 16-byte x rows (W % 8 == 0 for bf16); window starts at every
    # 16-byte phase (pad 2 / 3 / 4, advance 9 / 12) and several tasks per CTA (in-loop refill)
    ({**C3, "W": 40}, {"NW_INPUT_TMA": "0"}),                    # 256 channels
    ({**C3, "N": 6, "H": 64, "W": 64}, {"NW_INPUT_TMA": "0"}),   # 6 x 6 x 3 x 16 tasks
    ({**C2, "W": 56, "dtype": "bf16"}, {"NW_INPUT_TMA": "0"}),
    ({**C2, "N": 9, "H": 64, "W": 64, "dtype": "bf16"}, {"NW_INPUT_TMA": "0"}),   # 576 tasks
    ({**C2, "config": "c2k5", "W": 56, "dtype": "bf16"}, {"NW_INPUT_TMA": "0"}),  # F(4,2)(x)F(3,3), pad 2
    ({**C2, "config": "c2k7", "N": 5, "H": 61, "W": 64, "dtype": "bf16"}, {"NW_INPUT_TMA": "0"}),  # pad 3
    ({"config": "c2k9", "N": 2, "H": 40, "W": 40, "Cin": 32, "Cout": 64, "m_o": 3, "dtype": "bf16"},
     {"NW_INPUT_TMA": "0"}),
    ({"config": "c2k9", "N": 3, "H": 50, "W": 48, "Cin": 64, "Cout": 32, "m_o": 3, "dtype": "bf16"},
     {"NW_INPUT_TMA": "0"}),
    # warp-specialised TMA input transform (default for r_o = 3, fp32 and bf16 x) vs the first-round
    # kernel (fp32) and the single-role TMA kernel (bf16)
    ({**C2, "N": 9, "H": 64, "W": 64}, {"NW_ITMA_WS": "0"}),
    ({**C2, "W": 56}, {"NW_ITMA_WS": "0"}),
    ({**C3, "N": 6, "H": 64, "W": 64}, {"NW_ITMA_WS": "0"}),
    # streamed pipeline: kernels on disjoint SM sets linked by completion counters; 9 x 36 slices =
    # three 128-slice blocks, the last one partial
    ({**C2, "N": 9, "H": 64, "W": 64}, {"NW_STREAM": "1"}),
    ({**C2, "N": 9, "H": 64, "W": 64}, {"NW_STREAM": "2"}),
    ({**C2, "N": 9, "H": 64, "W": 64}, {"NW_STREAM": "3", "NW_STREAM_SB": "2"}),
    ({**C2, "N": 9, "H": 64, "W": 64, "dtype": "bf16"}, {"NW_STREAM": "3"}),
    ({**C2, "config": "c2k5", "N": 9, "H": 64, "W": 64}, {"NW_STREAM": "3", "NW_STREAM_IT": "40"}),
]


@pytest.mark.parametrize("spec,env", BITWISE, ids=[f"{s['config']}-{'-'.join(f'{k}={v}' for k, v in e.items())}"
                                                   for s, e in BITWISE])
def test_scheduling_tunables_bit_identical(spec, env, tmp_path):
    # the streamed pipeline's counters belong to the w-only fused contraction (NW_FUSE_AI=1)
    base = {"NW_FUSE_AI": "1"} if "NW_STREAM" in env else None
    # C3's scheduling tunables belong to the plain contraction (the default for 256 output channels
    # is the 128-channel fused kernel, NW_FUSE_WIDE)
    if spec.get("config") == "c3" and spec.get("Cout") == 256:
        base = {"NW_FUSE_WIDE": "0"}
    y0 = _run(dict(spec), base, tmp=tmp_path)
    y1 = _run(dict(spec), {**env, **(base or {})}, tmp=tmp_path)
    assert y0.shape == y1.shape
    assert np.array_equal(y0, y1), float(np.abs(y0 - y1).max())


ARITH = [
    (C2, {"NW_FUSE_AI": "0"}),
    (C2, {"NW_FUSE_AI": "1"}),      # inner output level along w only (default 2: both axes)
    (C4B, {"NW_FUSE_AI": "1"}),
    (C3, {"NW_FUSE_WIDE": "0"}),    # plain contraction instead of the 128-channel fused kernel
    ({**C3, "Cout": 128}, {"NW_FUSE_AI": "2"}),   # 128 output channels: the fused kernel without a CTA pair
    ({"config": "c5_conv1", "N": 2, "H": 37, "W": 45}, {"NW_FUSED_C1": "0"}),
]


@pytest.mark.parametrize("spec,env", ARITH, ids=["fuse_ai_off", "fuse_ai_w_c2", "fuse_ai_w_c4b", "fuse_wide_off", "fuse_wide_128", "fused_c1_off"])
def test_arithmetic_tunables_meet_gate(spec, env, tmp_path):
    y = _run(dict(spec), env, tmp=tmp_path)
    s = dict(spec)
    extra = {k: s.pop(k) for k in ("m_o", "r_o", "dtype", "xdist") if k in s}
    layer = synth.small(synth.CONFIGS[s.pop("config")], **s).with_(**extra)
    check_parity(y, _ref(layer, synth.make_inputs(layer)), "bf16x3", layer.dtype)


def test_bench_e2e_configuration_bit_identical(tmp_path):
    # bench.py's e2e leg: full C2 K=9 (N = 32) through nw_conv_forward_host with NW_HOST_CHUNKS=4
    spec = {"config": "c2k9"}
    y_dev = _run(dict(spec), None, tmp=tmp_path)
    y_host = _run(dict(spec), {"NW_HOST_CHUNKS": "4"}, host=True, tmp=tmp_path)
    assert np.array_equal(y_dev, y_host)


@pytest.mark.parametrize("chunks,N", [("3", 7), ("5", 11)])
def test_host_chunk_schedules_bit_identical(chunks, N, tmp_path):
    # ramp 1, 2, .. / full chunks / short tail / ramp down, with N not a multiple of the chunk
    spec = {**C2, "N": N, "Cin": 32, "Cout": 32}
    y_dev = _run(dict(spec), None, tmp=tmp_path)
    y_host = _run(dict(spec), {"NW_HOST_CHUNKS": chunks}, host=True, tmp=tmp_path)
    assert np.array_equal(y_dev, y_host)
