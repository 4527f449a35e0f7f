"""bench.py's roofline accounting on the CPU: algorithmic bytes per launch from the plan info
 and the dominant-kernel pick, for every workload's layers -- including the
single-kernel (one input channel) layers, whose three-kernel pipeline never launches."""
import bench
import synth
from paper_2102_13272_b200 import _lib


def _info(l):
    return _lib.Plan(l.K, l.stride, l.m_o, l.m_i, l.Cin, l.Cout, transposed=l.transposed,
                     output_padding=l.output_padding, outer_taps=l.r_o).info()


def test_c2k9_bytes_match_design_table():
    # per slice V = 900 points x 4 B per channel, M'' = (l_o m_i)^2 = 324 rows x 4 B
    # (the contraction's epilogue applies the inner output level along both axes)
    l = synth.CONFIGS["c2k9"]
    w = bench.kernel_work(l, _info(l), "bf16x3")
    T = l.N * 11 * 11                          # 128 / 12 -> 11 tiles per axis
    x_b = l.N * l.Cin * l.H * l.W * 4
    assert w["input_transform"]["bytes"] == x_b + 900 * T * 64 * 4
    assert w["contraction_tc"]["bytes"] == 900 * T * 64 * 4 + 900 * 64 * 64 * 4 + 324 * T * 64 * 4
    assert w["contraction_tc"]["flops"] == 3 * 2 * 900 * T * 64 * 64


def test_single_kernel_layers_and_roofline_pick():
    peaks = bench.load_peaks()
    for wl, names in bench.WORKLOADS.items():
        layers = [synth.CONFIGS[n] for n in names]
        works = [bench.kernel_work(l, _info(l), "bf16x3") for l in layers]
        for l, w in zip(layers, works):
            single = l.Cin == 1 and l.stride == 1 and not l.transposed
            assert ("fused_c1" in w) == single, (wl, l.name)
            # at most four contraction outputs (C5 deconv: 4 phases, SRCNN 1 <- 32): single kernel too
            small_out = (not single and not l.depthwise and (4 if l.transposed else 1) * l.Cout <= 4
                         and (l.stride == 1 or l.transposed) and not l.prelu)
            assert ("fused_co" in w) == small_out, (wl, l.name)
        # every kernel kind that launches has work attributed; the pick never divides by zero
        kinds = {k for w in works for k in w if k != "filter_transform"}
        prof = {k: (len(layers), 1.0 + i) for i, k in enumerate(sorted(kinds))}
        r = bench.roofline(prof, works, "bf16x3", peaks, 1, layers)
        assert r["frac"] > 0 and r["kernel"] in kinds


def test_multi_gpu_launch_command(monkeypatch):
    # `bench.py --gpus N` without a torchrun environment re-executes itself as N ranks on one node
    cmd = bench.torchrun_cmd(["--gpus", "4", "--steps", "3"], 4, 29555)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"] and cmd[-5].endswith("bench.py")

    class A:
        gpus = 2
    monkeypatch.setenv("WORLD_SIZE", "4")
    import pytest
    with pytest.raises(SystemExit):
        bench.ensure_ranks(A())          # torchrun world size must match --gpus
    monkeypatch.setenv("WORLD_SIZE", "2")
    bench.ensure_ranks(A())              # consistent: runs in this process
    monkeypatch.delenv("WORLD_SIZE")
    A.gpus = 1
    bench.ensure_ranks(A())              # single GPU: no re-exec
