#!/usr/bin/env python
"""Benchmark: nested-Winograd convolution layers on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c3|c4|c5] [--math bf16x3|fp32|bf16] [--path nested|ola|direct]

A step is one pass of the per-batch hot path over one batch of synthetic input:
for every layer of the workload, nested input transform -> per-point
contraction -> output transform (nw_conv_forward).  The filter transform (once
per weight set) runs before timing on rank 0 and its
result U is broadcast over NCCL; its time is reported separately.
Default workload = BASELINE configs[1] (K in {5,7,9}, N=32, Cin=Cout=64,
128x128, fp32): the configuration the metric is quoted on.
Multi-GPU: one process per GPU (torchrun), each rank processes its own batch
of N images (weak scaling), time = max over ranks of the CUDA-event time.

Rank 0 prints ONE JSON line.  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "direct-equiv TFLOP/s & % roofline, 5×5–9×9 conv layers, 1/2/4/8 B200"
WORKLOADS = {
    "c1": ["c1"],
    "c2": synth.C2_SWEEP,
    "c3": ["c3"],
    "c4": ["c4a", "c4b"],
    "c5": ["c5_conv1", "c5_deconv"],
    "table1": synth.TABLE1,
    "c5net": synth.C5_NET,
}
# workloads run as one network: layer i+1 consumes layer i's output (FSRCNN-s forward);
# layers with K <= 3 (1x1, 3x3) run the direct implicit-GEMM path of the library
CHAINS = {"c5net"}
WORKLOAD_DESC = {
    "c5net": "configs[4] as a network: conv5x5 1->32 +PReLU (nested) -> 1x1 32->5 -> 3x3 5->5 -> 1x1 5->32 "
             "(+PReLU each, direct implicit GEMM) -> 9x9 s2 deconv 32->1 (nested), N=16, 540x960 -> 1080x1920",
    "table1": "paper Table I shapes (P:154-160): SRCNN 9x9 64<-1, PNASNet depthwise 7x7 54 (83x83), "
              "SRCNN 5x5 32<-64, 5x5 1<-32 (256x256), N=8, fp32",
    "c1": "configs[0]: 5x5 s1 p2, N=1, Cin=Cout=16, 32x32, fp32, F(2,3)(x)F(2,3) + coverage phases",
    "c2": "configs[1]: filter-size sweep K in {5,7,9}, s1 same pad, N=32, Cin=Cout=64, 128x128, fp32",
    "c3": "configs[2]: 9x9 s1 p4, N=64, Cin=Cout=256, 64x64, bf16 storage, fp32 accumulate",
    "c4": "configs[3]: 7x7 s2 p3 N=256 3->64 224x224 + 9x9 s2 p4 N=256 64->64 112x112, fp32",
    "c5": "configs[4]: FSRCNN-s nested layers: conv5x5 1->32 (+PReLU) and 9x9 s2 deconv 32->1, N=16, 540x960",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5", "table1", "c5net"])
    ap.add_argument("--math", default="bf16x3", choices=["bf16x3", "fp32", "bf16"])
    ap.add_argument("--path", default="nested", choices=["nested", "ola", "direct"])
    ap.add_argument("--m-outer", type=int, default=None,
                    help="outer kernel F(m,3) of the nested plan (default: the config's, 3)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-compare", action="store_true", help="skip the OLA / direct comparison lines")
    ap.add_argument("--layer-streams", type=int, default=1,
                    help="1 (default): the workload's independent layers (not the c5net chain) run "
                         "concurrently, each on its own stream and workspace; 0: one stream")
    return ap.parse_args()


# ----------------------------------------------------------------------------
# clocks during the timed region (NVML, 20 ms period)
# ----------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # pragma: no cover - no NVML
            self.ok = False
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": sorted(self.reasons - {"gpu_idle"})}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "sm_max_mhz": d.get("sm_max_mhz", 1965.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0,
            "source": "fallback"}


# ----------------------------------------------------------------------------
# algorithmic work per launch of each kernel kind
# ----------------------------------------------------------------------------
def kernel_work(layer, info, math, path="nested"):
    """Algorithmic bytes and flops of one launch of each kernel for one layer."""
    es = 2 if layer.dtype == "bf16" else 4
    if path == "direct":
        # implicit GEMM over the (phase) pixel grid extended by Kp - 1 (a5)
        Kp = info["Kp"]
        if layer.transposed:
            Hq, Wq = -(-layer.Ho // 2), -(-layer.Wo // 2)
        else:
            Hq, Wq = layer.Ho, layer.Wo
        T = layer.N * (Hq + Kp - 1) * (Wq + Kp - 1)
        x_b = layer.N * layer.Cin * layer.H * layer.W * es
        y_b = layer.N * layer.Cout * layer.Ho * layer.Wo * es
        v_b, m_b = T * info["cin_e"] * 4, T * info["cout_e"] * 4
        u_b = Kp * Kp * info["cout_e"] * info["cin_e"] * 4
        passes = {"bf16x3": 3, "bf16": 1, "fp32": 1}[math]
        flops = 2 * T * Kp * Kp * info["cin_e"] * info["cout_e"]
        return {"pack_input": {"bytes": x_b + v_b, "flops": 0},
                "contraction_tc": {"bytes": v_b + u_b + m_b, "flops": flops * passes},
                "contraction_fp32_simt": {"bytes": v_b + u_b + m_b, "flops": flops},
                "unpack_output": {"bytes": m_b + y_b, "flops": 0},
                "filter_transform": {"bytes": u_b, "flops": 0}}
    P = info["points"]
    adv, nph = info["tile_out"], info["n_phase"]
    if layer.transposed:
        Hq, Wq = -(-layer.Ho // 2), -(-layer.Wo // 2)
    else:
        Hq, Wq = layer.Ho, layer.Wo
    T = layer.N * -(-Hq // adv) * -(-Wq // adv) * nph * nph
    cin_e, cout_e = info["cin_e"], info["cout_e"]
    x_b = layer.N * layer.Cin * layer.H * layer.W * es
    y_b = layer.N * layer.Cout * layer.Ho * layer.Wo * es
    v_b = P * T * cin_e * 4          # fp32 or bf16 hi+lo
    m_b = info["m_rows"] * T * cout_e * 4   # M, or M' (inner output level fused into the contraction)
    u_b = P * cout_e * cin_e * 4
    passes = {"bf16x3": 3, "bf16": 1, "fp32": 1}[math]
    flops = 2 * P * T * cin_e * cout_e
    if layer.depthwise:
        # depthwise (groups = C): no channel contraction; the per-channel product kernel reads V
        # and U and writes M (csrc/depthwise.cu), HBM-bound
        u_b = P * cout_e * 4
        return {
            "input_transform": {"bytes": x_b + v_b, "flops": 0},
            "depthwise_product": {"bytes": v_b + u_b + m_b, "flops": 0},
            "output_transform": {"bytes": m_b + y_b, "flops": 0},
            "filter_transform": {"bytes": u_b, "flops": 0},
        }
    if info.get("single_kernel"):
        # one input channel (fused_c1) or at most four contraction outputs (fused_co): transform,
        # channel sum and output transform in one kernel; HBM traffic is x, U and y only (the
        # kernel is bound by its CUDA-core transforms)
        kind = "fused_c1" if cin_e == 1 else "fused_co"
        return {kind: {"bytes": x_b + u_b + y_b, "flops": 0},
                "filter_transform": {"bytes": u_b, "flops": 0}}
    return {
        "input_transform": {"bytes": x_b + v_b, "flops": 0},
        "contraction_tc": {"bytes": v_b + u_b + m_b, "flops": flops * passes},
        "contraction_fp32_simt": {"bytes": v_b + u_b + m_b, "flops": flops},
        "output_transform": {"bytes": m_b + y_b, "flops": 0},
        "filter_transform": {"bytes": u_b, "flops": 0},
    }


def layer_bounds(layer, info, math, peaks, path="nested"):
    """Per-layer roofline bounds, microseconds.

    compulsory bytes = x + U (or w) + y, each once.  Contraction work of the method:
      nested  "paper" basis: 625 MACs per 9x9 tile per (cin_e, cout_e) -- the paper's
              F(3,3)(x)F(3,3) nesting, i.e. T9 * 625 * Cin_e * Cout_e -- and "plan"
              basis: the plan's own points (e.g. F(4,3)(x)F(3,3): 900 per 12x12 tile);
      ola     25 MACs per 3x3 tile per filter block (Eq. 2.3): T3 * 25 * nb^2 * Cin_e * Cout_e;
      direct  K^2 MACs per output (Eq. 2.1).
    R1 = max(1-pass contraction at the bf16 burst peak, compulsory bytes at HBM peak);
    R2 = the same with the passes the math mode issues (bf16x3: 3);
    R3 = R2's compute term against the path's own algorithmic pipeline bytes (V, M spilled).
    frac = bound / measured time (filled in by the caller)."""
    es = 2 if layer.dtype == "bf16" else 4
    x_b = layer.N * layer.Cin * layer.H * layer.W * es
    y_b = layer.N * layer.Cout * layer.Ho * layer.Wo * es
    cin_e, cout_e, Kp = info["cin_e"], info["cout_e"], info["Kp"]
    if layer.depthwise:   # one product per channel: the "contraction" has Cin_e x Cout_e -> C
        cin_e = 1
    if layer.transposed:
        Hq, Wq = -(-layer.Ho // 2), -(-layer.Wo // 2)
    else:
        Hq, Wq = layer.Ho, layer.Wo
    passes = {"bf16x3": 3, "bf16": 1, "fp32": 1}[math]
    if math == "fp32":   # CUDA-core FP32 FMA peak: 148 SMs x 128 lanes x 2 x max clock
        tpeak = 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6
    else:
        tpeak = peaks["bf16_tflops"] * 1e12
    if path == "nested":
        P9 = 625
        T9 = layer.N * -(-Hq // 9) * -(-Wq // 9)
        macs = T9 * P9 * cin_e * cout_e
        adv, nph = info["tile_out"], info["n_phase"]
        Tp = layer.N * -(-Hq // adv) * -(-Wq // adv) * nph * nph
        macs_plan = Tp * info["points"] * cin_e * cout_e
        u_b = info["points"] * cin_e * cout_e * 4
    elif path == "ola":
        nb = -(-Kp // 3)
        T3 = layer.N * -(-Hq // 3) * -(-Wq // 3)
        macs = macs_plan = T3 * 25 * nb * nb * cin_e * cout_e
        u_b = 25 * nb * nb * cin_e * cout_e * 4
    else:
        macs = macs_plan = layer.direct_flops() // 2
        u_b = (1 if layer.depthwise else layer.Cin) * layer.Cout * layer.K * layer.K * es
    hbm = peaks["hbm_gbs"] * 1e9
    comp_b = x_b + u_b + y_b
    t_b = comp_b / hbm * 1e6
    t1 = 2 * macs / tpeak * 1e6
    t2 = 2 * macs * passes / tpeak * 1e6
    t2_plan = 2 * macs_plan * passes / tpeak * 1e6
    return {"compulsory_bytes": int(comp_b), "macs_paper_basis": int(macs), "macs_plan": int(macs_plan),
            "passes": passes, "r1_us": round(max(t1, t_b), 2), "r2_us": round(max(t2, t_b), 2),
            "r2_plan_us": round(max(t2_plan, t_b), 2), "_t2_compute_us": t2_plan}


def attach_bounds(entry, bounds, works_l, peaks, ms):
    """Add r1/r2/r3 bounds and fractions (bound / measured) to a per-layer entry."""
    hbm = peaks["hbm_gbs"] * 1e9
    pipe_b = 0
    if works_l:
        pipe_b = sum(v["bytes"] for k, v in works_l.items()
                     if k not in ("filter_transform", "contraction_fp32_simt"))
    r3 = max(bounds["_t2_compute_us"], pipe_b / hbm * 1e6) if pipe_b else None
    us = ms * 1e3
    rf = {"r1": {"bound_us": bounds["r1_us"], "frac": round(bounds["r1_us"] / us, 4)},
          "r2": {"bound_us": bounds["r2_us"], "frac": round(bounds["r2_us"] / us, 4),
                 "basis": "paper F(3,3)(x)F(3,3) MACs x passes at bf16 burst peak vs compulsory x+U+y"},
          "r2_plan": {"bound_us": bounds["r2_plan_us"], "frac": round(bounds["r2_plan_us"] / us, 4),
                      "basis": "the plan's own transform points x passes vs compulsory bytes"}}
    if r3 is not None:
        rf["r3"] = {"bound_us": round(r3, 2), "frac": round(r3 / us, 4), "pipeline_bytes": int(pipe_b),
                    "basis": "pipeline bytes (V, M spilled: the implementation's own traffic)"}
    entry["roofline"] = rf
    return entry


def roofline(prof, works, math, peaks, steps, layers):
    """Pick the kernel with the largest total time; achieved = algorithmic work / mean launch time."""
    if not prof:
        return None
    kind = max(prof, key=lambda k: prof[k][1])
    launches, ms = prof[kind]
    ws_ = [w for w in works if kind in w]          # layers that launch this kernel (once per step each)
    bytes_per_launch = sum(w[kind]["bytes"] for w in ws_) / len(ws_)
    flops_per_launch = sum(w[kind]["flops"] for w in ws_) / len(ws_)
    avg_s = ms / launches / 1e3
    hbm = peaks["hbm_gbs"]
    if kind == "contraction_tc":
        tpeak = peaks["bf16_tflops_sustained"]          # kernel timed inside a long step
    elif kind == "contraction_fp32_simt":
        tpeak = 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6 / 1e12   # FP32 FMA lanes x 2 x clock
    else:
        tpeak = None
    t_bytes = bytes_per_launch / (hbm * 1e9)
    t_flops = flops_per_launch / (tpeak * 1e12) if tpeak else 0.0
    # ncu dram read+write bytes per launch of this kernel, averaged over the workload's
    # layers (profiles/traffic.json, written by tools/ncu_summary.py); null if any is missing
    trafile = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = None
    if os.path.exists(trafile):
        tab = json.load(open(trafile))
        vals = [tab.get(f"{kind}:{math}:{l.name}:m{l.m_o}") for l in layers]
        if vals and all(v is not None for v in vals):
            traffic = int(sum(vals) / len(vals))
    if t_flops > t_bytes:
        bound = "tensor" if kind == "contraction_tc" else "alu"
        achieved = flops_per_launch / avg_s / 1e12
        return {"kernel": kind, "bound": bound, "achieved": round(achieved, 2), "peak": round(tpeak, 1),
                "unit": "TFLOP/s", "frac": round(achieved / tpeak, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": int(bytes_per_launch), "avg_launch_ms": round(avg_s * 1e3, 4),
                "launches": launches, "peak_source": peaks["source"]}
    achieved = bytes_per_launch / avg_s / 1e9
    return {"kernel": kind, "bound": "hbm", "basis": "pipeline bytes: the kernel's own operand tensors (for the "
                                                      "contraction V + U + M', i.e. the spilled transform domain; "
                                                      "R3 reading) -- the compulsory-bytes readings R1 / R2 are "
                                                      "in per_layer[*].roofline and roofline_step",
            "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(achieved / hbm, 4), "traffic": traffic,
            "algorithmic_bytes_per_launch": int(bytes_per_launch), "avg_launch_ms": round(avg_s * 1e3, 4),
            "launches": launches, "peak_source": peaks["source"]}


# ----------------------------------------------------------------------------
# CPU oracle timing (bounded sample)
# ----------------------------------------------------------------------------
def oracle_sample_time(layers, target_s=10.0, max_images=None):
    """Time oracle.direct (FP64 Eq. 2.1) on the first images of each layer."""
    import numpy as np

    from oracle import direct
    inputs = [synth.make_inputs(l.with_(N=1)) for l in layers]

    def run(n_img):
        flops = 0
        t0 = time.perf_counter()
        for l, t in zip(layers, inputs):
            x = t["x"].double().numpy()
            w = t["w"].double().numpy()
            for _ in range(n_img):
                if l.transposed:
                    direct.conv_transpose2d(x, w, l.stride, l.pad, l.output_padding)
                elif l.depthwise:
                    direct.conv2d_depthwise(x, w, l.stride, l.pad)
                else:
                    direct.conv2d(x, w, l.stride, l.pad)
            flops += n_img * l.with_(N=1).direct_flops()
        return flops, time.perf_counter() - t0

    f1, t1 = run(1)
    n = max(1, min(max_images or 64, int(target_s / max(t1, 1e-3))))
    if n > 1:
        f1, t1 = run(n)
    return f1, t1, n, np.__version__


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cores_used():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ----------------------------------------------------------------------------
# multi-GPU launch: one process per GPU
# ----------------------------------------------------------------------------
def free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def torchrun_cmd(argv, gpus: int, port: int):
    """The command that re-runs this script as `gpus` ranks on one node (torch.distributed.run,
    rendezvous on 127.0.0.1), forwarding every argument."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def ensure_ranks(args) -> None:
    """`python bench.py --gpus N` with N > 1 and no torchrun environment re-executes itself under
    torch.distributed.run with N ranks (rank 0 prints the JSON line) and exits with its status.
    Under torchrun the world size must equal --gpus."""
    world = os.environ.get("WORLD_SIZE")
    if world is None:
        if args.gpus > 1:
            import subprocess
            r = subprocess.run(torchrun_cmd(sys.argv[1:], args.gpus, free_port()))
            sys.exit(r.returncode)
        return
    if int(world) != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")


def main():
    args = parse()
    ensure_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    layers_all = [synth.CONFIGS[n] for n in WORKLOADS[args.workload]]
    if args.m_outer:
        layers_all = [l.with_(m_o=args.m_outer) if l.m_i == 3 else l for l in layers_all]

    if args.impl == "reference":
        return reference_arm(args, layers_all, world, rank)
    if len(layers_all) > 1 and args.workload not in CHAINS:
        # host chunks per nw_conv_forward_host call (read once by the library, before any call):
        # with the e2e leg's independent layers overlapping on their own streams, 4 measured best
        # (C2: 1 / 2 / 4 / 8 / 16 chunks -> 54 / 72 / 73 / 70 / 64 TFLOP/s,
        # profiles/r3_e2e_chunks.md); a single layer keeps the library default (8)
        os.environ.setdefault("NW_HOST_CHUNKS", "4")

    import torch
    import torch.distributed as dist

    import paper_2102_13272_b200 as nw
    from paper_2102_13272_b200 import _lib
    from paper_2102_13272_b200 import dist as nwd

    # NW_BENCH_BACKEND=gloo (tests only) runs the multi-rank orchestration on a box with fewer
    # GPUs than ranks: ranks then share a device, which NCCL refuses; the product run is NCCL
    backend = os.environ.get("NW_BENCH_BACKEND", "nccl")
    dev_index = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    math = {"bf16x3": nw.MATH_BF16X3, "fp32": nw.MATH_FP32_SIMT, "bf16": nw.MATH_BF16}[args.math]
    peaks = load_peaks()
    stream = torch.cuda.current_stream()

    chain = args.workload in CHAINS
    paths = [("direct" if (chain and l.K <= 3) else args.path) for l in layers_all]
    convs, xs, ys, works = [], [], [], []
    filt_ms, bcast_ms, bcast_bytes = 0.0, 0.0, 0
    for li, l in enumerate(layers_all):
        t = synth.make_inputs(l.with_(seed=l.seed + 1000 * rank)) if rank else synth.make_inputs(l)
        if chain and li > 0:
            t["x"] = None                                   # consumes the previous layer's output
        w = synth.make_inputs(l, x=False)["w"].to(dev)     # same weights on every rank
        slopes = torch.full((l.Cout,), synth.PRELU_SLOPE, device=dev) if l.prelu else None
        conv = nw.NestedConv2d(w, l.stride, l.pad, l.m_o, l.m_i, math, transposed=l.transposed, outer_taps=l.r_o,
                               output_padding=l.output_padding, prelu_slopes=slopes, transform=False,
                               depthwise=l.depthwise)
        # filter transform once, on rank 0 only (timed separately); the other ranks receive U
        # through the one collective of the run: a broadcast over NCCL (NVLink / NVSwitch)
        if rank == 0:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            conv.transform_filter()
            e1.record()
            torch.cuda.synchronize()
            filt_ms += e0.elapsed_time(e1)
        if world > 1:
            torch.cuda.synchronize()
            b0 = time.perf_counter()
            nwd.broadcast_filter(conv.U, src=0)
            torch.cuda.synchronize()
            bcast_ms += (time.perf_counter() - b0) * 1e3
            bcast_bytes += conv.U.numel()
        x = ys[-1] if (chain and li > 0) else t["x"].to(dev)
        y = torch.empty(conv.out_shape(x.shape), dtype=x.dtype, device=dev)
        conv.workspace(*x.shape[:1], *x.shape[2:], path=paths[li])
        convs.append(conv)
        xs.append(x)
        ys.append(y)
        works.append(kernel_work(l, conv.info, args.math, paths[li]))
        del t
    torch.cuda.synchronize()

    # independent layers (not a chain) may run concurrently, each on its own stream with its own
    # workspace: one layer's kernel tails and transforms overlap another's
    lstreams = ([torch.cuda.Stream(device=dev) for _ in convs]
                if args.layer_streams and not chain and len(convs) > 1 else None)

    def step_seq():
        for conv, x, y, pth in zip(convs, xs, ys, paths):
            conv(x, y, path=pth)

    def step():
        if lstreams is None:
            step_seq()
            return
        cur = torch.cuda.current_stream()
        for st in lstreams:
            st.wait_stream(cur)
        for conv, x, y, pth, st in zip(convs, xs, ys, paths, lstreams):
            conv(x, y, path=pth, stream=st)
        for st in lstreams:
            cur.wait_stream(st)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = nw.launch_count()
    # the timed region: K steps between two events, no per-launch instrumentation inside
    with ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ
                      else dev_index) as clk:
        torch.cuda.synchronize()
        start.record(stream)
        for _ in range(args.steps):
            step()
        end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = nw.launch_count() - launches0
    ms = nwd.max_over_ranks(start.elapsed_time(end), dev)
    # per-layer breakdown + comparison paths (untimed against the headline)
    per_layer = []
    for l, conv, x, y in zip(layers_all, convs, xs, ys):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(10, args.steps)
        e0.record()
        pth = paths[len(per_layer)]
        for _ in range(reps):
            conv(x, y, path=pth)
        e1.record()
        torch.cuda.synchronize()
        lm = e0.elapsed_time(e1) / reps
        ent = {"layer": l.name, "path": pth, "ms": round(lm, 4),
               "tflops_direct_equiv": round(l.direct_flops() / (lm / 1e3) / 1e12, 2)}
        per_layer.append(attach_bounds(ent, layer_bounds(l, conv.info, args.math, peaks, pth),
                                       works[len(per_layer)], peaks, lm))

    # per-kernel times for the roofline: a second pass of K steps with every library launch
    # bracketed by CUDA events on its stream (nw_profile_begin / end), outside the timed region;
    # the layers run one after another here, so each launch's time is that kernel's alone (with
    # concurrent layer streams a launch's events would also span the other layers' kernels)
    _lib.profile_begin()
    for _ in range(args.steps):
        step_seq()
    torch.cuda.synchronize()
    prof = _lib.profile_end()
    # SURVEY 8(d) protocol: one step captured in a CUDA graph, replayed K times, 5 repetitions,
    # median reported beside the plain-stream value (launch overhead removed)
    graph = None
    try:
        g_ = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cap):
            step()                                 # warm the capture stream
        torch.cuda.current_stream().wait_stream(cap)
        torch.cuda.synchronize()
        with torch.cuda.graph(g_, stream=cap):
            step()
        reps = []
        for _ in range(5):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record()
            for _ in range(args.steps):
                g_.replay()
            b_.record()
            torch.cuda.synchronize()
            reps.append(a_.elapsed_time(b_) / args.steps)
        gms = nwd.max_over_ranks(statistics.median(reps), dev)
        graph = {"ms_per_step_median": round(gms, 4), "reps": [round(r, 4) for r in reps],
                 "value": round(sum(l.direct_flops() for l in layers_all) * world / (gms / 1e3) / 1e12, 3)}
        del g_
    except Exception as e:  # capture unsupported in this configuration: report why
        graph = {"unavailable": str(e)[:200]}
        torch.cuda.synchronize()
    ms_step = ms / args.steps
    flops_rank = sum(l.direct_flops() for l in layers_all)
    value = flops_rank * world / (ms_step / 1e3) / 1e12
    images = sum(l.N for l in layers_all) * world / len(layers_all) / (ms_step / 1e3)

    # step-level bounds: sum of the layers' bounds over the measured step
    step_roof = {k: {"bound_us": round(sum(e["roofline"][k]["bound_us"] for e in per_layer if k in e["roofline"]), 2)}
                 for k in ("r1", "r2", "r2_plan", "r3")}
    for k, v in step_roof.items():
        v["frac"] = round(v["bound_us"] / (ms_step * 1e3), 4)

    compare = {}
    if not args.no_compare and args.path == "nested" and not chain:
        # ola / direct: same kernels and math mode as the nested line.  direct_bf16: the direct
        # path in its cheapest mode that meets the same 5e-3 gate (plain bf16
        # passes for direct, not for OLA or nested -- tests/test_gpu_math_modes.py, R21)
        legs = [("ola", "ola", None), ("direct", "direct", None)]
        if args.math == "bf16x3":
            legs.append(("direct_bf16", "direct", nw.MATH_BF16))
        for name, path, lmath in legs:
            try:
                tot = 0.0
                flops_avail = 0
                lay = []
                for l, conv, x, y, pl in zip(layers_all, convs, xs, ys, per_layer):
                    if lmath is not None and l.depthwise:
                        lay.append({"layer": l.name, "unavailable": "plain bf16 is not built for depthwise layers"})
                        continue
                    flops_avail += l.direct_flops()
                    if lmath is not None:
                        conv = nw.NestedConv2d(conv.w, l.stride, l.pad, l.m_o, l.m_i, lmath, transposed=l.transposed,
                                               depthwise=l.depthwise,
                                               outer_taps=l.r_o, output_padding=l.output_padding,
                                               prelu_slopes=conv.prelu_slopes)
                    conv.workspace(x.shape[0], x.shape[2], x.shape[3], path)
                    for _ in range(3):   # warm-up (first-use allocations, clocks)
                        conv(x, y, path=path)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(10):
                        conv(x, y, path=path)
                    e1.record()
                    torch.cuda.synchronize()
                    lm = e0.elapsed_time(e1) / 10
                    tot += lm
                    lmath_name = "bf16" if lmath is not None else args.math
                    b = layer_bounds(l, conv.info, lmath_name, peaks, path)
                    wl = kernel_work(l, conv.info, lmath_name, path) if path == "direct" else None
                    if path == "ola":   # OLA pipeline: F(3,3) V and M per 3x3 tile, U per block
                        es = 2 if l.dtype == "bf16" else 4
                        nb = -(-conv.info["Kp"] // 3)
                        hq = -(-l.Ho // 2) if l.transposed else l.Ho
                        wq = -(-l.Wo // 2) if l.transposed else l.Wo
                        T3e = l.N * (-(-hq // 3) + nb - 1) * (-(-wq // 3) + nb - 1)
                        vb = 25 * T3e * conv.info["cin_e"] * 4
                        mb = 25 * T3e * conv.info["cout_e"] * 4
                        xb = l.N * l.Cin * l.H * l.W * es
                        yb = l.N * l.Cout * l.Ho * l.Wo * es
                        wl = {"input_transform": {"bytes": xb + vb}, "contraction_tc": {"bytes": vb + mb},
                              "output_transform": {"bytes": mb + yb}}
                    ent = {"layer": l.name, "ms": round(lm, 4), "nested_speedup": round(lm / pl["ms"], 3)}
                    attach_bounds(ent, b, wl, peaks, lm)
                    # the path's own bound: the slower of its contraction (passes issued) and its
                    # own pipeline bytes -- what "at its bound" means for this comparison path
                    own = ent["roofline"].get("r3", ent["roofline"]["r2_plan"])
                    ent["roofline_frac"] = own["frac"]
                    lay.append(ent)
                    del conv
                own_us = sum(e["roofline"].get("r3", e["roofline"]["r2_plan"])["bound_us"] for e in lay
                             if "roofline" in e)
                compare[name] = {"ms_per_step": round(tot, 4),
                                 "tflops_direct_equiv": round(flops_avail / (tot / 1e3) / 1e12, 2),
                                 "roofline_frac": round(own_us / (tot * 1e3), 4),
                                 "per_layer": lay}
                if lmath is not None:
                    compare[name]["math"] = "bf16"
                if args.workload == "table1" and path == "ola":
                    compare[name]["paper_nested_speedup_fpga"] = {
                        n: synth.TABLE1_PAPER_SPEEDUP[n] for n in WORKLOADS["table1"]}
            except nw.NWError as e:
                compare[name] = {"unavailable": str(e)}
            except RuntimeError as e:  # out of memory etc.
                compare[name] = {"unavailable": str(e)[:200]}

    # e2e: same metric through the C ABI with host buffers (copies inside the timed region)
    e2e = None
    if not args.no_e2e and chain:
        # network forward end to end: pinned host input -> device, the layer chain through the
        # C ABI, last output -> pinned host; copies inside the timed region
        hx0 = xs[0].cpu().pin_memory()
        hyl = torch.empty(ys[-1].shape, dtype=ys[-1].dtype).pin_memory()

        def e2e_chain():
            xs[0].copy_(hx0, non_blocking=True)
            step()
            hyl.copy_(ys[-1], non_blocking=True)

        for _ in range(2):
            e2e_chain()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ek = max(10, args.steps)
        s0.record(stream)
        for _ in range(ek):
            e2e_chain()
        s1.record(stream)
        torch.cuda.synchronize()
        ems = nwd.max_over_ranks(s0.elapsed_time(s1) / ek, dev)
        e2e = {"value": round(flops_rank * world / (ems / 1e3) / 1e12, 3), "unit": "TFLOP/s",
               "ms_per_step": round(ems, 3), "h2d_bytes_per_step": int(hx0.numel() * hx0.element_size()),
               "d2h_bytes_per_step": int(hyl.numel() * hyl.element_size())}
    elif not args.no_e2e:
        hx = [x.cpu().pin_memory() for x in xs]
        hy = [torch.empty(y.shape, dtype=y.dtype).pin_memory() for y in ys]
        wss = []
        for conv, x in zip(convs, xs):
            nbytes = conv.plan.workspace_size(x.shape[0], x.shape[2], x.shape[3], "host")
            wss.append(nbytes)
        # the sweep's layers are independent: each runs on its own stream with its own workspace,
        # so one layer's copies in overlap another's copies out (PCIe carries both directions)
        ws_l = [torch.empty(n, dtype=torch.uint8, device=dev) for n in wss]
        streams = [torch.cuda.Stream(device=dev) for _ in convs]

        def e2e_step():
            for conv, x, hxx, hyy, wsx, st in zip(convs, xs, hx, hy, ws_l, streams):
                conv.plan.forward_host(hxx, conv.U, hyy, x.shape[0], x.shape[2], x.shape[3], wsx, wsx.numel(),
                                       stream=st)

        for st in streams:
            st.wait_stream(stream)
        for _ in range(3):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ek = max(10, args.steps)
        s0.record(stream)
        for st in streams:
            st.wait_stream(stream)
        for _ in range(ek):
            e2e_step()
        for st in streams:
            stream.wait_stream(st)
        s1.record(stream)
        torch.cuda.synchronize()
        ems = nwd.max_over_ranks(s0.elapsed_time(s1) / ek, dev)
        e2e = {"value": round(flops_rank * world / (ems / 1e3) / 1e12, 3), "unit": "TFLOP/s",
               "ms_per_step": round(ems, 3),
               "h2d_bytes_per_step": int(sum(x.numel() * x.element_size() for x in xs)),
               "d2h_bytes_per_step": int(sum(y.numel() * y.element_size() for y in ys))}

    roof = roofline(prof, works, args.math, peaks, args.steps, layers_all)

    # multi-GPU verification (outside every timed region): each rank hashes its outputs; rank 0
    # regenerates every rank's seeded inputs, runs them through its own U (the broadcast's
    # source) and must reproduce each rank's hash, i.e. the sharded run equals a 1-rank run
    # bit for bit
    multi = None
    if world > 1:
        import hashlib

        def digest(tensors):
            h = hashlib.sha256()
            for y in tensors:
                h.update(y.contiguous().view(torch.uint8).cpu().numpy().tobytes())
            return h.hexdigest()

        step()
        torch.cuda.synchronize()
        mine = digest(ys)
        hashes = [None] * world
        dist.all_gather_object(hashes, mine)
        ok = True
        if rank == 0:
            for r in range(world):
                if chain:
                    xr = synth.make_inputs(layers_all[0].with_(seed=layers_all[0].seed + 1000 * r))["x"] if r \
                        else synth.make_inputs(layers_all[0])["x"]
                    xs[0].copy_(xr.to(dev))
                else:
                    for l, x in zip(layers_all, xs):
                        xr = synth.make_inputs(l.with_(seed=l.seed + 1000 * r))["x"] if r else synth.make_inputs(l)["x"]
                        x.copy_(xr.to(dev))
                step()
                torch.cuda.synchronize()
                ok = ok and digest(ys) == hashes[r]
        flag = torch.tensor([1 if ok else 0], device=dev)
        dist.broadcast(flag, src=0)
        multi = {"bit_identical_to_1_rank": bool(flag.item()), "ranks_checked": world,
                 "collectives": "one NCCL broadcast of U per layer from rank 0 (outside the timed region); "
                                "no data-path collective (batch-sharded)",
                 "u_broadcast_bytes": bcast_bytes, "u_broadcast_ms": round(bcast_ms, 3),
                 "filter_transform_ranks": [0]}
        if not ok:
            print("bench.py: multi-GPU outputs differ from the 1-rank recomputation", file=sys.stderr)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        f, t, n, _ = oracle_sample_time(layers_all, target_s=10.0)
        cpu = {"value": round(f / t / 1e12, 5), "unit": "TFLOP/s", "cores": cores_used(), "kind": "oracle",
               "cpu_model": cpu_model(),
               "sample": f"oracle.direct FP64 (Eq. 2.1) on {n} image(s) of each layer of the workload "
                         f"({f / 1e9:.1f} GFLOP direct-equivalent in {t:.1f} s)"}

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": {"bf16x3": "bf16x3", "fp32": "f32", "bf16": "bf16"}[args.math],
            "data": "synthetic (seeded; BASELINE distributions, DESIGN.md input recipe)",
            "config": {"workload": WORKLOAD_DESC[args.workload], "layers": [l.name for l in layers_all],
                       "nesting": [f"F({c.info['m_outer']},{c.info['r_outer']})(x)F({c.info['m_inner']},3)"
                                   for c in convs],
                       "path": paths if chain else args.path, "math": args.math,
                       "images_per_rank": layers_all[0].N,
                       "parallelism": f"dp{world}: batch-sharded, one process per GPU, U broadcast once"
                                      if world > 1 else "1 GPU",
                       "l2": "no flush: x (>=134 MB) and V/M (>1 GB per layer) exceed the 126 MB L2",
                       "timing": "K steps between CUDA events on the launching stream, no per-launch "
                                 "instrumentation inside; per-kernel times (roofline, kernel_ms) from a "
                                 "second instrumented pass; 'graph' = one step as a CUDA graph, median of 5",
                       "step": "input transform + contraction + output transform per layer (nw_conv_forward)",
                       "concurrency": ("the workload's independent layers run concurrently, one stream and "
                                       "workspace each (per_layer times are each layer alone)")
                                      if lstreams is not None else "layers in sequence on one stream"},
            "images_per_s": round(images, 1),
            "per_layer": per_layer,
            "filter_transform_ms": round(filt_ms, 4),
            "multi_gpu": multi,
            "compare": compare,
            "roofline": roof,
            "roofline_step": step_roof,
            "graph": graph,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "kernel_ms": {k: {"launches": v[0], "ms_total": round(v[1], 4)} for k, v in prof.items()},
            "clocks": clk.summary(),
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if multi is not None and not multi["bit_identical_to_1_rank"]:
        sys.exit(3)


def reference_arm(args, layers, world, rank):
    """--impl reference: the CPU oracle (FP64 direct conv) as it stands, bounded sample per step."""
    if rank != 0:
        return
    from oracle import direct
    inputs = [synth.make_inputs(l.with_(N=1)) for l in layers]
    arrays = [(t["x"].double().numpy(), t["w"].double().numpy()) for t in inputs]

    def step():
        for l, (x, w) in zip(layers, arrays):
            if l.transposed:
                direct.conv_transpose2d(x, w, l.stride, l.pad, l.output_padding)
            elif l.depthwise:
                direct.conv2d_depthwise(x, w, l.stride, l.pad)
            else:
                direct.conv2d(x, w, l.stride, l.pad)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    flops = sum(l.with_(N=1).direct_flops() for l in layers)
    v = flops / dt / 1e12
    out = {"metric": METRIC, "value": round(v, 5), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 2), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": WORKLOAD_DESC[args.workload], "layers": [l.name for l in layers],
                      "sample": "1 image of each layer per step"},
           "cpu_baseline": {"value": round(v, 5), "unit": "TFLOP/s", "cores": cores_used(), "kind": "oracle",
                            "cpu_model": cpu_model(),
                            "sample": "oracle.direct FP64 (Eq. 2.1), 1 image of each layer per step"},
           "e2e": {"value": round(v, 5), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
