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
    "table1": "paper Table I conv2d shapes (P:154-160): SRCNN 9x9 64<-1, 5x5 32<-64, 5x5 1<-32, 256x256, N=8, fp32",
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
    if info.get("single_kernel"):
        # one input channel: transform, pointwise product and output transform in one kernel;
        # HBM traffic is x, U and y only (the kernel is bound by its CUDA-core transforms)
        return {"fused_c1": {"bytes": x_b + u_b + y_b, "flops": 0},
                "filter_transform": {"bytes": u_b, "flops": 0}}
    return {
        "input_transform": {"bytes": x_b + v_b, "flops": 0},
        "contraction_tc": {"bytes": v_b + u_b + m_b, "flops": flops * passes},
        "contraction_fp32_simt": {"bytes": v_b + u_b + m_b, "flops": flops},
        "output_transform": {"bytes": m_b + y_b, "flops": 0},
        "filter_transform": {"bytes": u_b, "flops": 0},
    }


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
    return {"kernel": kind, "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
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
                else:
                    direct.conv2d(x, w, l.stride, l.pad)
            flops += n_img * l.with_(N=1).direct_flops()
        return flops, time.perf_counter() - t0

    f1, t1 = run(1)
    n = max(1, min(max_images or 64, int(target_s / max(t1, 1e-3))))
    if n > 1:
        f1, t1 = run(n)
    return f1, t1, n, np.__version__


def cores_used():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ----------------------------------------------------------------------------
def main():
    args = parse()
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

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    math = {"bf16x3": nw.MATH_BF16X3, "fp32": nw.MATH_FP32_SIMT, "bf16": nw.MATH_BF16}[args.math]
    peaks = load_peaks()
    stream = torch.cuda.current_stream()

    chain = args.workload in CHAINS
    paths = [("direct" if (chain and l.K <= 3) else args.path) for l in layers_all]
    convs, xs, ys, works = [], [], [], []
    filt_ms = 0.0
    for li, l in enumerate(layers_all):
        t = synth.make_inputs(l.with_(seed=l.seed + 1000 * rank)) if rank else synth.make_inputs(l)
        if chain and li > 0:
            t["x"] = None                                   # consumes the previous layer's output
        w = synth.make_inputs(l, x=False)["w"].to(dev)     # same weights on every rank
        slopes = torch.full((l.Cout,), synth.PRELU_SLOPE, device=dev) if l.prelu else None
        conv = nw.NestedConv2d(w, l.stride, l.pad, l.m_o, l.m_i, math, transposed=l.transposed, outer_taps=l.r_o,
                               output_padding=l.output_padding, prelu_slopes=slopes)
        # filter transform once on rank 0 (timed separately), broadcast U over NCCL
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        conv.transform_filter()
        e1.record()
        torch.cuda.synchronize()
        filt_ms += e0.elapsed_time(e1)
        nwd.broadcast_filter(conv.U, src=0)   # the one collective: U from rank 0 (NCCL / NVLink)
        x = ys[-1] if (chain and li > 0) else t["x"].to(dev)
        y = torch.empty(conv.out_shape(x.shape), dtype=x.dtype, device=dev)
        conv.workspace(*x.shape[:1], *x.shape[2:], path=paths[li])
        convs.append(conv)
        xs.append(x)
        ys.append(y)
        works.append(kernel_work(l, conv.info, args.math, paths[li]))
        del t
    torch.cuda.synchronize()

    def step():
        for conv, x, y, pth in zip(convs, xs, ys, paths):
            conv(x, y, path=pth)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = nw.launch_count()
    with ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ
                      else local) as clk:
        _lib.profile_begin()
        torch.cuda.synchronize()
        start.record(stream)
        for _ in range(args.steps):
            step()
        end.record(stream)
        torch.cuda.synchronize()
        prof = _lib.profile_end()
    if world > 1:
        dist.barrier()
    launches = nw.launch_count() - launches0
    ms = nwd.max_over_ranks(start.elapsed_time(end), dev)
    ms_step = ms / args.steps
    flops_rank = sum(l.direct_flops() for l in layers_all)
    value = flops_rank * world / (ms_step / 1e3) / 1e12
    images = sum(l.N for l in layers_all) * world / len(layers_all) / (ms_step / 1e3)

    # per-layer breakdown + comparison paths (untimed against the headline)
    per_layer = []
    for l, conv, x, y in zip(layers_all, convs, xs, ys):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(3, args.steps // 2)
        e0.record()
        pth = paths[len(per_layer)]
        for _ in range(reps):
            conv(x, y, path=pth)
        e1.record()
        torch.cuda.synchronize()
        lm = e0.elapsed_time(e1) / reps
        per_layer.append({"layer": l.name, "path": pth, "ms": round(lm, 4),
                          "tflops_direct_equiv": round(l.direct_flops() / (lm / 1e3) / 1e12, 2)})

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
                lay = []
                for l, conv, x, y, pl in zip(layers_all, convs, xs, ys, per_layer):
                    if lmath is not None:
                        conv = nw.NestedConv2d(conv.w, l.stride, l.pad, l.m_o, l.m_i, lmath, transposed=l.transposed,
                                               outer_taps=l.r_o, output_padding=l.output_padding,
                                               prelu_slopes=conv.prelu_slopes)
                    conv.workspace(x.shape[0], x.shape[2], x.shape[3], path)
                    conv(x, y, path=path)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(3):
                        conv(x, y, path=path)
                    e1.record()
                    torch.cuda.synchronize()
                    lm = e0.elapsed_time(e1) / 3
                    tot += lm
                    lay.append({"layer": l.name, "ms": round(lm, 4), "nested_speedup": round(lm / pl["ms"], 3)})
                    del conv
                compare[name] = {"ms_per_step": round(tot, 4),
                                 "tflops_direct_equiv": round(flops_rank / (tot / 1e3) / 1e12, 2),
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

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        f, t, n, _ = oracle_sample_time(layers_all, target_s=10.0)
        cpu = {"value": round(f / t / 1e12, 5), "unit": "TFLOP/s", "cores": cores_used(), "kind": "oracle",
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
                       "l2": "no flush: x (>=134 MB) and V/M (>1 GB per layer) exceed the 126 MB L2",
                       "step": "input transform + contraction + output transform per layer (nw_conv_forward)"},
            "images_per_s": round(images, 1),
            "per_layer": per_layer,
            "filter_transform_ms": round(filt_ms, 4),
            "compare": compare,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "kernel_ms": {k: {"launches": v[0], "ms_total": round(v[1], 4)} for k, v in prof.items()},
            "clocks": clk.summary(),
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


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
                            "sample": "oracle.direct FP64 (Eq. 2.1), 1 image of each layer per step"},
           "e2e": {"value": round(v, 5), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
