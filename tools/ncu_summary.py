#!/usr/bin/env python
"""Summarise ncu output into profiles/ (runs here, on the CPU box).

    python tools/ncu_summary.py --tag r1a --launches gpurun_out/launches_r1a.csv \
        --rep gpurun_out/prof_r1a_c2k9_input_transform.ncu-rep ... --bench gpurun_out/bench_r1a.json

Writes profiles/<tag>_launches.csv (per-kernel share of the launch list),
profiles/<tag>_ncu.md (key --set full metrics per captured kernel) and, when
--bench is given, copies the bench JSON line to profiles/<tag>_bench.json.
Also updates profiles/traffic.json with dram read+write bytes per launch,
keyed "<kind>:<math>:<layer>:m<m_outer>" (the layer tools/prof_layer.py ran; the
report file name carries it: prof_<tag>_<layer>_<kernel>.ncu-rep), which
bench.py averages over the workload's layers as roofline.traffic.
"""
from __future__ import annotations

import argparse
import collections
import csv
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
STALLS = re.compile(r"^smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$")
KIND = {"input_transform": "input_transform", "contraction": "contraction_tc",
        "output_transform": "output_transform", "gemm_simt": "contraction_fp32_simt",
        "filter_transform": "filter_transform", "ola": "ola", "direct": "direct", "fused_c1": "fused_c1",
        "depthwise_product": "depthwise_product"}


def short(name: str) -> str:
    n = name.split("(")[0]
    n = re.sub(r"^void ", "", n)
    return n.split("<")[0]


def launches(path: str, tag: str) -> str:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        a = agg.setdefault(short(r[ki]), [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(a[1] for a in agg.values())
    out = os.path.join(PROF, f"{tag}_launches.csv")
    with open(out, "w") as f:
        f.write("kernel,launches,total_us,mean_us,share\n")
        for k, (n, t) in agg.items():
            f.write(f"{k},{n},{t / 1e3:.1f},{t / 1e3 / n:.1f},{t / tot:.4f}\n")
    return out


def rep_metrics(path: str):
    if path.endswith(".csv"):   # raw page exported on the GPU box (ncu -i rep --page raw --csv)
        txt = open(path).read()
    else:
        txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        d = {"kernel": short(v[h.index("Kernel Name")])}
        for i, n in enumerate(h):
            if n in KEYS:
                d[n] = (v[i], units[i])
            m = STALLS.match(n)
            if m:
                try:
                    d.setdefault("stalls", {})[m.group(1)] = float(v[i])
                except ValueError:
                    pass
        out.append(d)
    return out


def to_bytes(val: str, unit: str) -> float:
    s = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    return float(val.replace(",", "")) * s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--bench")
    ap.add_argument("--math", default="bf16x3")
    ap.add_argument("--m-outer", type=int, default=4, help="outer kernel of the profiled plan")
    ap.add_argument("--note", default="")
    ap.add_argument("--dram", nargs="*", default=[],
                    help="lightweight ncu CSVs dram_<tag>_<layer>.csv (gpu__time_duration, dram bytes)")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    md = [f"# ncu summary {a.tag}", ""]
    if a.note:
        md += [a.note, ""]
    if a.launches:
        p = launches(a.launches, a.tag)
        md += [f"Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, cold-cache, "
               f"serialised; compare shares): `{os.path.relpath(p, ROOT)}`", "", "```",
               open(p).read().strip(), "```", ""]
    tfile = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(tfile)) if os.path.exists(tfile) else {}
    for rep in a.rep:
        for d in rep_metrics(rep):
            md += [f"## {d['kernel']} (`{os.path.basename(rep)}`)", "", "| metric | value |", "|---|---|"]
            for k in KEYS:
                if k in d:
                    md.append(f"| {k} | {d[k][0]} {d[k][1]} |")
            st = sorted(d.get("stalls", {}).items(), key=lambda kv: -kv[1])[:6]
            md.append("| top stalls (warps per issue) | " + ", ".join(f"{k} {v:.2f}" for k, v in st) + " |")
            md.append("")
            if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d:
                b = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
                base = os.path.basename(rep).split(".")[0]          # prof_<tag>_<layer>_<kernel>
                rest = base[len(f"prof_{a.tag}_"):] if base.startswith(f"prof_{a.tag}_") else base
                layer = "?"
                for kk in ("_input_transform", "_output_transform", "_contraction", "_depthwise", "_fused_c1"):
                    if rest.endswith(kk):
                        layer = rest[: -len(kk)]
                for key, kind in KIND.items():
                    if key in d["kernel"]:
                        traffic[f"{kind}:{a.math}:{layer}:m{a.m_outer}"] = int(b)
    for path in a.dram:
        layer = os.path.basename(path)[:-4].split("_")[-1]
        rows = [r for r in csv.reader(open(path)) if len(r) > 10]
        h = rows[0]
        ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
        ids = h.index("ID")
        per = collections.defaultdict(lambda: collections.defaultdict(float))
        for r in rows[1:]:
            if r[mi].startswith("dram__bytes"):
                per[(short(r[ki]), r[ids])]["bytes"] += to_bytes(r[vi], r[ui] or "byte")
            elif r[mi] == "gpu__time_duration.sum":
                per[(short(r[ki]), r[ids])]["ns"] += float(r[vi].replace(",", ""))
        agg = collections.defaultdict(list)
        for (kname, _), d in per.items():
            agg[kname].append(d)
        md += [f"## dram bytes per launch, {layer} (`{os.path.basename(path)}`)", "",
               "| kernel | launches | dram read+write per launch | time per launch |", "|---|---|---|---|"]
        for kname, lst in agg.items():
            b = sum(d["bytes"] for d in lst) / len(lst)
            t = sum(d["ns"] for d in lst) / len(lst)
            md.append(f"| {kname} | {len(lst)} | {b / 1e6:.1f} MB | {t / 1e3:.1f} us |")
            for key, kind in KIND.items():
                if key in kname:
                    traffic[f"{kind}:{a.math}:{layer}:m{a.m_outer}"] = int(b)
        md.append("")
    json.dump(traffic, open(tfile, "w"), indent=1, sort_keys=True)
    if a.bench:
        line = [l for l in open(a.bench).read().splitlines() if l.startswith("{")][-1]
        open(os.path.join(PROF, f"{a.tag}_bench.json"), "w").write(line + "\n")
    open(os.path.join(PROF, f"{a.tag}_ncu.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
