#!/usr/bin/env python
"""Aggregate an ncu --page source --csv (SASS view) export: stall samples and executed warp
instructions per opcode, and the hottest instructions.  python tools/sass_hot.py <source.csv> [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    op = r[ix["Source"]].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    data.append((r[ix["Address"]], r[ix["Source"]].strip(), int(r[ix["Warp Stall Sampling (All Samples)"]] or 0),
                 int(r[ix["Warp Stall Sampling (Not-issued Samples)"]] or 0), int(r[ix["Instructions Executed"]] or 0),
                 o.split(".")[0]))
tot_s = sum(d[2] for d in data)
tot_i = sum(d[4] for d in data)
by = collections.defaultdict(lambda: [0, 0])
for d in data:
    by[d[5]][0] += d[2]
    by[d[5]][1] += d[4]
print(f"total samples {tot_s}, warp instructions {tot_i}")
for k, v in sorted(by.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"  {k:10s} samples {v[0] / tot_s:6.1%}  instr {v[1] / tot_i:6.1%}")
print("hottest:")
for i, d in enumerate(sorted(data, key=lambda d: -d[2])[:top]):
    print(f"  {d[0][-5:]} {d[2] / tot_s:6.2%} (not issued {d[3] / tot_s:6.2%}) n={d[4]:9d}  {d[1][:80]}")
