#!/usr/bin/env python
"""Instruction mix (+ stall samples) of one kernel from an ncu report: python tools/sass_mix.py rep.ncu-rep [N]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h = rows[1]
data = rows[2:]
ii, si, ws = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ii] or 0) for r in data)
ops, st = collections.Counter(), collections.Counter()
for r in data:
    toks = r[si].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    ops[op] += int(r[ii] or 0)
    st[op] += int(r[ws] or 0)
tst = sum(st.values()) or 1
print("total warp instructions", tot)
for op, c in ops.most_common(top):
    print(f"{op:10s} {c:12d} {100 * c / tot:5.1f}%   stall samples {100 * st[op] / tst:5.1f}%")
