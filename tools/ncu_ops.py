#!/usr/bin/env python
"""Dynamic SASS opcode histogram (and optionally the hot listing) of an ncu report.

    python tools/ncu_ops.py report.ncu-rep [--hot N]
"""
import argparse
import collections
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--hot", type=int, default=0, help="print instructions executed >= N times")
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ie, src, smp = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ie] or 0) for r in data)
c, s = collections.Counter(), collections.Counter()
for r in data:
    t = r[src].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    c[op] += int(r[ie] or 0)
    s[op] += int(r[smp] or 0)
print("total warp instructions", tot)
for op, n in c.most_common(24):
    print(f"{op:10s} {n:11d} {100 * n / tot:5.1f}%  stall-samples {s[op]}")
if a.hot:
    for i, r in enumerate(data):
        if int(r[ie] or 0) >= a.hot:
            print(i, r[ie], r[smp], r[src].strip()[:100])
