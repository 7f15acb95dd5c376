#!/usr/bin/env python
"""Per-CUDA-source-line totals (instructions executed, stall samples) from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass` (dev tool).

    python tools/ncu_lines.py dump.csv [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ins = collections.Counter()
stall = collections.Counter()
src = {}
fname = ""
line = None
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ei = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= si:
        continue
    if r[0]:
        line = (fname, int(r[0]))
        src[line] = r[1].strip()
        continue
    if line is None:
        continue
    num = lambda v: float(v) if v not in ("", "-") else 0.0
    ins[line] += int(num(r[ei]))
    stall[line] += int(num(r[si]))
ti, ts = sum(ins.values()) or 1, sum(stall.values()) or 1
print(f"total inst {ti}  stall samples {ts}")
for k in sorted(set(ins) | set(stall), key=lambda k: -(ins[k] / ti + stall[k] / ts))[:top]:
    print(f"{ins[k]/ti:6.3f} inst {stall[k]/ts:6.3f} stall  {k[0]}:{k[1]:<4d} {src[k][:90]}")
