#!/usr/bin/env python
"""Group the SASS of an ncu source page (--page source --csv --print-source
sass) into basic-block-frequency regions and print each region's share of
warp stall samples, with its instruction mix.  Usage: ncu_regions.py <csv> [min_share]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
si = hdr.index("Source")
wi = hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
tot = sum(int(r[wi]) for r in data)
groups = []
for i, r in enumerate(data):
    n = int(r[ei]) if r[ei].isdigit() else 0
    s = int(r[wi])
    op = r[si].strip().split()
    op = op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "")
    if groups and groups[-1][0] == n:
        groups[-1][1] += s
        groups[-1][2] += 1
        groups[-1][3].append(op)
    else:
        groups.append([n, s, 1, [op], i])
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.003
for n, s, c, ops, i in groups:
    if s / tot > thr:
        top = ", ".join(f"{k}x{v}" for k, v in Counter(ops).most_common(6))
        print(f"sass line {i:5d} exec={n:11d} instrs={c:4d} stall-share={s / tot:.3f}  {top}")
