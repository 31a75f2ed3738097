#!/usr/bin/env python3
"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`.
usage: hot_sass.py <csv> [topN]  (the csv may hold several launches of one kernel)"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
agg = defaultdict(float)
src = {}
order = []
hdr = None
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) < 3:
        continue
    try:
        s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    key = r[0]
    if key not in src:
        order.append(key)
    src[key] = r[1]
    agg[key] += s
tot = sum(agg.values()) or 1
for k in sorted(agg, key=lambda x: -agg[x])[:top]:
    print(f"{100 * agg[k] / tot:5.1f}%  {k}  {src[k][:110]}")
