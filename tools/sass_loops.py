#!/usr/bin/env python3
"""Instruction and stall share of every loop (backward branch) of one kernel in
`ncu --page source --csv --print-source sass` output (first launch only).
usage: sass_loops.py <csv> [topN]"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
hdr = None
data = []
for r in rows:
    if r and r[0] == "Kernel Name" and data:
        break
    if len(r) > 3 and r[0] == "Address":
        hdr = r
        continue
    if hdr and r and r[0].startswith("0x"):
        ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        data.append((int(r[0], 16), r[1].strip(), float(r[ie] or 0), float(r[ss] or 0)))
tot = sum(d[2] for d in data) or 1
tots = sum(d[3] for d in data) or 1
addr = {d[0]: i for i, d in enumerate(data)}
loops = []
for i, d in enumerate(data):
    m = re.search(r"BRA (0x[0-9a-f]+)", d[1])
    if m:
        t = int(m.group(1), 16)
        if t < d[0] and t in addr:
            body = data[addr[t]:i + 1]
            loops.append((sum(x[2] for x in body) / tot, sum(x[3] for x in body) / tots, len(body),
                          hex(t), body[0][1][:50]))
loops.sort(key=lambda l: -l[0])
print(f"total instructions {tot:.3e}, stall samples {tots:.0f}")
for l in loops[:top]:
    print("inst %5.1f%%  stall %5.1f%%  len %4d  at %s: %s" % (100 * l[0], 100 * l[1], l[2], l[3], l[4]))
