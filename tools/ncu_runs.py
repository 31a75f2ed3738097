#!/usr/bin/env python3
"""Sum dram__bytes_read/write and gpu__time_duration over every kernel of
one ncu --csv launch list per bench line (tools/ncu_lines.sh) and record
them in profiles/ncu_summary.json as "run:<line>".
usage: ncu_runs.py <line>.csv ..."""
import csv
import io
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1,
         "s": 1, "nsecond": 1e-9}
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                    "ncu_summary.json")
summ = json.load(open(path)) if os.path.exists(path) else {}
for f in sys.argv[1:]:
    name = os.path.basename(f)[:-4]
    txt = open(f, errors="replace").read()
    rows = list(csv.reader(io.StringIO("\n".join(l for l in txt.splitlines() if l.startswith('"')))))
    if len(rows) < 2:
        print(f"{name}: no kernels captured")
        continue
    h = rows[0]
    ik, iname, iunit, ival = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Unit"),
                              h.index("Metric Value"))
    imet = h.index("Metric Name")
    tot = {"dram__bytes_read.sum": 0.0, "dram__bytes_write.sum": 0.0,
           "gpu__time_duration.sum": 0.0}
    kernels = {}
    ids = set()
    for r in rows[1:]:
        if len(r) <= ival or r[imet] not in tot:
            continue
        v = float(r[ival].replace(",", "")) * SCALE.get(r[iunit], 1)
        tot[r[imet]] += v
        ids.add(r[ik])
        k = r[iname].split("(")[0].split("::")[-1]
        kernels.setdefault(k, [0.0, 0.0])
        if r[imet].startswith("dram"):
            kernels[k][0] += v
        else:
            kernels[k][1] += v
    dram = tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]
    top = sorted(kernels.items(), key=lambda kv: -kv[1][1])[:6]
    summ["run:" + name] = {
        "dram_bytes_per_run": dram, "kernel_time_s_serialised": tot["gpu__time_duration.sum"],
        "launches": len(ids),
        "top_kernels": {k: {"dram_bytes": v[0], "time_s": v[1]} for k, v in top},
        "source": os.path.basename(f),
        "note": "one steady run under ncu (NVTX range 'steady'), kernels serialised and "
                "cold-cache: the DRAM bytes are the run's traffic, the times are not bench times"}
    print(f"{name}: {len(ids)} launches, DRAM {dram / 1e9:.3f} GB, serialised kernel time "
          f"{tot['gpu__time_duration.sum'] * 1e3:.2f} ms; top: " +
          ", ".join(f"{k} {v[1] * 1e3:.2f} ms/{v[0] / 1e9:.2f} GB" for k, v in top[:3]))
json.dump(summ, open(path, "w"), indent=1, sort_keys=True)
