#!/usr/bin/env python3
"""Summarise ncu output brought back under gpurun_out/ into profiles/.

  tools/ncu_summary.py launches <launches.csv> <out.md>
      per-kernel launch count, total/mean device time and share of the
      serialised launch list (ncu --metrics gpu__time_duration.sum).
  tools/ncu_summary.py full <prof.ncu-rep> <out.md> [--json profiles/ncu_summary.json --key NAME]
      key counters of each captured launch (--set full): duration, DRAM
      bytes, DRAM/L2 throughput, L2 hit rate, occupancy, warp efficiency.
"""

from __future__ import annotations

import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import OrderedDict, defaultdict


def _short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)          # drop the argument list
    name = name.replace("void ", "").replace("<unnamed>::", "")
    name = re.sub(r"\(anonymous namespace\)::", "", name)
    return name.strip()


def _rows(text: str):
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def launches(path: str, out: str) -> None:
    rows = _rows(open(path).read())
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = _short(r[ki])
        tot[k] += float(r[vi].replace(",", ""))
        cnt[k] += 1
    all_ns = sum(tot.values()) or 1.0
    with open(out, "w") as f:
        f.write(f"# ncu launch list: {os.path.basename(path)}\n\n")
        f.write("Serialised, cold-cache per-launch times (compare shares, not absolutes).\n\n")
        f.write("| kernel | launches | total ms | mean us | share |\n|---|---|---|---|---|\n")
        for k in sorted(tot, key=lambda x: -tot[x]):
            f.write(f"| `{k}` | {cnt[k]} | {tot[k] / 1e6:.3f} | {tot[k] / cnt[k] / 1e3:.1f} | "
                    f"{100 * tot[k] / all_ns:.1f}% |\n")
    print(open(out).read())


FULL_METRICS = OrderedDict([
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("lts__t_sectors.sum", "l2_sectors"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads_per_inst"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_insts"),
])


def _to_bytes(val: str, unit: str) -> float:
    v = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
             "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(unit, 1)
    return v * scale


def full(rep: str, out: str, json_path: str | None = None, key: str | None = None) -> None:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = _rows(txt)
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    res = []
    for r in data:
        d = {"kernel": _short(r[ki])}
        for m, nm in FULL_METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    d[nm] = _to_bytes(r[i], units[i])
                except ValueError:
                    d[nm] = r[i]
        res.append(d)
    with open(out, "w") as f:
        f.write(f"# ncu --set full: {os.path.basename(rep)}\n\n")
        f.write("| kernel | dur us | DRAM rd MB | DRAM wr MB | DRAM % | L2 hit % | SM % | "
                "occ % | thr/inst | regs | grid |\n|---|---|---|---|---|---|---|---|---|---|---|\n")
        for d in res:
            f.write("| `{}` | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | "
                    "{:.1f} | {:.0f} | {:.0f} |\n".format(
                        d["kernel"], d.get("duration", 0) * 1e6, d.get("dram_read", 0) / 1e6,
                        d.get("dram_write", 0) / 1e6, d.get("dram_pct", 0),
                        d.get("l2_hit_pct", 0), d.get("sm_pct", 0),
                        d.get("occupancy_pct", 0), d.get("threads_per_inst", 0),
                        d.get("regs", 0), d.get("grid", 0)))
    print(open(out).read())
    if json_path and key == "pr_iteration" and res:
        # one PR iteration = one launch each of k_pr_units, k_pr_fix, k_pr_epi
        try:
            cur = json.load(open(json_path))
        except Exception:
            cur = {}
        tot = sum(d.get("dram_read", 0) + d.get("dram_write", 0) for d in res)
        names = sorted({d["kernel"] for d in res})
        cur[key] = {"dram_bytes_per_launch": tot * len(names) / len(res),
                    "kernels": names, "source": os.path.basename(rep),
                    "note": "sum of the iteration's kernels' dram__bytes_read+write"}
        json.dump(cur, open(json_path, "w"), indent=1)
        return
    if json_path and key and res:
        try:
            cur = json.load(open(json_path))
        except Exception:
            cur = {}
        n = len(res)
        cur[key] = {
            "dram_bytes_per_launch": sum(d.get("dram_read", 0) + d.get("dram_write", 0)
                                         for d in res) / n,
            "duration_s_per_launch": sum(d.get("duration", 0) for d in res) / n,
            "l2_hit_pct": sum(d.get("l2_hit_pct", 0) for d in res) / n,
            "launches_captured": n,
            "source": os.path.basename(rep),
        }
        json.dump(cur, open(json_path, "w"), indent=1)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif mode == "full":
        jp = key = None
        if "--json" in sys.argv:
            jp = sys.argv[sys.argv.index("--json") + 1]
        if "--key" in sys.argv:
            key = sys.argv[sys.argv.index("--key") + 1]
        full(sys.argv[2], sys.argv[3], jp, key)
