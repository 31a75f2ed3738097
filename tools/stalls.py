#!/usr/bin/env python3
"""Print throughput, hit rates and warp-stall samples of each launch in an ncu report."""
import csv
import io
import subprocess
import sys

txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(l for l in txt.splitlines() if l.startswith('"')))))
h, u = rows[0], rows[1]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'launch__registers_per_thread',
        'smsp__inst_executed.sum']
brief = "--brief" in sys.argv


def val(d, k):
    try:
        return float(d[h.index(k)].replace(',', ''))
    except (ValueError, IndexError):
        return 0.0


if brief:
    print("kernel | us | DRAM MB | DRAM% | L1% | L2% | occ% | top stalls")
for d in rows[2:]:
    if brief:
        import re
        nm = re.sub(r"\(.*", "", d[h.index("Kernel Name")]).replace("void ", "")
        st = []
        for i, k in enumerate(h):
            if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
                try:
                    st.append((float(d[i].replace(',', '')), k.split('stalled_')[1]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        dur = val(d, 'gpu__time_duration.sum')
        unit = u[h.index('gpu__time_duration.sum')]
        us = dur * {'ms': 1e3, 'us': 1.0, 'ns': 1e-3, 'msecond': 1e3, 'usecond': 1.0,
                    'nsecond': 1e-3}.get(unit, 1.0)
        rd = val(d, 'dram__bytes_read.sum') * {'Gbyte': 1e3, 'Mbyte': 1.0, 'Kbyte': 1e-3,
                                               'byte': 1e-6}.get(u[h.index('dram__bytes_read.sum')], 1)
        print(f"{nm[:50]} | {us:.1f} | {rd:.1f} | "
              f"{val(d, 'dram__throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | "
              f"{val(d, 'l1tex__throughput.avg.pct_of_peak_sustained_active'):.0f} | "
              f"{val(d, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | "
              f"{val(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} | "
              + ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in sorted(st, reverse=True)[:3]))
        continue
    print("==", d[h.index("Kernel Name")][:90])
    for k in keys:
        if k in h:
            print(f"  {k} = {d[h.index(k)]} {u[h.index(k)]}")
    st = []
    for i, k in enumerate(h):
        if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
            try:
                st.append((float(d[i].replace(',', '')), k.split('stalled_')[1]))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("  stalls:", ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in sorted(st, reverse=True)[:7]))
