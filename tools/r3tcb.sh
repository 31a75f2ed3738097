#!/bin/bash
# TC upper-CSR build phases on RMAT-24 (trace + ncu launch list of the first call).
OUT=gpurun_out/r3tcb; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
SP_TC_TRACE=1 python tools/run_algo.py tc_rmat24 2 > $OUT/trace.txt 2>&1
SP_TC_TRACE=1 python tools/run_algo.py tc 2 >> $OUT/trace.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv python tools/run_algo.py tc_rmat24 1 > $OUT/ncu.log 2>&1
cat $OUT/trace.txt
python - $OUT/launches.csv <<'PY'
import csv,sys
rows=[r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith('=='))]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
for r in rows[1:]:
    if len(r)>vi:
        v=float(r[vi].replace(',','')); u=r[ui]
        ms=v/1e6 if u=='nsecond' else v/1e3 if u=='usecond' else v
        print(f"{ms:10.3f} ms  {r[ki][:110]}")
PY
