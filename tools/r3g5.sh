#!/bin/bash
# Grid SSSP with shortcut rows: delta sweep.
OUT=gpurun_out/r3g5; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
{
for d in 1600 2400 3200 4000 4800 6400; do echo "== DELTA=$d"; SP_SSSP_DELTA=$d SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async" | tail -1 | sed 's/.*ring [0-9]*, //'; done
for d in 1600 3200; do echo "== SHORTCUT=0 DELTA=$d"; SP_NF_SHORTCUT=0 SP_SSSP_DELTA=$d SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async" | tail -1 | sed 's/.*ring [0-9]*, //'; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
