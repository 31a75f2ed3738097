#!/bin/bash
# ncu --set full of the grid SSSP shortcut kernel (one launch).
OUT=gpurun_out/r3g14; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_nf_async" -s 1 -c 1 -o $OUT/grid python tools/run_algo.py sssp_grid 2 > $OUT/ncu.log 2>&1
tail -1 $OUT/ncu.log
