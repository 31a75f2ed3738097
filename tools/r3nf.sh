#!/bin/bash
OUT=gpurun_out/r3nf; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for d in 800 1600 3200; do SP_SSSP_DELTA=$d SP_SSSP_TRACE=1 timeout 60 python tools/run_algo.py sssp_grid 2 2>&1 | grep async | tail -1; done
