#!/bin/bash
OUT=gpurun_out/r3p2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
SP_HOSTLOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pr_units_rel" -s 1 -c 1 -o $OUT/pr_rmat24_units python tools/run_algo.py pr_rmat24 3 > $OUT/ncu.log 2>&1
tail -1 $OUT/ncu.log
