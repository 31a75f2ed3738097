#!/bin/bash
# ncu --set full of one k_pr_epi launch (cfg2), with source.
OUT=gpurun_out/r3e2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
SP_HOSTLOOP=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pr_epi -s 3 -c 1 -o $OUT/epi python tools/run_algo.py pr 2 > $OUT/ncu.log 2>&1
tail -2 $OUT/ncu.log
