#!/bin/bash
# ncu --set full of one PR iteration (cfg2 hot-encoded; RMAT-24 relabelled) on the round-2 code.
OUT=gpurun_out/r3p1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
# cfg2: 3rd run (hot set built on the 2nd), one iteration = gather + units + epi (+ advance)
SP_HOSTLOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pr_(hot_gather|units_hot|epi)" -s 36 -c 3 -o $OUT/pr_cfg2 python tools/run_algo.py pr 3 > $OUT/ncu_cfg2.log 2>&1
tail -1 $OUT/ncu_cfg2.log
SP_HOSTLOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pr_(units_rel|epi)" -s 4 -c 2 -o $OUT/pr_rmat24 python tools/run_algo.py pr_rmat24 3 > $OUT/ncu_rmat24.log 2>&1
tail -1 $OUT/ncu_rmat24.log
