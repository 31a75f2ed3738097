#!/bin/bash
OUT=gpurun_out/r3sv; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for v in base sp5 sp6 dc4 dc5; do
  if [ $v = base ]; then L=""; else L=build/variants/$v/libstarplat_b200.so; fi
  echo "== $v"; SP_LIB=$L timeout 200 python tools/run_algo.py sssp_rmat24 4 2>&1 | tail -1
done
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N -k regex:k_nf_async -s 1 -c 1 -o $OUT/async python tools/run_algo.py sssp_grid 2 > $OUT/ncu_async.log 2>&1
SP_HOSTLOOP=1 timeout 600 $N -k regex:"k_pr_units_rel|k_pr_epi" -s 8 -c 2 -o $OUT/pr24_rel python tools/run_algo.py pr_rmat24 3 > $OUT/ncu_rel.log 2>&1
SP_PR_REL=0 SP_HOSTLOOP=1 timeout 600 $N -k regex:"k_pr_units_hot|k_pr_epi" -s 8 -c 2 -o $OUT/pr24_hot python tools/run_algo.py pr_rmat24 3 > $OUT/ncu_hot.log 2>&1
tail -1 $OUT/ncu_*.log
