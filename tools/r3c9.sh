#!/bin/bash
# Frontier vertices per warp: one batch per warp (share 2/4) vs >= one batch per warp.
OUT=gpurun_out/r3c9; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
{
for rep in 1 2; do
for v in base vpw2 vpw4; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  echo "== $v"; SP_LIB=$L python tools/run_algo.py sssp 8 2>&1 | tail -1
  [ $rep = 1 ] && SP_LIB=$L python tools/run_algo.py sssp_rmat22 4 2>&1 | tail -1
  [ $rep = 1 ] && SP_LIB=$L python tools/run_algo.py sssp_rmat24 3 2>&1 | tail -1
  [ $rep = 1 ] && SP_LIB=$L python tools/run_algo.py bc256 2 2>&1 | tail -1
done; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt | sed 's/launches.*iters/iters/'
