#!/bin/bash
# cfg1 through the direction-optimising loop with smaller grids for small graphs.
OUT=gpurun_out/r3c10; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for rep in 1 2; do for v in base dg2 dg4; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  echo "== $v DO"; SP_LIB=$L SP_SSSP_DO=1 python tools/run_algo.py sssp 6 2>&1 | tail -1 | sed 's/launches.*iters/iters/'
  [ $rep = 1 ] && { echo "== $v DO trace"; SP_LIB=$L SP_SSSP_DO=1 SP_HOSTLOOP=2 SP_SSSP_TRACE=1 python tools/run_algo.py sssp 3 2>&1 | grep "do it" | tail -9; }
done; done
echo "== BF default"; python tools/run_algo.py sssp 6 2>&1 | tail -1 | sed 's/launches.*iters/iters/'
