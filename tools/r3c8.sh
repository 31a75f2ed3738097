#!/bin/bash
# cfg1 / RMAT-22 BF device loop (packed words): grid blocks per SM.
OUT=gpurun_out/r3c8; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
{
for rep in 1 2; do
for gm in 2 3 4 5 6; do
  echo "== GRID_MUL=$gm"; SP_SSSP_GRID_MUL=$gm python tools/run_algo.py sssp 8 2>&1 | tail -1
  [ $rep = 1 ] && SP_SSSP_GRID_MUL=$gm python tools/run_algo.py sssp_rmat20 4 2>&1 | tail -1
done; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
