#!/bin/bash
# Grid SSSP, 2-hop shortcut rows: threads per block / blocks per SM.
OUT=gpurun_out/r3g8; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
{
for rep in 1 2; do
for cfg in "256 1" "512 1" "384 1" "128 2" "256 2" "128 4"; do
  set -- $cfg
  echo "== threads $1 bps $2"; SP_NF_ASYNC_THREADS=$1 SP_NF_ASYNC_BPS=$2 SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async" | tail -1 | sed 's/ ring [0-9]*,//; s/far entries.*//'
done; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
