#!/bin/bash
OUT=gpurun_out/r3g20; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for rep in 1 2; do
for t in 256 320 384; do echo "== threads $t"; SP_NF_ASYNC_THREADS=$t SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async" | tail -1 | sed 's/ ring [0-9]*,//; s/far entries.*//'; done
for d in 3264 4080; do echo "== delta $d"; SP_SSSP_DELTA=$d SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async" | tail -1 | sed 's/ ring [0-9]*,//; s/far entries.*//'; done
done
