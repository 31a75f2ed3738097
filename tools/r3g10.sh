#!/bin/bash
# Grid SSSP, 2-hop rows at 384 threads: delta and backoff.
OUT=gpurun_out/r3g10; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
{
for d in 1200 1632 2000 2400; do echo "== DELTA=$d"; SP_SSSP_DELTA=$d SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async" | tail -1 | sed 's/ ring [0-9]*,//; s/far entries.*//'; done
for b in 64 128 512 1024; do echo "== BACKOFF=$b"; SP_NF_ASYNC_BACKOFF=$b SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async" | tail -1 | sed 's/ ring [0-9]*,//; s/far entries.*//'; done
for t in 320 448; do echo "== THREADS=$t"; SP_NF_ASYNC_THREADS=$t SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async" | tail -1 | sed 's/ ring [0-9]*,//; s/far entries.*//'; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
