#!/bin/bash
# cfg1 SSSP: the asynchronous kernel forced onto RMAT-16 (hub rows walked by one warp), single phase.
OUT=gpurun_out/r3c5; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
{
for d in 1000000000 2000 200; do echo "== async delta $d"; SP_NF_ASYNC=2 SP_SSSP_DELTA=$d SP_SSSP_TRACE=1 timeout 120 python tools/run_algo.py sssp 4 2>&1 | grep -v "sssp:" | tail -3; done
echo "== default"; python tools/run_algo.py sssp 4 2>&1 | tail -1
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
