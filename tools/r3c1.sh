#!/bin/bash
# cfg1 SSSP (RMAT-16) latency: per-iteration trace, loop forms, grid sizes, ncu of the relax kernels.
OUT=gpurun_out/r3c1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
{
echo "== host loop trace"; SP_HOSTLOOP=1 SP_SSSP_TRACE=1 python tools/run_algo.py sssp 3 2>&1 | tail -16
echo "== default"; python tools/run_algo.py sssp 5 2>&1 | tail -2
for gm in 1 2 8; do echo "== GRID_MUL=$gm"; SP_SSSP_GRID_MUL=$gm python tools/run_algo.py sssp 5 2>&1 | tail -1; done
echo "== DO"; SP_SSSP_DO=1 python tools/run_algo.py sssp 5 2>&1 | tail -2
echo "== DO trace"; SP_SSSP_DO=1 SP_HOSTLOOP=2 SP_SSSP_TRACE=1 python tools/run_algo.py sssp 3 2>&1 | tail -16
} > $OUT/log.txt 2>&1
SP_HOSTLOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_expand|k_chunks|Relax" -s 0 -c 30 -o $OUT/cfg1 python tools/run_algo.py sssp 1 > $OUT/ncu.log 2>&1
cat $OUT/log.txt; tail -3 $OUT/ncu.log
