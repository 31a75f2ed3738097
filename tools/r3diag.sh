#!/bin/bash
# SSSP RMAT-24 per-iteration breakdown (host-driven DO loop) + ncu of its kernels; k_tc_big on RMAT-22.
OUT=gpurun_out/r3diag; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
SP_HOSTLOOP=2 SP_SSSP_TRACE=1 python tools/run_algo.py sssp_rmat24 3 > $OUT/sssp24_trace.txt 2>&1
python tools/run_algo.py sssp_rmat24 3 >> $OUT/sssp24_trace.txt 2>&1
N="ncu --set full --clock-control none --import-source on"
SP_HOSTLOOP=2 timeout 900 $N -k regex:"k_do_push|k_spull_units|k_do_push_chunks" -s 0 -c 24 -o $OUT/sssp24_do python tools/run_algo.py sssp_rmat24 1 > $OUT/ncu_sssp24.log 2>&1
timeout 900 $N -k regex:"k_tc_big" -s 0 -c 1 -o $OUT/tc22_big python tools/run_algo.py tc_rmat22 1 > $OUT/ncu_tc22.log 2>&1
tail -40 $OUT/sssp24_trace.txt; tail -2 $OUT/ncu_*.log
