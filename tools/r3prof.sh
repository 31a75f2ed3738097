#!/bin/bash
# Round 2: native sharded-SSSP tests + ncu captures of the SSSP and TC kernels.
OUT=gpurun_out/r3prof; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parallel.py tests/test_host.py -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
N="ncu --set full --clock-control none --import-source on"
# SSSP: whole device loops (conditional graphs) profiled as one workload each
timeout 600 $N --graph-profiling graph -s 1 -c 1 -o $OUT/sssp_rmat24_graph python tools/run_algo.py sssp_rmat24 2 > $OUT/ncu_sssp24.log 2>&1
timeout 600 $N --graph-profiling graph -s 1 -c 1 -o $OUT/sssp_cfg1_graph python tools/run_algo.py sssp 2 > $OUT/ncu_sssp1.log 2>&1
timeout 900 $N -k regex:k_nf_persistent -s 1 -c 1 -o $OUT/sssp_grid_nf python tools/run_algo.py sssp_grid 2 > $OUT/ncu_grid.log 2>&1
# SSSP kernels one by one (host-driven loop) on RMAT-24
SP_HOSTLOOP=1 timeout 600 $N -k regex:k_expand -s 4 -c 4 -o $OUT/sssp_rmat24_expand python tools/run_algo.py sssp_rmat24 1 > $OUT/ncu_sssp24x.log 2>&1
# TC: cfg3 warp kernel, RMAT-24 big-row kernel
timeout 900 $N -k regex:k_tc_fwd_plain -s 1 -c 1 -o $OUT/tc_cfg3 python tools/run_algo.py tc 2 > $OUT/ncu_tc3.log 2>&1
timeout 1200 $N -k regex:"k_tc_big|k_tc_fwd_hash" -s 0 -c 2 -o $OUT/tc_rmat24 python tools/run_algo.py tc_rmat24 1 > $OUT/ncu_tc24.log 2>&1
for f in $OUT/ncu_*.log; do echo "== $f"; tail -2 $f; done
ls -la $OUT
