#!/bin/bash
# PR hot set split over a 2-CTA cluster (DSMEM) vs one CTA's shared memory.
OUT=gpurun_out/r3k1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
SP_PR_HOT_MAX=40960 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pagerank or pr_ or sssp_pull_hot" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
{
for rep in 1 2; do
for hm in 20480 28672 40960; do
  echo "== HOT_MAX=$hm"; SP_PR_HOT_MAX=$hm SP_PR_HOT_VERBOSE=1 python tools/run_algo.py pr 6 2>&1 | grep -E "hot set|rep 5" | tail -2
  [ $rep = 1 ] && SP_PR_REL=0 SP_PR_HOT_MAX=$hm SP_PR_HOT_VERBOSE=1 python tools/run_algo.py pr_rmat24 4 2>&1 | grep -E "hot set|rep 3" | tail -2
done; done
SP_PR_HOT_MAX=40960 SP_HOSTLOOP=1 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:"k_pr_units_hot" -c 3 python tools/run_algo.py pr 2 2>&1 | grep -E "k_pr_units|duration|wavefronts|sectors" | tail -8
SP_HOSTLOOP=1 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:"k_pr_units_hot" -c 3 python tools/run_algo.py pr 2 2>&1 | grep -E "k_pr_units|duration|wavefronts|sectors" | tail -8
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
