#!/bin/bash
# PR hot copy as two 32-bit halves (split) vs doubles.
OUT=gpurun_out/r3p3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pagerank or pr_" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
{
for rep in 1 2 3; do
for v in base nosplit; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  echo "== $v"; SP_LIB=$L python tools/run_algo.py pr 6 2>&1 | tail -1
  [ $rep = 1 ] && SP_LIB=$L python tools/run_algo.py pr_rmat24 4 2>&1 | tail -1
done; done
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__throughput.avg.pct_of_peak_sustained_active
for v in base nosplit; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  echo "== ncu $v"; SP_LIB=$L SP_HOSTLOOP=1 ncu --metrics $M --clock-control none -k regex:"k_pr_units_(hot|rel)" -s 2 -c 1 python tools/run_algo.py pr 3 2>&1 | grep -E "duration|wavefronts|throughput" | tail -3
done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
