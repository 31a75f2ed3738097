#!/bin/bash
# PR epilogue without the end-of-block barrier (last warp publishes the diff) vs the barrier form.
OUT=gpurun_out/r3e3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pagerank or pr_" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
{
for rep in 1 2 3; do
for v in base epibar; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  echo "== $v"; SP_LIB=$L python tools/run_algo.py pr 6 2>&1 | tail -1
  [ $rep = 1 ] && SP_LIB=$L python tools/run_algo.py pr_rmat24 4 2>&1 | tail -1
done; done
SP_HOSTLOOP=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pr_epi -c 6 python tools/run_algo.py pr 2 2>&1 | grep -E "duration" | tail -3
SP_LIB=build/variants/epibar/libstarplat_b200.so SP_HOSTLOOP=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pr_epi -c 6 python tools/run_algo.py pr 2 2>&1 | grep -E "duration" | tail -3
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
