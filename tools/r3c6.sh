#!/bin/bash
# Block-aggregated end-of-kernel frontier flush: A/B on cfg1, RMAT-22 (BF loop), RMAT-24 (DO loop), BC cfg4.
OUT=gpurun_out/r3c6; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sssp or bc" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
{
for rep in 1 2; do
for v in base nobf rl4; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  echo "== $v"
  SP_LIB=$L python tools/run_algo.py sssp 6 2>&1 | tail -1
  SP_LIB=$L python tools/run_algo.py sssp_rmat22 4 2>&1 | tail -1
  [ $rep = 1 ] && SP_LIB=$L python tools/run_algo.py sssp_rmat24 3 2>&1 | tail -1
  [ $rep = 1 ] && SP_LIB=$L python tools/run_algo.py bc256 2 2>&1 | tail -1
done; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
