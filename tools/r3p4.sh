#!/bin/bash
# PR: loop advance by the epilogue's last block vs a separate advance node.
OUT=gpurun_out/r3p4; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "pagerank or pr_ or cfg2" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
{
for rep in 1 2 3; do
for v in base sepadv; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  echo "== $v"; SP_LIB=$L python tools/run_algo.py pr 8 2>&1 | tail -1
  [ $rep = 1 ] && SP_LIB=$L python tools/run_algo.py pr_rmat24 4 2>&1 | tail -1
  [ $rep = 1 ] && SP_LIB=$L python tools/run_algo.py sssp_grid_pr 6 2>&1 | tail -1
done; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
