#!/bin/bash
OUT=gpurun_out/r3sv2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for i in 1 2 3; do for v in base sp5dc4 sp5 dc4; do
  L=build/variants/$v/libstarplat_b200.so
  echo "== $v"; SP_LIB=$L timeout 200 python tools/run_algo.py sssp_rmat24 5 2>&1 | tail -1
done; done
for v in base sp5dc4; do L=build/variants/$v/libstarplat_b200.so; echo "== $v rmat26"; SP_LIB=$L timeout 300 python tools/run_algo.py sssp_rmat26 3 2>&1 | tail -1; done
