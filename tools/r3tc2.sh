#!/bin/bash
OUT=gpurun_out/r3tc2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for i in 1 2; do for v in base tch5 tcp6 tcp8; do
  L=build/variants/$v/libstarplat_b200.so; [ $v = base ] && L=""
  echo "== $v"; SP_LIB=$L timeout 200 python tools/run_algo.py tc 3 2>&1 | tail -1
  SP_LIB=$L timeout 300 python tools/run_algo.py tc_rmat24 2 2>&1 | tail -1
done; done
echo "== bc new defaults"; for i in 1 2; do timeout 200 python tools/run_algo.py bc256 3 2>&1 | tail -1; done
