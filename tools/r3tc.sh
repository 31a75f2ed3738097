#!/bin/bash
OUT=gpurun_out/r3tc; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for v in base tcb128 tcb512 tcbnf tcb128nf; do
  if [ $v = base ]; then L=""; else L=build/variants/$v/libstarplat_b200.so; fi
  echo "== $v"
  SP_LIB=$L timeout 200 python tools/run_algo.py tc_rmat22 3 2>&1 | tail -1
  SP_LIB=$L timeout 300 python tools/run_algo.py tc_rmat24 2 2>&1 | tail -1
done
