#!/bin/bash
OUT=gpurun_out/r3bc2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for i in 1 2; do for v in base b5r6 pr5 pr6 fin5; do
  L=build/variants/$v/libstarplat_b200.so
  echo "== $v"; SP_LIB=$L timeout 200 python tools/run_algo.py bc256 3 2>&1 | tail -1
done; done
