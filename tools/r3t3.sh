#!/bin/bash
OUT=gpurun_out/r3t3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for rep in 1 2; do for v in base pu1 pu3 pu4; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  echo "== $v"; SP_LIB=$L python tools/run_algo.py tc 3 2>&1 | tail -1 | sed 's/launches.*triangles/triangles/'
done; done
