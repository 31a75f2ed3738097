#!/bin/bash
# Grid SSSP: ring ownership granularity (2^shift consecutive vertices per ring chunk).
OUT=gpurun_out/r3g17; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
{
for rep in 1 2; do
for v in own3 own4 own5; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  echo "== $v"; SP_LIB=$L SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp_grid rep 2|sssp async" | tail -2
done; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
