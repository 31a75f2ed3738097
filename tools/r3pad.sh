#!/bin/bash
OUT=gpurun_out/r3pad; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for v in base pad4 pad16; do
  L=build/variants/$v/libstarplat_b200.so; [ $v = base ] && L=""
  echo "== $v"; SP_LIB=$L timeout 200 python tools/run_algo.py tc 3 2>&1 | tail -1
  SP_LIB=$L timeout 300 python tools/run_algo.py tc_rmat24 2 2>&1 | tail -1
  SP_LIB=$L SP_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "steady/" --metrics dram__bytes_read.sum,gpu__time_duration.sum --csv --log-file $OUT/$v.csv python tools/run_algo.py tc 2 > /dev/null 2>&1
  grep -h "dram__bytes_read" $OUT/$v.csv | tail -1 | cut -c1-300
done
