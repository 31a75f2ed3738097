#!/bin/bash
# Grid SSSP shortcut rows: 12 slots (the grid's 4 + 8 targets exactly) vs 16.
OUT=gpurun_out/r3g11; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
SP_LIB=build/variants/s12/libstarplat_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "async" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
{
for rep in 1 2; do
for v in base s12; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  for t in 384 512; do echo "== $v threads $t"; SP_LIB=$L SP_NF_ASYNC_THREADS=$t SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async" | tail -1 | sed 's/ ring [0-9]*,//; s/far entries.*//'; done
done; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
