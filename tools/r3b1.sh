#!/bin/bash
# BC pull discovery: flattened warp form vs thread per row.
OUT=gpurun_out/r3b1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "bc or betweenness" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
{
for rep in 1 2; do
for v in base pullthread; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  echo "== $v"; SP_LIB=$L python tools/run_algo.py bc256 3 2>&1 | tail -1
done; done
M=gpu__time_duration.sum
for v in base pullthread; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  echo "== ncu $v"; SP_LIB=$L SP_BC_WORKERS=1 ncu --metrics $M --clock-control none -k regex:"k_bb_pull_rows" -c 40 python tools/run_algo.py bc 1 2>&1 | grep -E "duration" | awk '{s+=$3} END {print "pull_rows total us", s, "launches", NR}'
done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "bc" > $OUT/pytest_full.log 2>&1; tail -2 $OUT/pytest_full.log
