#!/bin/bash
# SSSP RMAT-24 pull sweeps with larger hot snapshots (int32 dist: 30 K / 40 K sources = 120 / 160 KB).
OUT=gpurun_out/r3s1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
{
for rep in 1 2; do
for hm in 20480 30720 40960 12288; do
  echo "== HOT_MAX=$hm"; SP_PR_HOT_MAX=$hm SP_PR_HOT_VERBOSE=1 python tools/run_algo.py sssp_rmat24 4 2>&1 | grep -E "hot set|rep 3" | tail -2
  [ $rep = 1 ] && SP_PR_HOT_MAX=$hm python tools/run_algo.py sssp_rmat26 3 2>&1 | tail -1
done; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
