#!/bin/bash
# DO-SSSP: pull also when the push step's next frontier holds > m/k out-slots.
OUT=gpurun_out/r3s2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
{
for sd in 0 2 4 8 16; do
  echo "== SLOT_DIV=$sd"; SP_SSSP_SLOT_DIV=$sd python tools/run_algo.py sssp_rmat24 4 2>&1 | tail -1
  SP_SSSP_SLOT_DIV=$sd SP_HOSTLOOP=2 SP_SSSP_TRACE=1 python tools/run_algo.py sssp_rmat24 3 2>&1 | grep "sssp do it" | tail -11
done
for sd in 0 4; do echo "== rmat26 SLOT_DIV=$sd"; SP_SSSP_SLOT_DIV=$sd python tools/run_algo.py sssp_rmat26 3 2>&1 | tail -1; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
