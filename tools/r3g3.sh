#!/bin/bash
# Grid SSSP with 2-hop shortcut rows (kD = 16) vs the 1-hop ELL rows.
OUT=gpurun_out/r3g4; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "async or sssp_seeded or grid or sssp" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
{
for rep in 1 2; do
for v in 1 0; do
  echo "== SHORTCUT=$v"; SP_NF_SHORTCUT=$v SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp_grid rep 2|sssp async" | tail -2
done; done
for d in 3200; do echo "== SHORTCUT=1 DELTA=$d"; SP_SSSP_DELTA=$d SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp_grid rep 2|sssp async" | tail -2; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "grid" > $OUT/pytest_full.log 2>&1; tail -2 $OUT/pytest_full.log
