#!/bin/bash
# Grid SSSP: 3-hop shortcut rows (32 slots) vs 2-hop (16).
OUT=gpurun_out/r3g7; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
SP_NF_SHORTCUT=3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "async or sssp_seeded" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
{
for rep in 1 2; do
for v in 2 3; do echo "== SHORTCUT=$v"; SP_NF_SHORTCUT=$v SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async" | tail -1 | sed 's/.*ring [0-9]*, //'; done
done
for d in 1600 3200 4800; do echo "== SHORTCUT=3 DELTA=$d"; SP_NF_SHORTCUT=3 SP_SSSP_DELTA=$d SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async" | tail -1 | sed 's/.*ring [0-9]*, //'; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
SP_NF_SHORTCUT=3 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "grid" > $OUT/pytest_full.log 2>&1; tail -2 $OUT/pytest_full.log
