#!/bin/bash
OUT=gpurun_out/r3loc; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sssp or SSSP or golden" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -1 $OUT/pytest.log; grep -m3 "Error\|assert" $OUT/pytest.log
for e in 1 0 1 0; do echo "== local=$e"; SP_NF_LOCAL=$e SP_SSSP_TRACE=1 timeout 60 python tools/run_algo.py sssp_grid 3 2>&1 | grep "async" | tail -1; done
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "grid_cfg5_bellman" > $OUT/pf$i.log 2>&1; echo "rc=$?" >> $OUT/pf$i.log; tail -1 $OUT/pf$i.log; done
