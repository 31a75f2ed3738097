#!/bin/bash
OUT=gpurun_out/r3ab8; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tc or TC or golden" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
echo "== tc rmat24"; timeout 200 python tools/run_algo.py tc_rmat24 2 2>&1 | tail -1
echo "== tc rmat22"; timeout 200 python tools/run_algo.py tc_rmat22 3 2>&1 | tail -1
for d in 400 600 800 1200; do
  echo "== delta $d"; SP_SSSP_DELTA=$d SP_SSSP_TRACE=1 timeout 60 python tools/run_algo.py sssp_grid 2 2>&1 | grep "async\|rep 1"
done
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "tc_rmat24" > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
tail -1 $OUT/pytest_full.log
