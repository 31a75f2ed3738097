#!/bin/bash
OUT=gpurun_out/r3hot; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sssp or SSSP" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -1 $OUT/pytest.log; grep -m3 "Error\|assert" $OUT/pytest.log
for i in 1 2; do for h in 0 ""; do
  echo "== hot=$h"; SP_SSSP_HOT=$h timeout 200 python tools/run_algo.py sssp_rmat24 5 2>&1 | tail -1
  SP_SSSP_HOT=$h timeout 200 python tools/run_algo.py sssp_rmat26 3 2>&1 | tail -1
done; done
SP_HOSTLOOP=2 SP_SSSP_TRACE=1 timeout 200 python tools/run_algo.py sssp_rmat24 3 2>&1 | grep "do it" | tail -10
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "sssp_rmat24 or rmat26" > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log; tail -1 $OUT/pytest_full.log
