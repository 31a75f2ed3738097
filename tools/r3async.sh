#!/bin/bash
# Asynchronous near-far SSSP: parity + grid timings (every step under its own timeout).
OUT=gpurun_out/r3async; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sssp or SSSP or golden" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for v in "SP_NF_ASYNC=0" "SP_NF_ASYNC=1" "SP_NF_ASYNC=1 SP_NF_ASYNC_BPS=2" "SP_NF_ASYNC=1 SP_SSSP_DELTA=1600" "SP_NF_ASYNC=1 SP_SSSP_DELTA=400"; do
  echo "== $v"; env $v timeout 120 python tools/run_algo.py sssp_grid 3 2>&1 | tail -2
done
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "grid" > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
tail -3 $OUT/pytest_full.log
