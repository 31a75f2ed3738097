#!/bin/bash
OUT=gpurun_out/r3ab2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tc or TC or golden" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
echo "== tc cfg3"; timeout 120 python tools/run_algo.py tc 3 2>&1 | tail -2
echo "== tc rmat24"; timeout 200 python tools/run_algo.py tc_rmat24 2 2>&1 | tail -1
for v in "SP_NF_ASYNC_THREADS=32" "SP_NF_ASYNC_THREADS=64" "SP_NF_ASYNC_THREADS=128" "SP_NF_ASYNC_THREADS=256" "SP_NF_ASYNC_THREADS=64 SP_NF_ASYNC_BACKOFF=2048" "SP_NF_ASYNC_THREADS=64 SP_NF_ASYNC_BACKOFF=128"; do
  echo "== $v"; env $v timeout 60 python tools/run_algo.py sssp_grid 2 2>&1 | tail -1
done
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "tc_cfg3" > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
tail -2 $OUT/pytest_full.log
