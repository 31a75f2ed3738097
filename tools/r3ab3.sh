#!/bin/bash
OUT=gpurun_out/r3ab3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sssp or SSSP or golden" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for v in "SP_NF_ASYNC_THREADS=32" "SP_NF_ASYNC_THREADS=128" "SP_NF_ASYNC_THREADS=256" "SP_NF_ASYNC_THREADS=128 SP_SSSP_DELTA=3200"; do
  echo "== $v"; env $v timeout 60 python tools/run_algo.py sssp_grid 2 2>&1 | tail -1
done
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "grid" > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
tail -2 $OUT/pytest_full.log
SP_NF_ASYNC_THREADS=128 timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_nf_async -s 1 -c 1 -o $OUT/async python tools/run_algo.py sssp_grid 2 > $OUT/ncu.log 2>&1; tail -1 $OUT/ncu.log
