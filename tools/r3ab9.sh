#!/bin/bash
OUT=gpurun_out/r3ab9; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sssp or SSSP or golden or tc or TC" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log; grep -m3 "Error\|assert" $OUT/pytest.log
for t in 256 512 128; do
  echo "== threads $t"; SP_SSSP_TRACE=1 SP_NF_ASYNC_THREADS=$t timeout 60 python tools/run_algo.py sssp_grid 3 2>&1 | grep "async\|rep 2"
done
for i in 1 2; do
timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "grid_cfg5_bellman" > $OUT/pytest_full$i.log 2>&1; echo "rc=$?" >> $OUT/pytest_full$i.log
tail -1 $OUT/pytest_full$i.log
done
