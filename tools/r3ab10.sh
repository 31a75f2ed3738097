#!/bin/bash
OUT=gpurun_out/r3ab10; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parallel.py tests/test_host.py tests/test_gpu_parity.py -m gpu -x -q -k "parallel or tc or TC or host or pagerank or PR" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log; grep -m5 "Error\|assert" $OUT/pytest.log
echo "== tc rmat24"; timeout 200 python tools/run_algo.py tc_rmat24 2 2>&1 | tail -1
echo "== tc rmat22"; timeout 200 python tools/run_algo.py tc_rmat22 3 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "tc_rmat24" > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
tail -1 $OUT/pytest_full.log
bash tools/ncu_lines.sh r3lines2 > $OUT/ncu_lines.log 2>&1; tail -10 $OUT/ncu_lines.log
