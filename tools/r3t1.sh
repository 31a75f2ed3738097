#!/bin/bash
# TC upper-CSR build with 4 element groups in flight: parity and build phases.
OUT=gpurun_out/r3t1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tc or triangle" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
SP_TC_TRACE=1 python tools/run_algo.py tc_rmat24 2 > $OUT/trace.txt 2>&1
SP_TC_TRACE=1 python tools/run_algo.py tc 2 >> $OUT/trace.txt 2>&1
grep -E "upper build|rep" $OUT/trace.txt
