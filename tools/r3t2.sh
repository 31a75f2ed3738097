#!/bin/bash
OUT=gpurun_out/r3t2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tc_big_row_forms" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
