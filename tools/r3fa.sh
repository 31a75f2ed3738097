#!/bin/bash
OUT=gpurun_out/r3fa; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_forall.py tests/test_gpu_parity.py -m gpu -x -q -k "forall or reduction or neighbor_sum" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -3 $OUT/pytest.log; grep -m5 "Error\|assert" $OUT/pytest.log
