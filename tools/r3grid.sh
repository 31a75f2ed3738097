#!/bin/bash
OUT=gpurun_out/r3grid; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "grid" --durations=5 > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -8 $OUT/pytest.log
