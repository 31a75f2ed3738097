#!/bin/bash
OUT=gpurun_out/r3g21; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "shortcut_rows or preprocessing" > $OUT/pytest.log 2>&1; tail -5 $OUT/pytest.log
