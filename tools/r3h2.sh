#!/bin/bash
OUT=gpurun_out/r3h2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
SP_PR_TRACE=1 python tools/diag_e2e3.py 2>&1 | tail -20
