#!/bin/bash
OUT=gpurun_out/r3b2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for rep in 1 2; do for k in 3 4 5 6 8; do echo "== workers $k"; SP_BC_WORKERS=$k python tools/run_algo.py bc256 3 2>&1 | tail -1 | sed 's/launches.*//'; done; done
