#!/bin/bash
# Where the TC upper-CSR build stalls inside the full bench (after BC); e2e PR phase trace.
OUT=gpurun_out/r3m1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
SP_PR_TRACE=1 python tools/diag_e2e2.py > $OUT/e2e.txt 2>&1; tail -24 $OUT/e2e.txt
SP_TC_TRACE=1 timeout 900 python bench.py --algos bc,rmat24 --steps 3 --warmup 3 --no-cpu > $OUT/b1.json 2> $OUT/b1.err
echo "== bc,rmat24"; grep -E "^tc" $OUT/b1.err | head -12
SP_BC_WORKERS=1 SP_TC_TRACE=1 timeout 900 python bench.py --algos bc,rmat24 --steps 3 --warmup 3 --no-cpu > $OUT/b2.json 2> $OUT/b2.err
echo "== bc(1 worker),rmat24"; grep -E "^tc" $OUT/b2.err | head -12
