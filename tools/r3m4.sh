#!/bin/bash
# TC build stall inside the bench (bc,rmat24): pool state per phase.
OUT=gpurun_out/r3m4; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
SP_TC_TRACE=1 timeout 900 python bench.py --algos bc,rmat24 --steps 3 --warmup 3 --no-cpu > $OUT/b1.json 2> $OUT/b1.err
grep -E "^tc" $OUT/b1.err | head -12
