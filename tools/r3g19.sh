#!/bin/bash
OUT=gpurun_out/r3g19; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
python tools/run_algo.py sssp_grid 5 2>&1 | tail -3
for i in 1 2; do timeout 900 python bench.py --algos grid --steps 5 --warmup 3 --no-cpu > $OUT/b$i.json 2> $OUT/b$i.err; python -c "
import json; d=json.loads(open('$OUT/b$i.json').read().strip().splitlines()[-1]); a=d['algorithms']['sssp_cfg5_grid']; print('bench grid', a['ms'], a.get('iterations'), a.get('first_call_ms'))"; done
