#!/bin/bash
OUT=gpurun_out/r3z; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --algos grid --steps 3 --warmup 3 > $OUT/b.json 2> $OUT/b.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'grid', round(d['algorithms']['sssp_cfg5_grid']['ms'],2), 'cpu', d['cpu_baseline']['value'])"
