#!/bin/bash
OUT=gpurun_out/r3g9; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_parallel.py -q -x -k "sssp or grid or async" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for i in 1 2; do SP_SSSP_TRACE=1 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async|rep 2" | tail -2; done
timeout 900 python bench.py --algos grid --steps 3 --warmup 3 --no-cpu > $OUT/b.json 2> $OUT/b.err; python -c "
import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); a=d['algorithms']['sssp_cfg5_grid']; print('bench grid', a['ms'], a.get('iterations'))"
