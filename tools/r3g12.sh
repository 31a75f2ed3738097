#!/bin/bash
# Grid SSSP with 12-slot shortcut rows (default): parity, threads sweep, bench line.
OUT=gpurun_out/r3g18; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_parallel.py -q -x -k "sssp or grid or async" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
{
for t in 320; do echo "== threads $t"; SP_NF_ASYNC_THREADS=$t SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async" | tail -1 | sed 's/ ring [0-9]*,//; s/far entries.*//'; done
for d in 2448; do echo "== delta $d"; SP_SSSP_DELTA=$d SP_SSSP_TRACE=1 timeout 300 python tools/run_algo.py sssp_grid 3 2>&1 | grep -E "sssp async" | tail -1 | sed 's/ ring [0-9]*,//; s/far entries.*//'; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
timeout 900 python bench.py --algos grid --steps 3 --warmup 3 --no-cpu > $OUT/b.json 2> $OUT/b.err; python -c "
import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); a=d['algorithms']['sssp_cfg5_grid']; print('bench grid', a['ms'], a.get('iterations'))"
