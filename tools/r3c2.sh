#!/bin/bash
# cfg1 SSSP: fused single-kernel iterations vs the two-kernel form; parity; TC first-call inside the bench.
OUT=gpurun_out/r3c2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sssp" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
{
for f in 1 0 1 0; do echo "== FUSED=$f"; SP_SSSP_FUSED=$f python tools/run_algo.py sssp 6 2>&1 | tail -2; done
for gm in 2 3; do echo "== FUSED GRID_MUL=$gm"; SP_SSSP_GRID_MUL=$gm python tools/run_algo.py sssp 6 2>&1 | tail -1; done
echo "== rmat22 fused default"; python tools/run_algo.py sssp_rmat22 4 2>&1 | tail -1
echo "== rmat22 FUSED=0"; SP_SSSP_FUSED=0 python tools/run_algo.py sssp_rmat22 4 2>&1 | tail -1
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
SP_TC_TRACE=1 timeout 900 python bench.py --algos rmat24 --steps 3 --warmup 3 --no-cpu > $OUT/bench_rmat24.json 2> $OUT/bench_rmat24.err
grep "tc upper" $OUT/bench_rmat24.err; python -c "
import json; d=json.loads(open('$OUT/bench_rmat24.json').read().strip().splitlines()[-1])
for k,v in d.get('algorithms',{}).items(): print(k, v.get('ms'), v.get('first_call_ms'), v.get('upper_csr_build_ms'))"
