#!/bin/bash
# cfg1 SSSP: packed words with / without the dist[x] pre-read.
OUT=gpurun_out/r3c4; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "packed_words or cfg1 or negative" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
{
for f in 0 1 0 1; do echo "== PROBE=$f"; SP_SSSP_PROBE=$f python tools/run_algo.py sssp 6 2>&1 | tail -2; done
for f in 0 1; do echo "== rmat20 PROBE=$f"; SP_SSSP_PROBE=$f python tools/run_algo.py sssp_rmat20 4 2>&1 | tail -1; done
for f in 0 1; do echo "== rmat22 PROBE=$f"; SP_SSSP_PROBE=$f python tools/run_algo.py sssp_rmat22 4 2>&1 | tail -1; done
echo "== trace probe0"; SP_HOSTLOOP=1 SP_SSSP_TRACE=1 SP_SSSP_PROBE=0 python tools/run_algo.py sssp 2 2>&1 | tail -11
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
SP_TC_TRACE=1 timeout 900 python bench.py --algos tc,rmat24 --steps 3 --warmup 3 --no-cpu > $OUT/bench_tc.json 2> $OUT/bench_tc.err
grep "^tc" $OUT/bench_tc.err | tail -30
