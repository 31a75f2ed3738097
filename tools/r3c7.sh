#!/bin/bash
# SSSP packed path + prep timers: GPU tests, memcheck/synccheck of the SSSP parity tests, quick bench of tc/rmat24.
OUT=gpurun_out/r3c7; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -k "not fullsize" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 10 \
    python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "packed_words or cfg1 or negative or preprocessing" -p no:cacheprovider > $OUT/$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $OUT/$tool.log | tail -2
done
timeout 900 python bench.py --algos tc,rmat24 --steps 3 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err
python -c "
import json; d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1])
for k,v in d.get('algorithms',{}).items(): print(k, round(v.get('ms'),3), v.get('first_call_ms'), v.get('first_calls_ms'), v.get('upper_csr_build_ms'), v.get('preprocessing_ms'))"
tail -3 $OUT/bench.err
