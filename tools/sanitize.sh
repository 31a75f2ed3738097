#!/bin/bash
# compute-sanitizer over the GPU parity tests: memcheck and synccheck on the
# whole parity file (golden fixtures, seeded graphs, edge cases), racecheck
# on the heavier cases.  Summaries under gpurun_out/$1.
TAG=${1:-san}; OUT=gpurun_out/$TAG; mkdir -p $OUT
make -s -C paper_2305_03317_b200/csrc > /dev/null 2>&1
run() {  # tool, -k selection
  SP_HOSTLOOP=$3 timeout 2400 compute-sanitizer --tool $1 --error-exitcode 99 --print-limit 20 \
      python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$2" -p no:cacheprovider \
      > $OUT/$1_$3.log 2>&1
  echo "$1 (SP_HOSTLOOP=$3) rc=$?" >> $OUT/summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $OUT/$1_$3.log | tail -3 >> $OUT/summary.txt
}
run memcheck "not loader" 0
run memcheck "sssp or pagerank" 1
run synccheck "not loader" 0
run racecheck "rand200 or rmat10 or unif or hub or multigraph" 1
cat $OUT/summary.txt
