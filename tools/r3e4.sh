#!/bin/bash
# PR: unrolled init/unperm (base) vs init1; epilogue rows per thread 2/4; cfg2 and RMAT-24.
OUT=gpurun_out/r3e4; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pagerank or pr_" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
{
for rep in 1 2; do
for v in base init1 epi2 epi4; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  echo "== $v"; SP_LIB=$L python tools/run_algo.py pr 6 2>&1 | tail -1
  SP_LIB=$L python tools/run_algo.py pr_rmat24 4 2>&1 | tail -1
done; done
SP_HOSTLOOP=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_pr_init|k_pr_unperm|k_pr_epi" -c 6 python tools/run_algo.py pr_rmat24 1 2>&1 | grep -E "k_pr_|duration" | tail -12
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
