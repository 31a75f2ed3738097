#!/bin/bash
# DO-SSSP loop with conditional IF nodes (push / pull / clear+convert) vs every kernel every step.
OUT=gpurun_out/r3d1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sssp" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
{
for rep in 1 2; do
for v in 1 0; do
  echo "== DO_IF=$v"
  SP_SSSP_DO_IF=$v python tools/run_algo.py sssp_rmat24 4 2>&1 | tail -1
  SP_SSSP_DO_IF=$v SP_SSSP_DO=1 python tools/run_algo.py sssp_rmat22 4 2>&1 | tail -1
  SP_SSSP_DO_IF=$v SP_SSSP_DO=1 python tools/run_algo.py sssp 4 2>&1 | tail -1
done; done
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "rmat24 and sssp or rmat26" > $OUT/pytest_full.log 2>&1; tail -2 $OUT/pytest_full.log
