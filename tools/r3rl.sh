#!/bin/bash
OUT=gpurun_out/r3rl; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
for i in 1 2; do for v in base rl5 rl6; do
  L=build/variants/$v/libstarplat_b200.so; [ $v = base ] && L=""
  echo "== $v"; SP_LIB=$L timeout 200 python tools/run_algo.py sssp 6 2>&1 | tail -1
  SP_LIB=$L timeout 200 python tools/run_algo.py sssp_rmat22 4 2>&1 | tail -1
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tc or TC or bc or BC" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -1 $OUT/pytest.log
