#!/bin/bash
OUT=gpurun_out/r3hub3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tc or TC or golden" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log; grep -m5 "Error\|assert" $OUT/pytest.log
for v in base hm128 hm64 hm32 hs48 hs16; do
  L=build/variants/$v/libstarplat_b200.so; [ $v = base ] && L=""
  echo "== $v"; SP_LIB=$L timeout 300 python tools/run_algo.py tc_rmat24 2 2>&1 | tail -1
  SP_LIB=$L timeout 300 python tools/run_algo.py tc_rmat22 3 2>&1 | tail -1
done
