#!/bin/bash
OUT=gpurun_out/r3hub2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tc or TC or golden" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log; grep -m5 "Error\|assert" $OUT/pytest.log
for v in "SP_TC_HUB=0" "SP_TC_HUB=2" "SP_TC_HUB=1"; do
  echo "== $v"; env $v timeout 300 python tools/run_algo.py tc_rmat24 2 2>&1 | tail -1
  env $v timeout 300 python tools/run_algo.py tc_rmat22 3 2>&1 | tail -1
  env $v timeout 300 python tools/run_algo.py tc 2 2>&1 | tail -1
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "tc" > $OUT/pf.log 2>&1; echo "rc=$?" >> $OUT/pf.log; tail -1 $OUT/pf.log
