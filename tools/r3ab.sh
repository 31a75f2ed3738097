#!/bin/bash
# A/B: TC window-bitmap owners; SSSP slot-based direction test + pull prefetch/min-blocks.
OUT=gpurun_out/r3ab; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tc or TC or sssp or SSSP" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for v in "SP_SSSP_SLOT_PCT=100000" "SP_SSSP_SLOT_PCT=40" "SP_SSSP_SLOT_PCT=40 SP_SPULL_MINB=4" "SP_SSSP_SLOT_PCT=25"; do
  echo "== $v"; env $v python tools/run_algo.py sssp_rmat24 4 2>&1 | tail -2
done
SP_HOSTLOOP=2 SP_SSSP_TRACE=1 python tools/run_algo.py sssp_rmat24 2 2>&1 | grep "do it" | tail -12
echo "== tc cfg3"; python tools/run_algo.py tc 3 2>&1 | tail -2
echo "== tc rmat24"; python tools/run_algo.py tc_rmat24 2 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "tc_cfg3 or sssp_rmat24" > $OUT/pytest_full.log 2>&1; echo "rc=$?" >> $OUT/pytest_full.log
tail -3 $OUT/pytest_full.log
