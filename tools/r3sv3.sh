#!/bin/bash
OUT=gpurun_out/r3sv3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sssp or SSSP" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -1 $OUT/pytest.log
for i in 1 2; do for v in base dp5 dp6; do
  L=build/variants/$v/libstarplat_b200.so
  echo "== $v"; SP_LIB=$L timeout 200 python tools/run_algo.py sssp_rmat24 5 2>&1 | tail -1
done; done
for v in "SP_NF_ASYNC_THREADS=256" "SP_NF_ASYNC_THREADS=256 SP_NF_ASYNC_BPS=2" "SP_NF_ASYNC_THREADS=384" "SP_NF_ASYNC_THREADS=192" "SP_NF_ASYNC_BACKOFF=128" "SP_NF_ASYNC_BACKOFF=1024" "SP_NF_ASYNC_THREADS=128 SP_NF_ASYNC_BPS=2"; do
  echo "== $v"; env $v SP_SSSP_TRACE=1 timeout 60 python tools/run_algo.py sssp_grid 3 2>&1 | grep "async" | tail -1
done
