#!/bin/bash
# cfg1 SSSP: packed (dist, stamp) words vs separate arrays; parity of the SSSP forms.
OUT=gpurun_out/r3c3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sssp" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
{
for f in 1 0 1 0; do echo "== PACKED=$f"; SP_SSSP_PACKED=$f python tools/run_algo.py sssp 6 2>&1 | tail -2; done
echo "== rmat22 packed"; python tools/run_algo.py sssp_rmat22 4 2>&1 | tail -1
echo "== rmat22 PACKED=0"; SP_SSSP_PACKED=0 python tools/run_algo.py sssp_rmat22 4 2>&1 | tail -1
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
