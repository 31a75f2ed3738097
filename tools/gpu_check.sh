#!/bin/bash
# One gpurun call: GPU parity tests, bench line, ncu launch list + full capture.
# usage: gpurun -- bash tools/gpu_check.sh [tag]
set -x
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvsmi.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --algos none > $OUT/ncu_launch_bench.log 2>&1
SP_HOSTLOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pr_units|k_pr_hot_gather|k_pr_epi" -s 28 -c 3 \
   -o $OUT/prof_pr python bench.py --steps 1 --warmup 1 --no-cpu --algos none > $OUT/ncu_full.log 2>&1
