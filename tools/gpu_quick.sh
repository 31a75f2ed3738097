#!/bin/bash
# Quick GPU iteration: build, the -m gpu tests (optionally filtered), a PR-only
# bench line, and an ncu capture of one kernel.
# usage: gpurun -- bash tools/gpu_quick.sh TAG [pytest -k expr] [ncu kernel regex] [bench args]
TAG=${1:-q}; KEXPR=${2:-}; KREGEX=${3:-}; BARGS=${4:---algos none --no-cpu}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
if [ -n "$KEXPR" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$KEXPR" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  tail -15 $OUT/pytest_gpu.log
fi
eval timeout 600 python bench.py $BARGS > $OUT/bench.json 2> $OUT/bench.err; cat $OUT/bench.json; tail -3 $OUT/bench.err
if [ -n "$KREGEX" ]; then
  eval timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 4 -c 2 \
     -o $OUT/prof python bench.py --steps 1 --warmup 1 $BARGS > $OUT/ncu_full.log 2>&1
  tail -2 $OUT/ncu_full.log
fi
