#!/bin/bash
# Randomised parity sweep of every fast form against the oracle (round-2 code).
OUT=gpurun_out/r3f1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 1800 python tools/fuzz_parity.py 200 2024 > $OUT/fuzz.log 2>&1; echo "rc=$?"; tail -5 $OUT/fuzz.log
