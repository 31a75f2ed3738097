#!/bin/bash
OUT=gpurun_out/r3f2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 2400 python tools/fuzz_parity.py 2000 77 > $OUT/fuzz.log 2>&1; echo "rc=$?"; tail -5 $OUT/fuzz.log
