#!/bin/bash
OUT=gpurun_out/r3h1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
python tools/prof_e2e_host.py > $OUT/prof.txt 2>&1; head -60 $OUT/prof.txt
