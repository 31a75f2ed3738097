#!/bin/bash
# ncu launch list (gpu__time_duration) of a command on the GPU box.
# usage: gpurun -- bash tools/launches.sh TAG <command...>
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
make -s -C paper_2305_03317_b200/csrc > $OUT/make.log 2>&1 || { tail -20 $OUT/make.log; exit 1; }
"$@" > $OUT/plain.log 2>&1; cat $OUT/plain.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv "$@" > $OUT/ncu.log 2>&1
tail -2 $OUT/ncu.log
