#!/bin/bash
# ncu --set full of one kernel on the GPU box.
# usage: gpurun -- bash tools/ncu_one.sh TAG REGEX SKIP COUNT <command...>
TAG=$1; RX=$2; SKIP=$3; CNT=$4; shift 4
OUT=gpurun_out/$TAG; mkdir -p $OUT
make -s -C paper_2305_03317_b200/csrc > $OUT/make.log 2>&1 || { tail -20 $OUT/make.log; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$RX -s $SKIP -c $CNT \
    -o $OUT/prof_$RX "$@" > $OUT/ncu_$RX.log 2>&1
tail -3 $OUT/ncu_$RX.log
