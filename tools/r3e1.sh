#!/bin/bash
# PR epilogue: upper bound of removing its nzrow-dependent loads (timing only; the variant's ranks are wrong).
OUT=gpurun_out/r3e1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
{
for v in base epinodep base epinodep; do
  L=""; [ $v != base ] && L=build/variants/$v/libstarplat_b200.so
  echo "== $v"; SP_LIB=$L python tools/run_algo.py pr 4 2>&1 | tail -1
done
SP_HOSTLOOP=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_pr_epi -c 6 python tools/run_algo.py pr 2 2>&1 | grep -E "k_pr_epi|duration|bytes" | tail -8
SP_LIB=build/variants/epinodep/libstarplat_b200.so SP_HOSTLOOP=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_pr_epi -c 6 python tools/run_algo.py pr 2 2>&1 | grep -E "duration|bytes" | tail -6
} > $OUT/log.txt 2>&1
cat $OUT/log.txt
