#!/bin/bash
# synccheck + memcheck over the whole GPU parity file (device loops on)
OUT=gpurun_out/${1:-sanq}; mkdir -p $OUT
make -s -C paper_2305_03317_b200/csrc > /dev/null 2>&1
for tool in synccheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 10 \
      python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "not loader" -p no:cacheprovider > $OUT/$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $OUT/$tool.log | tail -2
done
