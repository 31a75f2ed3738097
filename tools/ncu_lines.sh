#!/bin/bash
# DRAM bytes of one steady run per bench line: ncu launch metrics over the
# kernels inside the NVTX range "steady" (the last rep of tools/run_algo.py),
# summed by tools/ncu_runs.py into profiles/ncu_summary.json ("run:<line>").
# usage: gpurun -- bash tools/ncu_lines.sh TAG
TAG=${1:-lines}; OUT=gpurun_out/$TAG; mkdir -p $OUT
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
run() {  # name algo [env...]
  local name=$1 algo=$2; shift 2
  env SP_NVTX=1 "$@" timeout 900 ncu --nvtx --nvtx-include "steady/" --metrics $M --clock-control none \
      --csv --log-file $OUT/$name.csv python tools/run_algo.py $algo 2 > $OUT/$name.log 2>&1
  echo "$name rc=$?"
}
run pr_cfg2 pr SP_HOSTLOOP=1
run sssp_cfg1 sssp SP_HOSTLOOP=2
run sssp_rmat24 sssp_rmat24 SP_HOSTLOOP=2
run sssp_grid sssp_grid
run pr_grid sssp_grid_pr SP_HOSTLOOP=1
run bc_cfg4 bc SP_NONE=0
run tc_cfg3 tc
run tc_rmat24 tc_rmat24
run pr_rmat24 pr_rmat24 SP_HOSTLOOP=1
python tools/ncu_runs.py $OUT/*.csv
