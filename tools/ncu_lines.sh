#!/bin/bash
# DRAM bytes of one steady run per bench line: ncu launch metrics over the
# kernels inside the NVTX range "steady" (the last rep of tools/run_algo.py),
# summed by tools/ncu_runs.py into profiles/ncu_summary.json ("run:<line>").
# usage: gpurun -- bash tools/ncu_lines.sh TAG
TAG=${1:-lines}; OUT=gpurun_out/$TAG; mkdir -p $OUT
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
run() {  # name algo reps [env...] -- the last of `reps` runs is measured (the
  # earlier ones build the lazily cached per-graph structures)
  local name=$1 algo=$2 reps=$3; shift 3
  env SP_NVTX=1 "$@" timeout 900 ncu --nvtx --nvtx-include "steady/" --metrics $M --clock-control none \
      --csv --log-file $OUT/$name.csv python tools/run_algo.py $algo $reps > $OUT/$name.log 2>&1
  echo "$name rc=$?"
}
# SP_HOSTLOOP: host-driven loops (ncu cannot profile the kernel nodes of a
# conditional graph); BC with one worker: NVTX ranges are per host thread
run pr_cfg2 pr 3 SP_HOSTLOOP=1
run sssp_cfg1 sssp 2 SP_HOSTLOOP=1
run sssp_rmat24 sssp_rmat24 3 SP_HOSTLOOP=2
run sssp_grid sssp_grid 2
run pr_grid sssp_grid_pr 3 SP_HOSTLOOP=1
run bc_cfg4 bc256 2 SP_BC_WORKERS=1
run tc_cfg3 tc 2
run tc_rmat24 tc_rmat24 2
run pr_rmat24 pr_rmat24 3 SP_HOSTLOOP=1
python tools/ncu_runs.py $OUT/*.csv
