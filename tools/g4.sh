#!/bin/bash
# ncu --set full of one PR iteration's row-sum kernel: relabelled vs hot-encoded layout (RMAT-22)
OUT=gpurun_out/g4; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
export SP_HOSTLOOP=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pr_units_rel|k_pr_epi|k_pr_unperm|k_pr_init" -s 14 -c 4 \
   -o $OUT/prof_rel python bench.py --steps 1 --warmup 1 --no-cpu --algos none > $OUT/ncu_rel.log 2>&1
SP_PR_REL=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pr_units_hot|k_pr_epi" -s 14 -c 2 \
   -o $OUT/prof_enc python bench.py --steps 1 --warmup 1 --no-cpu --algos none > $OUT/ncu_enc.log 2>&1
tail -2 $OUT/ncu_rel.log $OUT/ncu_enc.log
