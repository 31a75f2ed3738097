OUT=gpurun_out/g3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python tools/diag_pr.py 22 > $OUT/diag.txt 2>&1
SP_HOSTLOOP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --algos none > $OUT/ncu.log 2>&1
python tools/ncu_summary.py launches $OUT/launches.csv > $OUT/launches.md 2>&1
cat $OUT/diag.txt; head -30 $OUT/launches.md
