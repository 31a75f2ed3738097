#!/bin/bash
# Round-2 session-2 baseline: full GPU tests, default bench, launch list.
OUT=gpurun_out/r3base; mkdir -p $OUT
nvidia-smi > $OUT/nvsmi.txt 2>&1; lscpu > $OUT/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -25 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log
python - $OUT/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value",d["value"],"ms",d["ms_per_step"],"frac",d["roofline"]["frac"],"mean_it_ms",d["roofline"]["mean_launch_ms"],"e2e",d["e2e"]["value"],d["e2e"]["ms_per_step"], "launches", d.get("gpu_launches"))
for k,v in d.get("algorithms",{}).items(): print(k, round(v["ms"],3), v.get("gteps"), v.get("roofline",{}).get("frac"))
PY
tail -3 $OUT/bench.err
