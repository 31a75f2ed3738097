#!/bin/bash
# Full round-2 pass: GPU tests, smoke, default bench, per-line ncu traffic, launch list.
OUT=gpurun_out/r3full9; mkdir -p $OUT
nvidia-smi > $OUT/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -15 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log
python - $OUT/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value",d["value"],"ms",d["ms_per_step"],"frac",d["roofline"]["frac"],"mean_it_ms",d["roofline"]["mean_launch_ms"],"e2e",d["e2e"]["value"],d["e2e"]["ms_per_step"], "launches", d.get("gpu_launches"))
for k,v in d.get("algorithms",{}).items(): print(k, round(v["ms"],3), v.get("gteps"), v.get("roofline",{}).get("frac"), {kk:vv for kk,vv in v.items() if kk.startswith(("first","upper"))})
PY
tail -3 $OUT/bench.err
bash tools/ncu_lines.sh r3lines9 > $OUT/ncu_lines.log 2>&1; cat $OUT/ncu_lines.log | tail -12
