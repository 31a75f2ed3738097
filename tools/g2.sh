#!/bin/bash
# quick PR-focused GPU pass: build, PR + boundary tests, bench line (PR + RMAT-24 rows)
OUT=gpurun_out/${1:-g2}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "${2:-pr or PR or lists or from_csr or random or hook or smoke}" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -25 $OUT/pytest.log
timeout 600 python bench.py --algos ${3:-rmat24} --no-cpu > $OUT/bench.json 2> $OUT/bench.err
python - $OUT/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value",d["value"],"ms",d["ms_per_step"],"frac",d["roofline"]["frac"],"mean_it_ms",d["roofline"]["mean_launch_ms"],"e2e",d["e2e"]["value"],d["e2e"]["ms_per_step"], "launches", d.get("gpu_launches"))
for k,v in d.get("algorithms",{}).items(): print(k, v["ms"], v.get("roofline",{}).get("frac"))
PY
tail -3 $OUT/bench.err
