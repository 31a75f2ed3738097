#!/bin/bash
# TC build after the RMAT-24 directed PR/SSSP lines (the bench order): allocation stalls?
OUT=gpurun_out/r3m3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
cat > $OUT/t.py <<'PY'
import sys, time, os
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2305_03317_b200 as sp
from paper_2305_03317_b200 import corpus
PR = {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
mode = sys.argv[1]
def mem(tag):
    f, t = torch.cuda.mem_get_info(); print(f"{tag}: free {f/2**30:.1f} GiB", file=sys.stderr)
if mode != "none":
    g = sp.generate("rmat", 24, 16, seed=1)
    for _ in range(4): sp.run(corpus.PR, g, PR, device_outputs=True)
    if mode == "prsssp":
        for _ in range(4): sp.run(corpus.SSSP, g, {"src": 0}, device_outputs=True)
    mem("after directed lines")
    g.close()
    mem("after close")
t = sp.generate("rmat", 24, 16, seed=1, undirected=True)
mem("after sym generate")
t0 = time.perf_counter(); sp.run(corpus.TC, t, {}); print("tc first", (time.perf_counter()-t0)*1e3, file=sys.stderr)
print(t.preprocessing_ms(), file=sys.stderr)
PY
for mode in none pr prsssp; do echo "== $mode"; SP_TC_TRACE=1 python $OUT/t.py $mode 2>&1 | grep -E "upper build|tc first|tc_upper|free" ; done
