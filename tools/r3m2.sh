#!/bin/bash
# TC build after a 4-worker BC run: which allocation stalls.
OUT=gpurun_out/r3m2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
cat > $OUT/t.py <<'PY'
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2305_03317_b200 as sp
from paper_2305_03317_b200 import corpus
g = sp.generate("rmat", 20, 16, seed=1, undirected=True)
deg = np.diff(np.asarray(g.offsets))
srcs = np.random.default_rng(1).choice(np.flatnonzero(deg > 0), size=256, replace=False).tolist()
if sys.argv[1] == "bc":
    for _ in range(2): sp.run(corpus.BC, g, {"sourceSet": srcs})
g.close()
t = sp.generate("rmat", 24, 16, seed=1, undirected=True)
t0 = time.perf_counter(); sp.run(corpus.TC, t, {}); print("tc first", (time.perf_counter()-t0)*1e3, file=sys.stderr)
print(t.preprocessing_ms(), file=sys.stderr)
PY
for mode in nobc bc; do echo "== $mode"; SP_TC_TRACE=1 python $OUT/t.py $mode 2>&1 | grep -E "upper build|tc first|tc_upper" ; done
echo "== bc, workers 1"; SP_BC_WORKERS=1 SP_TC_TRACE=1 python $OUT/t.py bc 2>&1 | grep -E "upper build|tc first|tc_upper"
