"""Time the reference's own Python interpreter (trident.interp.run) on
BASELINE cfg1 -- SSSP from vertex 0 on weighted RMAT-16 -- with the same
edges our device generator produces (gen.rmat is bit-identical to it).
Runs only where /root/reference exists (this container, not the GPU box);
writes profiles/reference_python_cfg1.json."""
import json
import os
import sys
import time

REF = os.environ.get("TRIDENT_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from trident.graph import from_edges  # noqa: E402
from trident.interp import run  # noqa: E402
from trident.parser import parse_source  # noqa: E402
from trident.sema import analyze  # noqa: E402

from paper_2305_03317_b200 import gen  # noqa: E402

u, v, w, n = gen.rmat(16, 16, seed=1)
t0 = time.perf_counter()
g = from_edges(list(zip(u.tolist(), v.tolist(), w.tolist())), directed=True)
t_build = time.perf_counter() - t0
src = open(os.path.join(REF, "trident", "corpus", "programs", "sssp.sp")).read()
tp = analyze(parse_source(src))
res = run(tp, g, {"src": 0})
dist = res.env.node_props["dist"]
offs = g.offsets
reached = sum(offs[x + 1] - offs[x] for x in range(g.n) if dist[x] < 2147483647)
out = {"workload": "sssp_cfg1 (RMAT-16 ef16 seed 1, src 0)", "n": g.n, "m": len(g.adj),
       "csr_build_s": t_build, "run_wall_seconds": res.wall_seconds,
       "gteps": reached / res.wall_seconds / 1e9,
       "fixedpoint_iterations": res.fixedpoint_iterations,
       "host": "graft build container (not the GPU box): " + os.popen("nproc").read().strip()
               + " cores, single-threaded interpreter",
       "python": sys.version.split()[0]}
os.makedirs("profiles", exist_ok=True)
json.dump(out, open("profiles/reference_python_cfg1.json", "w"), indent=1)
print(json.dumps(out))
