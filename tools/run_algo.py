"""Run one corpus program on a BASELINE config graph (profiling driver).
usage: python tools/run_algo.py {sssp,pr,bc,tc} [reps] [nsrc]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, '.')
import paper_2305_03317_b200 as sp  # noqa: E402
from paper_2305_03317_b200 import corpus  # noqa: E402

algo = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
nsrc = int(sys.argv[3]) if len(sys.argv) > 3 else 16
if algo == "sssp":
    g = sp.generate("rmat", 16, 16, seed=1)
    prog, args = corpus.SSSP, {"src": 0}
elif algo.startswith("sssp_rmat"):
    g = sp.generate("rmat", int(algo[9:]), 16, seed=1)
    prog, args = corpus.SSSP, {"src": 0}
elif algo == "sssp_grid":
    g = sp.generate("grid", 4096, 4096, seed=1)
    prog, args = corpus.SSSP, {"src": 0}
elif algo.startswith("pr_rmat"):
    g = sp.generate("rmat", int(algo[7:]), 16, seed=1)
    prog, args = corpus.PR, {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
elif algo.startswith("tc_rmat"):
    g = sp.generate("rmat", int(algo[7:]), 16, seed=1, undirected=True)
    prog, args = corpus.TC, {}
elif algo == "pr":
    g = sp.generate("rmat", 22, 16, seed=1)
    prog, args = corpus.PR, {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
elif algo == "bc":
    g = sp.generate("rmat", 20, 16, seed=1, undirected=True)
    deg = np.diff(np.asarray(g.offsets))
    srcs = np.random.default_rng(1).choice(np.flatnonzero(deg > 0), size=256, replace=False)
    prog, args = corpus.BC, {"sourceSet": srcs[:nsrc].tolist()}
elif algo == "bc256":  # the bench's cfg4 line: all 256 sources
    g = sp.generate("rmat", 20, 16, seed=1, undirected=True)
    deg = np.diff(np.asarray(g.offsets))
    srcs = np.random.default_rng(1).choice(np.flatnonzero(deg > 0), size=256, replace=False)
    prog, args = corpus.BC, {"sourceSet": srcs.tolist()}
elif algo == "sssp_grid_pr":
    g = sp.generate("grid", 4096, 4096, seed=1)
    prog, args = corpus.PR, {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
elif algo == "tc":
    g = sp.generate("uniform", 1 << 24, 1 << 28, seed=1, undirected=True)
    prog, args = corpus.TC, {}
nvtx = os.environ.get("SP_NVTX") == "1"  # the last rep inside an NVTX range "steady"
if nvtx:
    import torch
for i in range(reps):
    last = i == reps - 1
    if nvtx and last:
        torch.cuda.nvtx.range_push("steady")
    t0 = time.perf_counter()
    r = sp.run(prog, g, args, device_outputs=True)
    if nvtx and last:
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    print(f"{algo} rep {i}: wall {(time.perf_counter() - t0) * 1e3:.2f} ms, device "
          f"{r.stats['device_ms']:.2f} ms, launches {r.stats['kernel_launches']}, "
          f"edges {r.stats['edges_visited']}, vertices {r.stats['vertices_visited']}, "
          f"iters {r.stats['iterations']}, model bytes {r.stats['model_bytes']}, "
          f"m {g.m}" + (f", triangles {r.env.scalars['triangle_count']}" if prog is corpus.TC else ""),
          flush=True)
