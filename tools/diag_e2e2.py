"""e2e PR step (bench's e2e leg) phase by phase, with the library's PR phase
trace (SP_PR_TRACE=1 set by the caller): from_csr, run, close, wall."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2305_03317_b200 as sp  # noqa: E402
from paper_2305_03317_b200 import corpus  # noqa: E402

g = sp.generate("rmat", 22, 16, seed=1)
off = torch.from_numpy(np.array(g.offsets)).pin_memory().numpy()
adj = torch.from_numpy(np.array(g.adj)).pin_memory().numpy()
args = {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
for i in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gg = sp.from_csr(off, adj, None, directed=True)
    t1 = time.perf_counter()
    r = sp.run(corpus.PR, gg, args)
    t2 = time.perf_counter()
    rank = r.env.node_props["rank"]
    assert isinstance(rank, np.ndarray)
    gg.close()
    t3 = time.perf_counter()
    print(f"step {i}: from_csr {1e3 * (t1 - t0):.2f} ms  run {1e3 * (t2 - t1):.2f} ms (device "
          f"{r.stats['device_ms']:.2f})  close {1e3 * (t3 - t2):.2f} ms  total "
          f"{1e3 * (t3 - t0):.2f} ms", file=sys.stderr, flush=True)
