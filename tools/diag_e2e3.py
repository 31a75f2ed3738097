"""Where the e2e PR step's run() time goes outside the kernels (GPU box)."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2305_03317_b200 as sp  # noqa: E402
from paper_2305_03317_b200 import _lib, corpus, interp  # noqa: E402

g = sp.generate("rmat", 22, 16, seed=1)
off = torch.from_numpy(np.array(g.offsets)).pin_memory().numpy()
adj = torch.from_numpy(np.array(g.adj)).pin_memory().numpy()
args = {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
L = _lib.lib()
for i in range(6):
    gg = sp.from_csr(off, adj, None, directed=True)
    t0 = time.perf_counter()
    rank, mem = interp._out(gg.n, np.float64, None)
    t1 = time.perf_counter()
    it, its, diff, st = C.c_int64(), C.c_int64(), C.c_double(), _lib.Stats()
    rc = L.sp_pagerank(gg.handle, 0.85, 1e-6, 100, 2 * gg.n + 16, 0, interp._ptr(rank), mem,
                       C.byref(it), C.byref(diff), C.byref(its), _lib.ITER_CB(), None, C.byref(st))
    t2 = time.perf_counter()
    cp = interp._host_copy(rank)
    t3 = time.perf_counter()
    r = sp.run(corpus.PR, gg, args)
    t4 = time.perf_counter()
    gg.close()
    print(f"step {i}: _out {1e3*(t1-t0):.2f}  sp_pagerank {1e3*(t2-t1):.2f} (device "
          f"{st.device_ms:.2f})  _host_copy {1e3*(t3-t2):.2f}  full run() {1e3*(t4-t3):.2f} ms",
          flush=True)
