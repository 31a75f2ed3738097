"""from_csr phase profile (GPU box): pinned host CSR -> device graph, 4 calls."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2305_03317_b200 as sp  # noqa: E402

g = sp.generate("rmat", 22, 16, seed=1)
off = torch.from_numpy(np.array(g.offsets)).pin_memory().numpy()
adj = torch.from_numpy(np.array(g.adj)).pin_memory().numpy()
g.close()
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gg = sp.from_csr(off, adj, None, directed=True)
    t1 = time.perf_counter()
    gg.close()
    print(f"from_csr {1e3 * (t1 - t0):.2f} ms", flush=True)
