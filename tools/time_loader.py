"""Time load_edge_list (native multithreaded parser + device CSR build) on a
generated RMAT edge-list file (GPU box diagnostic)."""
import os
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_2305_03317_b200 as sp  # noqa: E402
from paper_2305_03317_b200 import gen  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
u, v, w, n = gen.rmat(scale, 16, seed=1)
path = f"/tmp/rmat{scale}.txt"
t0 = time.perf_counter()
np.savetxt(path, np.stack([u, v, w], axis=1), fmt="%d")
print(f"wrote {len(u)} lines, {os.path.getsize(path) / 1e6:.0f} MB in "
      f"{time.perf_counter() - t0:.1f} s", flush=True)
for i in range(3):
    t0 = time.perf_counter()
    g = sp.load_edge_list(path)
    dt = time.perf_counter() - t0
    print(f"load_edge_list: {dt * 1e3:.1f} ms, {len(u) / dt / 1e6:.1f} M edges/s, "
          f"n={g.n} m={g.m}", flush=True)
    g.close()
