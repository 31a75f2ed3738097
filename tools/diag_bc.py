import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2305_03317_b200 as sp
from paper_2305_03317_b200 import corpus
g = sp.generate("rmat", 20, 16, seed=1, undirected=True)
deg = np.diff(np.asarray(g.offsets))
srcs = np.random.default_rng(1).choice(np.flatnonzero(deg > 0), size=256, replace=False).tolist()
for dev in (False, True, False):
    for k in (1, 4, 16):
        t0 = time.perf_counter()
        r = sp.run(corpus.BC, g, {"sourceSet": srcs[:k]}, device_outputs=dev)
        print(dev, k, f"wall {(time.perf_counter()-t0)*1e3:.1f} dev {r.stats['device_ms']:.1f} launches {r.stats['kernel_launches']} levels {r.stats['iterations']}", flush=True)
