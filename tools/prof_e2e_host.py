"""Host-side profile (cProfile) of the e2e PR step: from_csr -> run -> close (GPU box)."""
import cProfile, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2305_03317_b200 as sp
from paper_2305_03317_b200 import corpus
g = sp.generate("rmat", 22, 16, seed=1)
off = torch.from_numpy(np.array(g.offsets)).pin_memory().numpy()
adj = torch.from_numpy(np.array(g.adj)).pin_memory().numpy()
args = {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
def step():
    gg = sp.from_csr(off, adj, None, directed=True)
    r = sp.run(corpus.PR, gg, args)
    gg.close()
    return r
for _ in range(3): step()
pr = cProfile.Profile(); pr.enable()
for _ in range(5): step()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
