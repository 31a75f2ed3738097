"""CPU stand-in for parallel.NativeBackend (TEST INFRASTRUCTURE ONLY).

Runs the per-rank compute of paper_2305_03317_b200.parallel on host numpy /
torch CPU tensors with the semantics of the native block kernels, so that the
sharding, exchange and convergence logic of parallel.py can be exercised on
gloo with world_size > 1 in a container without a GPU.  Whole-program
results are checked against the single-process oracle (oracle/cpu_ref).
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import cpu_ref

INT_MAX = 2147483647


class OracleBackend:
    torch = torch

    def __init__(self):
        self.device = torch.device("cpu")

    def graph(self, g):
        return g  # an oracle Csr

    def offsets(self, g):
        return g.off

    def to_host(self, x):
        return x.numpy()

    # BC: the oracle run over this rank's sources
    def bc(self, g, srcs, deterministic):
        if len(srcs):
            b, sg, dl = cpu_ref.bc(g, srcs)
        else:
            b = np.zeros(g.n)
            sg = np.zeros(g.n)
            dl = np.zeros(g.n)
        return torch.from_numpy(b), torch.from_numpy(sg), torch.from_numpy(dl)

    # TC share with the native range semantics (see include/starplat_b200.h)
    def tc(self, g, v0, v1) -> int:
        off, adj = g.off, g.adj
        cnt = 0
        if g.directed:
            for v in range(v0, v1):
                row = adj[off[v]:off[v + 1]]
                us = [u for u in row if u < v]
                ws = [w for w in row if w > v]
                for u in us:
                    nu = adj[off[u]:off[u + 1]]
                    for w in ws:
                        cnt += int(np.count_nonzero(nu == w))
            return cnt
        deg = np.diff(off)

        def up(a):
            return [x for x in adj[off[a]:off[a + 1]]
                    if x != a and (deg[x], x) > (deg[a], a)]
        for a in range(v0, v1):
            A = up(a)
            for b in A:
                for x in up(b):
                    cnt += A.count(x)
        return cnt

    # PR block step, left folds in reverse-CSR order (bit-exact mode)
    def pr_init(self, g, v0, v1):
        n = g.n
        outdeg = np.diff(g.off)
        r0 = 1.0 / n
        rank = np.full(max(1, v1 - v0), r0)
        contrib = np.array([r0 / outdeg[v] if outdeg[v] > 0 else 0.0 for v in range(v0, v1)]
                           + [0.0] * (1 if v1 == v0 else 0))
        return torch.from_numpy(rank), torch.from_numpy(contrib)

    def pr_step(self, g, v0, v1, damping, contrib_full, rank, contrib, deterministic):
        n = g.n
        cf = contrib_full.numpy()
        outdeg = np.diff(g.off)
        base = (1.0 - damping) / n
        d = 0.0
        for v in range(v0, v1):
            s = 0.0
            for k in range(g.roff[v], g.roff[v + 1]):
                s = s + float(cf[g.radj[k]])
            nr = base + damping * s
            dd = abs(nr - float(rank[v - v0]))
            d = max(d, dd)
            rank[v - v0] = nr
            contrib[v - v0] = nr / outdeg[v] if outdeg[v] > 0 else 0.0
        return d

    # SSSP supersteps
    def sssp_init(self, g, src):
        dist = np.full(max(1, g.n), INT_MAX, dtype=np.int32)
        dist[src] = 0
        last = np.full(max(1, g.n), INT_MAX, dtype=np.int32)
        return torch.from_numpy(dist), torch.from_numpy(last)

    def sssp_step(self, g, v0, v1, dist, last):
        d = dist.numpy()
        ls = last.numpy()
        F = [v for v in range(v0, v1) if d[v] < ls[v]]
        relaxed = 0
        for v in F:
            ls[v] = d[v]
        for v in F:
            for e in range(g.off[v], g.off[v + 1]):
                relaxed += 1
                x = g.adj[e]
                cand = int(d[v]) + int(g.weff[e])
                if cand < INT_MAX and cand < d[x]:
                    if cand < -2 ** 31:
                        raise OverflowError("int32 underflow")
                    d[x] = cand
        return len(F), relaxed
