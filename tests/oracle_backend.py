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

    def pr_shard(self, g, v0, v1, damping, deterministic):
        return _OraclePrShard(g, v0, v1, damping)

    # SSSP owner-computes shard (sp_sssp_shard_* semantics)
    def sssp_shard(self, g, src, v0, v1, per, world):
        return _OracleShard(g, src, v0, v1, per, world)


class _OraclePrShard:
    """sp_pagerank_shard_* semantics: left folds in reverse-CSR order."""

    def __init__(self, g, v0, v1, damping):
        self.g, self.v0, self.v1, self.damping = g, v0, v1, damping

    def step(self, contrib_full, rank, contrib, diff):
        g, v0, v1, damping = self.g, self.v0, self.v1, self.damping
        cf = contrib_full.numpy()
        outdeg = np.diff(g.off)
        base = (1.0 - damping) / g.n
        d = 0.0
        for v in range(v0, v1):
            s = 0.0
            for k in range(g.roff[v], g.roff[v + 1]):
                s = s + float(cf[g.radj[k]])
            nr = base + damping * s
            d = max(d, abs(nr - float(rank[v - v0])))
            rank[v - v0] = nr
            contrib[v - v0] = nr / outdeg[v] if outdeg[v] > 0 else 0.0
        diff[0] = d

    def close(self):
        pass


class _OracleShard:
    def __init__(self, g, src, v0, v1, per, world):
        self.g, self.v0, self.v1, self.per, self.world = g, v0, v1, per, world
        self.dist = torch.full((per * world,), INT_MAX, dtype=torch.int32)
        self.dist[src] = 0
        self.q = [src] if v0 <= src < v1 else []
        self.send = torch.zeros(max(1, g.n), dtype=torch.int64)

    def relax(self, max_rounds):
        g, d = self.g, self.dist.numpy()
        out = set()
        upd = rel = rounds = 0
        while self.q and rounds < max_rounds:
            nxt = []
            seen = set()
            for v in self.q:
                dv = int(d[v])
                for e in range(g.off[v], g.off[v + 1]):
                    rel += 1
                    x = int(g.adj[e])
                    cand = dv + int(g.weff[e])
                    if cand >= INT_MAX or cand >= d[x]:
                        continue
                    if cand < -2 ** 31:
                        raise OverflowError("int32 underflow")
                    d[x] = cand
                    if self.v0 <= x < self.v1:
                        if x not in seen:
                            seen.add(x)
                            nxt.append(x)
                    else:
                        out.add(x)
            self.q = nxt
            upd += len(nxt)
            rounds += 1
        ids = sorted(out, key=lambda x: x // self.per)
        counts = np.zeros(self.world, dtype=np.int64)
        for i, x in enumerate(ids):
            counts[x // self.per] += 1
            self.send[i] = (x << 32) | (int(d[x]) & 0xffffffff)
        return counts, np.array([upd, rel, rounds, len(self.q)], dtype=np.int64)

    def apply(self, msgs=None, k=0, block=None):
        d = self.dist.numpy()
        seen = set(self.q)
        if block is not None:
            b = block.numpy()
            for v in range(self.v0, self.v1):
                if b[v - self.v0] < d[v]:
                    d[v] = b[v - self.v0]
                    if v not in seen:
                        seen.add(v)
                        self.q.append(v)
        else:
            for m in (msgs[:k].tolist() if k else []):
                x = m >> 32
                c = ((m & 0xffffffff) ^ 0x80000000) - 0x80000000
                if c < d[x]:
                    d[x] = c
                    if x not in seen:
                        seen.add(x)
                        self.q.append(x)
        return len(self.q)

    def result(self):
        return self.dist.numpy()[: self.g.n]

    def close(self):
        pass
