#!/usr/bin/env python3
"""Generate tests/golden/weights/*.npz with the PYTHON REFERENCE's own
trident.graph.assign_random_weights (graph.py:154-190).

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_weights_golden.py [--ref /root/reference/pkg/src]

Graphs: directed and undirected multigraphs with parallel edges and
self-loops (the cases the mirror-by-position rule exists for), a corpus
fixture and a seeded RMAT graph; several (lo, hi, seed) triples each.
"""

from __future__ import annotations

import argparse
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)


def multigraph(n, ne, seed):
    r = random.Random(seed)
    edges = []
    for _ in range(ne):
        u, v = r.randrange(n), r.randrange(n)
        edges.append((u, v, 1))
        if r.random() < 0.2:  # a parallel copy
            edges.append((u, v, 1))
    edges += [(3, 3, 1), (3, 3, 1)]  # self-loops, stored once per copy (F9)
    return edges


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    a = ap.parse_args()
    sys.path.insert(0, a.ref)
    from trident.graph import assign_random_weights, from_edges

    from paper_2305_03317_b200 import gen

    u, v, _, n = gen.rmat(9, 8, seed=3)
    cases = {
        "multi60": multigraph(60, 400, 1),
        "multi300": multigraph(300, 3000, 2),
        "k5": [(i, j, 1) for i in range(5) for j in range(5) if i < j],
        "rmat9": list(zip(u.tolist(), v.tolist(), [1] * len(u))),
    }
    out = os.path.join(HERE, "weights")
    os.makedirs(out, exist_ok=True)
    for name, edges in cases.items():
        for directed in (True, False):
            g = from_edges(edges, directed=directed)
            for lo, hi, seed in ((1, 100, 7), (-5, 5, 0), (1, 1 << 30, 123)):
                w = assign_random_weights(g, lo, hi, seed).weights
                tag = f"{name}_{'d' if directed else 'u'}_{seed}"
                np.savez_compressed(os.path.join(out, tag + ".npz"),
                                    off=np.asarray(g.offsets, np.int64),
                                    adj=np.asarray(g.adj, np.int32),
                                    directed=directed, lo=lo, hi=hi, seed=seed,
                                    w=np.asarray(w, np.int64))
                print(tag, g.n, g.m)


if __name__ == "__main__":
    main()
