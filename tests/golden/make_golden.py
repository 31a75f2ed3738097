#!/usr/bin/env python3
"""Generate tests/golden/*.npz by running the PYTHON REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

For every case it records the reference's own outputs:
  * CSR arrays of trident.graph.from_edges / load_edge_list (graph.py:68-151)
  * trident.interp.run on corpus/programs/{sssp,pr,bc,tc}.sp
    (dist + fixedpoint iterations; rank/iter/diff; bc/sigma/delta; count),
    including NonConvergenceError (flag, cap) where the default cap trips
    (SURVEY F5), in which case the values come from a rerun with a large cap.
Cases: the 14 corpus fixture graphs x {directed, undirected} plus seeded
RMAT / uniform / grid graphs from paper_2305_03317_b200.gen.

These vectors pin the CPU oracle (oracle/cpu_ref.c) and, through it, the GPU
path.  The script is the only code in the repo that imports the reference.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

FIXTURES = ["path3", "path10", "cycle3", "cycle4", "cycle10", "star13", "k3",
            "k4", "k5", "isolated4", "rand200_a", "rand200_b", "rand50_u",
            "grid5x5"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    sys.path.insert(0, a.ref)
    from trident.errors import NonConvergenceError
    from trident.graph import from_edges, load_edge_list
    from trident.interp import run
    from trident.parser import parse_source
    from trident.sema import analyze

    from paper_2305_03317_b200 import gen

    corpus = os.path.join(a.ref, "trident", "corpus")
    progs = {}
    for name in ("sssp", "pr", "bc", "tc", "sssp_pull"):
        with open(os.path.join(corpus, "programs", name + ".sp")) as f:
            progs[name] = analyze(parse_source(f.read()))

    def record(case, g, u, v, w, directed, sssp_srcs, bc_srcs, do_tc=True):
        out = dict(u=np.asarray(u, np.int32), v=np.asarray(v, np.int32),
                   w=np.asarray(w, np.int32), n=g.n, directed=directed,
                   csr_off=np.asarray(g.offsets, np.int64),
                   csr_adj=np.asarray(g.adj, np.int32),
                   csr_w=np.asarray(g.weights, np.int32),
                   csr_roff=np.asarray(g.rev_offsets, np.int64),
                   csr_radj=np.asarray(g.rev_adj, np.int32),
                   csr_reid=np.asarray(g.rev_eid, np.int64))
        t0 = time.time()
        out["sssp_srcs"] = np.asarray(sssp_srcs, np.int32)
        dists, its = [], []
        for s in sssp_srcs:
            r = run(progs["sssp"], g, {"src": s})
            dists.append(np.asarray(r.env.node_props["dist"], np.int64))
            its.append(r.fixedpoint_iterations["finished"])
            rp = run(progs["sssp_pull"], g, {"src": s})
            assert rp.env.node_props["dist"] == r.env.node_props["dist"]
        out["sssp_dist"] = np.stack(dists) if dists else np.zeros((0, g.n))
        out["sssp_iters"] = np.asarray(its, np.int64)
        prargs = {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
        try:
            r = run(progs["pr"], g, prargs)
            out["pr_err_cap"] = -1
        except NonConvergenceError as e:
            assert e.flag == "converged"
            out["pr_err_cap"] = e.cap
            r = run(progs["pr"], g, prargs, max_iters=10 ** 6)
        out["pr_rank"] = np.asarray(r.env.node_props["rank"], np.float64)
        out["pr_rank_nxt"] = np.asarray(r.env.node_props["rank_nxt"], np.float64)
        out["pr_iter"] = r.env.scalars["iter"]
        out["pr_diff"] = r.env.scalars["diff"]
        out["pr_iters"] = r.fixedpoint_iterations["converged"]
        out["bc_srcs"] = np.asarray(bc_srcs, np.int32)
        r = run(progs["bc"], g, {"sourceSet": list(bc_srcs)})
        out["bc"] = np.asarray(r.env.node_props["bc"], np.float64)
        if bc_srcs:
            out["bc_sigma"] = np.asarray(r.env.node_props["sigma"], np.float64)
            out["bc_delta"] = np.asarray(r.env.node_props["delta"], np.float64)
        if do_tc:
            r = run(progs["tc"], g, {})
            out["tc"] = int(r.env.scalars["triangle_count"])
        np.savez_compressed(os.path.join(HERE, case + ".npz"), **out)
        print(f"{case}: n={g.n} m={g.m} {time.time() - t0:.1f}s", flush=True)

    for fx in FIXTURES:
        path = os.path.join(corpus, "graphs", fx + ".txt")
        for directed in (True, False):
            case = f"fx_{fx}_{'d' if directed else 'u'}"
            if a.only and a.only not in case:
                continue
            g = load_edge_list(path, directed=directed)
            # raw edge triples in file order, as from_edges saw them
            u, v, w = [], [], []
            with open(path) as f:
                for line in f:
                    s = line.strip()
                    if not s or s.startswith("#"):
                        continue
                    p = s.split()
                    u.append(int(p[0])); v.append(int(p[1]))
                    w.append(int(p[2]) if len(p) == 3 else 1)
            srcs = [0] if g.n <= 1 else [0, g.n - 1]
            bcs = list(range(min(g.n, 40))) + ([0] if g.n else [])
            record(case, g, u, v, w, directed, srcs, bcs)

    synth = [
        ("syn_rmat10_d", lambda: gen.rmat(10, 16, seed=1), True, [0, 5], [0, 1, 2, 3, 7, 0]),
        ("syn_rmat10_u", lambda: gen.rmat(10, 8, seed=2, undirected=True), False, [0], [0, 9, 17, 33, 65, 129, 9]),
        ("syn_unif1k_u", lambda: gen.uniform(1024, 8192, seed=3), False, [0, 100], [0, 1, 2, 3]),
        ("syn_unif2k_d", lambda: gen.uniform(2048, 16384, seed=4, undirected=False), True, [0], [5, 6]),
        ("syn_grid16_u", lambda: gen.grid(16, 16, seed=5), False, [0, 255], [0, 136, 255]),
    ]
    for case, mk, directed, srcs, bcs in synth:
        if a.only and a.only not in case:
            continue
        u, v, w, n = mk()
        edges = list(zip(u.tolist(), v.tolist(), w.tolist()))
        g = from_edges(edges, directed=directed, n=n)
        record(case, g, u, v, w, directed, srcs, bcs)


if __name__ == "__main__":
    main()
