"""Randomised parity sweep (GPU box): random graphs of varied size/density/
direction, every fast form of BC (batched auto / push / pull / per-source),
SSSP push / direction-optimising / pull form, TC row forms, PR -- against
the CPU oracle.  usage: python tools/fuzz_parity.py [cases] [seed]"""
import os
import sys

import numpy as np

sys.path.insert(0, '.')
import paper_2305_03317_b200 as sp  # noqa: E402
from oracle import cpu_ref  # noqa: E402
from paper_2305_03317_b200 import corpus, gen  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
PR = {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}


def rel(a, b):
    b = np.asarray(b, np.float64)
    return float(np.abs(np.asarray(a, np.float64) - b).max(initial=0) /
                 max(np.abs(b).max(initial=0), 1e-300))


def env(**kv):
    for k in ("SP_BC_BATCH", "SP_BC_PULL", "SP_SSSP_DO", "SP_SSSP_PULL_DIV", "SP_TC_WARP_MAX",
              "SP_TC_HASH_MAX", "SP_TC_BIG_MAX"):
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in kv.items()})


fails = 0
for ci in range(cases):
    kind = rng.choice(["rmat", "uniform", "multi"])
    directed = bool(rng.integers(0, 2))
    if kind == "rmat":
        u, v, w, n = gen.rmat(int(rng.integers(8, 14)), int(rng.integers(2, 24)),
                              seed=int(rng.integers(1 << 30)), undirected=not directed)
    elif kind == "uniform":
        n0 = int(rng.integers(50, 5000))
        u, v, w, n = gen.uniform(n0, int(n0 * rng.integers(1, 20)), seed=int(rng.integers(1 << 30)),
                                 undirected=not directed)
    else:
        n = int(rng.integers(20, 2000))
        m = int(n * rng.integers(1, 30))
        u = rng.integers(0, n, m)
        v = rng.integers(0, n, m)
        w = rng.integers(1, 100, m)
        if rng.integers(0, 2) and directed:  # negative weights on a DAG
            keep = u < v
            u, v, w = u[keep], v[keep], w[keep] - 50
    if len(u) == 0:
        continue
    g = sp.from_arrays(u, v, w, directed=directed, n=n)
    o = cpu_ref.build_csr(u, v, w, directed, n)
    tag = f"case {ci}: {kind} n={n} m={g.m} directed={directed}"
    try:
        srcs = rng.integers(0, n, int(rng.integers(1, 30))).tolist()
        bc, sg, dl = cpu_ref.bc(o, srcs, nthreads=8)
        for form in ({}, {"SP_BC_PULL": 0}, {"SP_BC_PULL": 10 ** 12}, {"SP_BC_BATCH": 0}):
            env(**form)
            r = sp.run(corpus.BC, g, {"sourceSet": srcs})
            assert rel(r.env.node_props["bc"], bc) <= 1e-11, ("bc", form)
            assert r.env.node_props["sigma"].tobytes() == sg.tobytes(), ("sigma", form)
            assert rel(r.env.node_props["delta"], dl) <= 1e-11, ("delta", form)
        s = int(rng.integers(0, n))
        dist, _, rc = cpu_ref.sssp(o, s)
        if rc == 0:
            for form in ({}, {"SP_SSSP_DO": 1}, {"SP_SSSP_DO": 1, "SP_SSSP_PULL_DIV": 10 ** 9}):
                env(**form)
                for prog in (corpus.SSSP, corpus.SSSP_PULL):
                    d = sp.run(prog, g, {"src": s}).env.node_props["dist"]
                    assert np.array_equal(d, dist), ("sssp", form)
        env()
        rank, it, diff, its, prc = cpu_ref.pagerank(o, 0.85, 1e-6, 100, cap=10 ** 6, nthreads=8)
        rr = sp.run(corpus.PR, g, PR, max_iters=10 ** 6)
        assert rel(rr.env.node_props["rank"], rank) <= 1e-12 and rr.env.scalars["iter"] == it, "pr"
        if not directed:
            t = cpu_ref.tc(o, nthreads=8)
            for form in ({}, {"SP_TC_WARP_MAX": 8}, {"SP_TC_WARP_MAX": 8, "SP_TC_HASH_MAX": 16},
                         {"SP_TC_WARP_MAX": 8, "SP_TC_HASH_MAX": 16, "SP_TC_BIG_MAX": 32}):
                env(**form)
                gg = sp.from_arrays(u, v, w, directed=False, n=n)  # fresh: upper CSR per form
                assert sp.run(corpus.TC, gg, {}).env.scalars["triangle_count"] == t, ("tc", form)
                gg.close()
        env()
    except AssertionError as e:
        fails += 1
        print("FAIL", tag, e, flush=True)
    g.close()
print(f"fuzz: {cases} cases, {fails} failures", flush=True)
sys.exit(1 if fails else 0)
