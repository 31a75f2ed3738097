"""GPU parity: libstarplat_b200.so (through the drop-in host layer and its C
ABI) against the golden vectors of the Python reference and against the
CPU oracle (oracle/cpu_ref.c, itself pinned bit-exact to the reference in
test_oracle_golden.py).

Tolerances:
  SSSP dist, TC count, CSR arrays: bit-exact.
  PR deterministic mode: bit-exact ranks, same iter and diff.
  PR fast mode: |d|_inf / |ref|_inf <= 1e-12 (hub rows use a tree order),
     same iteration count.
  BC deterministic mode: bit-exact bc/sigma/delta; fast mode <= 1e-12.
"""

import numpy as np
import pytest

from conftest import golden_cases, load_golden
from oracle import cpu_ref

pytestmark = pytest.mark.gpu

sp = pytest.importorskip("paper_2305_03317_b200")
from paper_2305_03317_b200 import corpus, gen  # noqa: E402
from paper_2305_03317_b200.errors import (ExecError,  # noqa: E402
                                          NonConvergenceError)

CASES = golden_cases()
PR_ARGS = {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = max(np.abs(b).max(initial=0.0), 1e-300)
    return float(np.abs(a - b).max(initial=0.0) / den)


def _graph(z):
    return sp.from_arrays(z["u"], z["v"], z["w"], directed=bool(z["directed"]),
                          n=int(z["n"]))


@pytest.fixture(scope="module")
def graphs():
    cache = {}

    def get(case):
        if case not in cache:
            z = load_golden(case)
            cache[case] = (z, _graph(z))
        return cache[case]
    return get


@pytest.mark.parametrize("case", CASES)
def test_csr_build(case, graphs):
    z, g = graphs(case)
    assert g.n == int(z["n"]) and g.m == len(z["csr_adj"])
    np.testing.assert_array_equal(g.offsets, z["csr_off"])
    np.testing.assert_array_equal(g.adj, z["csr_adj"])
    np.testing.assert_array_equal(g.weights, z["csr_w"])
    np.testing.assert_array_equal(g.rev_offsets, z["csr_roff"])
    np.testing.assert_array_equal(g.rev_adj, z["csr_radj"])
    np.testing.assert_array_equal(g.rev_eid, z["csr_reid"])
    o = cpu_ref.build_csr(z["u"], z["v"], z["w"], bool(z["directed"]), int(z["n"]))
    np.testing.assert_array_equal(g.effective_weights, o.weff)


@pytest.mark.parametrize("case", CASES)
def test_sssp(case, graphs):
    z, g = graphs(case)
    for i, s in enumerate(z["sssp_srcs"]):
        for prog in (corpus.SSSP, corpus.SSSP_PULL):
            r = sp.run(prog, g, {"src": int(s)})
            np.testing.assert_array_equal(r.env.node_props["dist"].astype(np.int64),
                                          z["sssp_dist"][i])
            assert r.env.scalars == {"finished": True}
            assert not r.env.node_props["modified"].any()
            assert r.fixedpoint_iterations["finished"] >= 1


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("det", [True, False])
def test_pagerank(case, det, graphs):
    z, g = graphs(case)
    cap = int(z["pr_err_cap"])
    if cap >= 0:
        with pytest.raises(NonConvergenceError) as ei:
            sp.run(corpus.PR, g, PR_ARGS, deterministic=det)
        assert ei.value.flag == "converged" and ei.value.cap == cap
        r = sp.run(corpus.PR, g, PR_ARGS, max_iters=10 ** 6, deterministic=det)
    else:
        r = sp.run(corpus.PR, g, PR_ARGS, deterministic=det)
    rank = r.env.node_props["rank"]
    assert r.env.scalars["iter"] == int(z["pr_iter"])
    assert r.fixedpoint_iterations["converged"] == int(z["pr_iters"])
    if det:
        assert rank.tobytes() == z["pr_rank"].tobytes()
        assert r.env.scalars["diff"] == float(z["pr_diff"])
    else:
        assert rel_err(rank, z["pr_rank"]) <= 1e-12
    np.testing.assert_array_equal(r.env.node_props["rank_nxt"], rank)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("det", [True, False])
def test_bc(case, det, graphs):
    z, g = graphs(case)
    srcs = z["bc_srcs"].tolist()
    r = sp.run(corpus.BC, g, {"sourceSet": srcs}, deterministic=det)
    bc = r.env.node_props["bc"]
    if det:
        assert bc.tobytes() == z["bc"].tobytes()
        assert r.env.node_props["sigma"].tobytes() == z["bc_sigma"].tobytes()
        assert r.env.node_props["delta"].tobytes() == z["bc_delta"].tobytes()
    else:
        assert rel_err(bc, z["bc"]) <= 1e-12


@pytest.mark.parametrize("case", CASES)
def test_tc(case, graphs):
    z, g = graphs(case)
    r = sp.run(corpus.TC, g, {})
    assert r.env.scalars == {"triangle_count": int(z["tc"])}


# ---------------------------------------------------------------------------
# device generators == host generators (same edge lists -> same CSR)

@pytest.mark.parametrize("kind,p0,p1,undirected", [
    ("rmat", 10, 16, False), ("rmat", 12, 8, True), ("uniform", 5000, 40000, True),
    ("uniform", 3000, 20000, False), ("grid", 17, 23, True)])
def test_device_generator_matches_host(kind, p0, p1, undirected):
    if kind == "rmat":
        u, v, w, n = gen.rmat(p0, p1, seed=3, undirected=undirected)
    elif kind == "uniform":
        u, v, w, n = gen.uniform(p0, p1, seed=3, undirected=undirected)
    else:
        u, v, w, n = gen.grid(p0, p1, seed=3)
    gh = sp.from_arrays(u, v, w, directed=not undirected, n=n)
    gd = sp.generate(kind, p0, p1, seed=3, undirected=undirected)
    assert (gd.n, gd.m, gd.directed) == (gh.n, gh.m, gh.directed)
    np.testing.assert_array_equal(gd.offsets, gh.offsets)
    np.testing.assert_array_equal(gd.adj, gh.adj)
    np.testing.assert_array_equal(gd.weights, gh.weights)


# ---------------------------------------------------------------------------
# larger seeded graphs against the CPU oracle

def _pair(kind, p0, p1, seed, undirected):
    if kind == "rmat":
        u, v, w, n = gen.rmat(p0, p1, seed=seed, undirected=undirected)
    elif kind == "uniform":
        u, v, w, n = gen.uniform(p0, p1, seed=seed, undirected=undirected)
    else:
        u, v, w, n = gen.grid(p0, p1, seed=seed)
    return (sp.from_arrays(u, v, w, directed=not undirected, n=n),
            cpu_ref.build_csr(u, v, w, not undirected, n))


def test_sssp_cfg1_rmat16_bit_exact():
    """BASELINE cfg1: SSSP from 0 on weighted RMAT-16 (directed)."""
    g, o = _pair("rmat", 16, 16, 1, False)
    r = sp.run(corpus.SSSP, g, {"src": 0})
    dist, _, rc = cpu_ref.sssp(o, 0)
    assert rc == 0
    np.testing.assert_array_equal(r.env.node_props["dist"], dist)


@pytest.mark.parametrize("kind,p0,p1,und", [("rmat", 14, 16, False), ("grid", 64, 64, True),
                                            ("uniform", 1 << 14, 1 << 17, True)])
def test_sssp_seeded(kind, p0, p1, und):
    g, o = _pair(kind, p0, p1, 11, und)
    for s in (0, g.n // 2):
        dist, _, rc = cpu_ref.sssp(o, s)
        for prog in (corpus.SSSP, corpus.SSSP_PULL):  # push and pull forms
            r = sp.run(prog, g, {"src": s})
            np.testing.assert_array_equal(r.env.node_props["dist"], dist)


@pytest.mark.parametrize("packed", ["1", "0"])
@pytest.mark.parametrize("kind,p0,p1,und", [("rmat", 16, 16, False), ("rmat", 12, 48, True),
                                            ("uniform", 1 << 12, 1 << 17, False)])
def test_sssp_packed_words(kind, p0, p1, und, packed, monkeypatch):
    """Bellman-Ford device loop with (dist, enqueue stamp) packed in one
    64-bit word per vertex (one atomicMin relaxes and dedupes the next
    frontier; the default) and with separate dist / enq arrays
    (SP_SSSP_PACKED=0): the oracle's dist bit for bit, from several sources
    including the largest hub, repeated (the atomics' order is racy)."""
    monkeypatch.setenv("SP_SSSP_PACKED", packed)
    monkeypatch.setenv("SP_SSSP_DELTA", "0")  # Bellman-Ford even on thin graphs
    g, o = _pair(kind, p0, p1, 31, und)
    deg = np.diff(np.asarray(g.offsets))
    hub = int(np.argmax(deg))
    for s in (0, hub, g.n // 2):
        dist, _, rc = cpu_ref.sssp(o, s)
        assert rc == 0
        for rep in range(3):
            r = sp.run(corpus.SSSP, g, {"src": s})
            np.testing.assert_array_equal(r.env.node_props["dist"], dist, err_msg=f"rep {rep}")
            assert not r.env.node_props["modified"].any()


@pytest.mark.parametrize("kind,p0,p1,und,delta", [
    ("grid", 300, 280, True, None), ("grid", 512, 512, True, "40"), ("grid", 97, 1031, True, None),
    ("uniform", 1 << 16, 1 << 18, True, None), ("uniform", 1 << 16, 1 << 18, False, "7"),
    ("grid", 64, 64, True, "0")])
def test_sssp_async_near_far_stress(kind, p0, p1, und, delta, monkeypatch):
    """The asynchronous near-far loop (thin graphs, non-negative weights, no
    caller cap): per-block rings, in-queue flags, phase splits -- racy by
    design, so every graph runs several times, with small and large delta
    (many / few phases; "0" = Bellman-Ford, the reference form), against
    the oracle's dist bit for bit; the 1-hop row form (SP_NF_SHORTCUT=0; the
    default relaxes 2-hop shortcut rows on out-degree <= 4 graphs) and the
    synchronous near-far kernel (SP_NF_ASYNC=0) give the same dist."""
    if delta is not None:
        monkeypatch.setenv("SP_SSSP_DELTA", delta)
    g, o = _pair(kind, p0, p1, 23, und)
    for s in (0, g.n // 3):
        dist, _, rc = cpu_ref.sssp(o, s)
        assert rc == 0
        for rep in range(4):
            r = sp.run(corpus.SSSP, g, {"src": s})
            np.testing.assert_array_equal(r.env.node_props["dist"], dist, err_msg=f"rep {rep}")
    monkeypatch.setenv("SP_NF_SHORTCUT", "0")  # 1-hop ELL rows (default: 2-hop shortcut rows)
    for rep in range(2):
        r = sp.run(corpus.SSSP, g, {"src": 0})
        np.testing.assert_array_equal(r.env.node_props["dist"], cpu_ref.sssp(o, 0)[0])
    monkeypatch.delenv("SP_NF_SHORTCUT")
    monkeypatch.setenv("SP_NF_ASYNC_RING", "64")  # rings overflow: the synchronous fallback
    r = sp.run(corpus.SSSP, g, {"src": 0})
    np.testing.assert_array_equal(r.env.node_props["dist"], cpu_ref.sssp(o, 0)[0])
    monkeypatch.delenv("SP_NF_ASYNC_RING")
    monkeypatch.setenv("SP_NF_ASYNC", "0")
    r = sp.run(corpus.SSSP, g, {"src": 0})
    np.testing.assert_array_equal(r.env.node_props["dist"], cpu_ref.sssp(o, 0)[0])


@pytest.mark.parametrize("directed", [True, False])
def test_sssp_shortcut_rows_random_low_degree(directed, monkeypatch):
    """The asynchronous kernel's 2-hop shortcut rows on a random graph of
    out-degree <= 4 (rows with more than 12 distinct 1-2-hop targets keep
    the 1-hop ones and the first 2-hop ones), with self-loops, parallel
    edges and zero weights: the oracle's dist bit for bit, also against the
    1-hop rows (SP_NF_SHORTCUT=0)."""
    rng = np.random.default_rng(41)
    n = 20000
    deg = rng.integers(0, 5, n)
    u = np.repeat(np.arange(n), deg)
    v = rng.integers(0, n, len(u))
    loops = rng.random(len(u)) < 0.01
    v[loops] = u[loops]
    w = rng.integers(0, 60, len(u))
    dup = rng.random(len(u)) < 0.02
    u = np.concatenate([u, u[dup]])
    v = np.concatenate([v, v[dup]])
    w = np.concatenate([w, w[dup] + 3])
    # every row <= 4 slots (undirected: both mirrors count; a self-loop once, F9)
    cnt = np.zeros(n, dtype=np.int64)
    keep = np.zeros(len(u), dtype=bool)
    for i in range(len(u)):
        a, b = int(u[i]), int(v[i])
        if cnt[a] + 1 <= 4 and (directed or a == b or cnt[b] + 1 <= 4):
            keep[i] = True
            cnt[a] += 1
            if not directed and a != b:
                cnt[b] += 1
    u, v, w = u[keep], v[keep], w[keep]
    g = sp.from_arrays(u, v, w, directed=directed, n=n)
    assert np.diff(np.asarray(g.offsets)).max() <= 4  # the shortcut-row form applies
    o = cpu_ref.build_csr(u, v, w, directed, n)
    for s in (0, n // 2, int(np.argmax(np.bincount(u, minlength=n)))):
        dist, _, rc = cpu_ref.sssp(o, s)
        assert rc == 0
        for form in ("2", "0"):
            monkeypatch.setenv("SP_NF_SHORTCUT", form)
            for rep in range(2):
                r = sp.run(corpus.SSSP, g, {"src": s})
                np.testing.assert_array_equal(r.env.node_props["dist"], dist,
                                              err_msg=f"form {form} rep {rep}")


@pytest.mark.parametrize("pull_div", ["8", "1"])
def test_sssp_pull_hot_snapshot(pull_div, monkeypatch):
    """Direction-optimising SSSP whose pull sweeps read the hottest sources'
    dist from a shared-memory snapshot (SP_SSSP_HOT=1: from the first run;
    RMAT-20 qualifies for the hot encoding): the oracle's dist bit for bit,
    from several sources, also with every iteration after the first a
    sweep (pull_div 1)."""
    monkeypatch.setenv("SP_SSSP_DO", "1")
    monkeypatch.setenv("SP_SSSP_HOT", "1")
    monkeypatch.setenv("SP_SSSP_PULL_DIV", pull_div)
    g, o = _pair("rmat", 20, 16, 29, False)
    for s in (0, 7, g.n // 2):
        dist, _, rc = cpu_ref.sssp(o, s)
        assert rc == 0
        r = sp.run(corpus.SSSP, g, {"src": s})
        np.testing.assert_array_equal(r.env.node_props["dist"], dist)
        r = sp.run(corpus.SSSP_PULL, g, {"src": s})
        np.testing.assert_array_equal(r.env.node_props["dist"], dist)


@pytest.mark.parametrize("pull_div", ["8", "1000000"])
@pytest.mark.parametrize("graph", ["rmat_dir", "rmat_sym", "hub", "multi", "neg_dag"])
def test_sssp_direction_optimising(graph, pull_div, monkeypatch):
    """Push-form SSSP through the direction-optimising loop (the default from
    2^27 slots; forced here): push iterations, edge-balanced pull sweeps for
    large frontiers (pull_div 8) or for every frontier after the root
    (pull_div huge), spill rows across units, negative weights -- the
    oracle's dist bit for bit."""
    monkeypatch.setenv("SP_SSSP_DO", "1")
    monkeypatch.setenv("SP_SSSP_PULL_DIV", pull_div)
    if graph.startswith("rmat"):
        u, v, w, n = gen.rmat(13, 16, seed=17, undirected=graph == "rmat_sym")
        directed = graph == "rmat_dir"
    elif graph == "hub":
        u, v, w, n = _hub_graph(True)
        directed = True
    elif graph == "multi":
        u, v, w, n = _multigraph(6)
        directed = True
    else:
        u, v, w, n = _multigraph(5, neg=True)
        directed = True
    g = sp.from_arrays(u, v, w, directed=directed, n=n)
    o = cpu_ref.build_csr(u, v, w, directed, n)
    for s in (int(u[0]), 0):
        dist, _, rc = cpu_ref.sssp(o, s)
        assert rc == 0
        r = sp.run(corpus.SSSP, g, {"src": s})
        np.testing.assert_array_equal(r.env.node_props["dist"], dist)


@pytest.mark.parametrize("kind,p0,p1,und", [("rmat", 14, 16, False), ("rmat", 13, 16, True),
                                            ("grid", 32, 32, True), ("rmat", 16, 16, False)])
def test_pagerank_seeded(kind, p0, p1, und):
    g, o = _pair(kind, p0, p1, 5, und)
    rank, it, diff, its, rc = cpu_ref.pagerank(o, 0.85, 1e-6, 100, cap=10 ** 6, nthreads=4)
    rd = sp.run(corpus.PR, g, PR_ARGS, max_iters=10 ** 6, deterministic=True)
    assert rd.env.node_props["rank"].tobytes() == rank.tobytes()
    assert rd.env.scalars["iter"] == it and rd.env.scalars["diff"] == diff
    rf = sp.run(corpus.PR, g, PR_ARGS, max_iters=10 ** 6)
    assert rel_err(rf.env.node_props["rank"], rank) <= 1e-12
    assert rf.env.scalars["iter"] == it


@pytest.mark.parametrize("und", [False, True])
def test_pagerank_hot_source_path(und, monkeypatch):
    """PR's hot-source variant (the top out-degree sources' contribs in
    shared memory, built on a graph's second fast call) gives the plain
    kernel's bits; forced on with SP_PR_HOT_COVER=0 on RMAT-17."""
    monkeypatch.setenv("SP_PR_HOT_COVER", "0")
    g, o = _pair("rmat", 17, 16, 3, und)
    rank, it, diff, its, rc = cpu_ref.pagerank(o, 0.85, 1e-6, 100, cap=10 ** 6, nthreads=4)
    r1 = sp.run(corpus.PR, g, PR_ARGS)   # plain kernel
    r2 = sp.run(corpus.PR, g, PR_ARGS)   # hot-source kernel
    assert r2.env.node_props["rank"].tobytes() == r1.env.node_props["rank"].tobytes()
    assert rel_err(r2.env.node_props["rank"], rank) <= 1e-12
    assert r1.env.scalars["iter"] == r2.env.scalars["iter"] == it


@pytest.mark.parametrize("kind,p0,p1,und", [("rmat", 13, 16, True), ("rmat", 12, 16, False),
                                            ("grid", 40, 40, True)])
def test_bc_seeded(kind, p0, p1, und):
    g, o = _pair(kind, p0, p1, 7, und)
    rng = np.random.default_rng(1)
    srcs = rng.choice(g.n, size=6, replace=False).tolist() + [0]
    bc, sg, dl = cpu_ref.bc(o, srcs, nthreads=4)
    rd = sp.run(corpus.BC, g, {"sourceSet": srcs}, deterministic=True)
    assert rd.env.node_props["bc"].tobytes() == bc.tobytes()
    assert rd.env.node_props["sigma"].tobytes() == sg.tobytes()
    assert rd.env.node_props["delta"].tobytes() == dl.tobytes()
    rf = sp.run(corpus.BC, g, {"sourceSet": srcs})
    assert rel_err(rf.env.node_props["bc"], bc) <= 1e-12


def _two_components(directed):
    """Two RMAT blocks with no edges between them plus isolated vertices:
    lanes of one batch reach disjoint vertex sets."""
    u1, v1, w1, n1 = gen.rmat(11, 8, seed=2, undirected=not directed)
    u2, v2, w2, n2 = gen.rmat(10, 8, seed=3, undirected=not directed)
    u = np.concatenate([u1, u2 + n1])
    v = np.concatenate([v1, v2 + n1])
    w = np.concatenate([w1, w2])
    return u, v, w, n1 + n2 + 50


# Fast-mode forms: batched sources with the automatic push/pull choice,
# push-only, pull at every step after the root's, and the per-source path.
BC_FORMS = [{}, {"SP_BC_PULL": "0"}, {"SP_BC_PULL": "1e12"}, {"SP_BC_BATCH": "0"}]


@pytest.mark.parametrize("form", BC_FORMS, ids=["auto", "push", "pull", "per_source"])
@pytest.mark.parametrize("graph", ["rmat_sym", "rmat_dir", "hub_dir", "hub_sym", "multi",
                                   "two_comp_sym", "two_comp_dir"])
def test_bc_fast_forms(graph, form, monkeypatch):
    """Every fast-mode BC form against the oracle: 19 sources (two full
    8-source batches and a partial one, with duplicates inside a batch),
    bc within 1e-12, sigma of the last source bit-exact (integer path
    counts), delta of the last source within 1e-12."""
    for k, val in form.items():
        monkeypatch.setenv(k, val)
    if graph.startswith("rmat"):
        u, v, w, n = gen.rmat(12, 16, seed=21, undirected=graph == "rmat_sym")
        directed = graph == "rmat_dir"
    elif graph.startswith("hub"):
        directed = graph == "hub_dir"
        u, v, w, n = _hub_graph(directed)
    elif graph == "multi":
        u, v, w, n = _multigraph(8)
        directed = True
    else:
        directed = graph == "two_comp_dir"
        u, v, w, n = _two_components(directed)
    g = sp.from_arrays(u, v, w, directed=directed, n=n)
    o = cpu_ref.build_csr(u, v, w, directed, n)
    rng = np.random.default_rng(5)
    srcs = rng.choice(n, size=16, replace=False).tolist()
    srcs = srcs[:5] + [srcs[2]] + srcs[5:] + [0, n - 1, srcs[0]]  # 19, duplicates
    bc, sg, dl = cpu_ref.bc(o, srcs, nthreads=4)
    r = sp.run(corpus.BC, g, {"sourceSet": srcs})
    assert rel_err(r.env.node_props["bc"], bc) <= 1e-12
    assert r.env.node_props["sigma"].tobytes() == sg.tobytes()
    assert rel_err(r.env.node_props["delta"], dl) <= 1e-12
    for k in ("edges_visited", "vertices_visited", "iterations"):
        assert r.stats[k] == sp.run(corpus.BC, g, {"sourceSet": srcs},
                                    deterministic=True).stats[k]


@pytest.mark.parametrize("kind,p0,p1,und", [("rmat", 13, 16, True), ("rmat", 12, 16, False),
                                            ("uniform", 1 << 15, 1 << 19, True)])
def test_tc_seeded(kind, p0, p1, und):
    g, o = _pair(kind, p0, p1, 9, und)
    r = sp.run(corpus.TC, g, {})
    assert r.env.scalars["triangle_count"] == cpu_ref.tc(o, nthreads=8)


def _hub_graph(directed):
    """A 20000-leaf star plus random leaf edges: rows far above the hub
    thresholds (PR in-degree > 4096, BC rows > 8192, SSSP/BFS > 2048)."""
    rng = np.random.default_rng(4)
    k = 20000
    u = np.concatenate([np.arange(1, k + 1), rng.integers(1, k + 1, 30000)])
    v = np.concatenate([np.zeros(k, np.int64), rng.integers(1, k + 1, 30000)])
    w = rng.integers(1, 100, len(u))
    if directed:  # leaves -> hub and hub -> leaves both present
        u, v, w = np.concatenate([u, v[:k]]), np.concatenate([v, u[:k]]), np.concatenate([w, w[:k]])
    return u, v, w, k + 1


@pytest.mark.parametrize("directed", [True, False])
def test_hub_paths(directed):
    u, v, w, n = _hub_graph(directed)
    g = sp.from_arrays(u, v, w, directed=directed, n=n)
    o = cpu_ref.build_csr(u, v, w, directed, n)
    dist, _, _ = cpu_ref.sssp(o, 5)
    np.testing.assert_array_equal(sp.run(corpus.SSSP, g, {"src": 5}).env.node_props["dist"], dist)
    rank, it, diff, its, rc = cpu_ref.pagerank(o, cap=10 ** 6)
    rd = sp.run(corpus.PR, g, PR_ARGS, max_iters=10 ** 6, deterministic=True)
    assert rd.env.node_props["rank"].tobytes() == rank.tobytes() and rd.env.scalars["iter"] == it
    rf = sp.run(corpus.PR, g, PR_ARGS, max_iters=10 ** 6)
    assert rel_err(rf.env.node_props["rank"], rank) <= 1e-12 and rf.env.scalars["iter"] == it
    srcs = [0, 7, 19999, 7]
    bc, sg, dl = cpu_ref.bc(o, srcs)
    rd = sp.run(corpus.BC, g, {"sourceSet": srcs}, deterministic=True)
    assert rd.env.node_props["bc"].tobytes() == bc.tobytes()
    assert rd.env.node_props["delta"].tobytes() == dl.tobytes()
    rf = sp.run(corpus.BC, g, {"sourceSet": srcs})
    assert rel_err(rf.env.node_props["bc"], bc) <= 1e-12
    assert sp.run(corpus.TC, g, {}).env.scalars["triangle_count"] == cpu_ref.tc(o)


# ---------------------------------------------------------------------------
# edge cases the reference exercises

def _multigraph(seed, n=300, m=3000, directed=True, neg=False):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    # parallel edges and self-loops on purpose
    u[: m // 10] = u[m // 10: 2 * (m // 10)]
    v[: m // 10] = v[m // 10: 2 * (m // 10)]
    u[-20:] = v[-20:]
    w = rng.integers(1, 100, m)
    if neg:  # negative weights on a DAG (u < v): no negative cycle
        keep = u < v
        u, v, w = u[keep], v[keep], w[keep] - 60
    return u, v, w, n


@pytest.mark.parametrize("directed", [True, False])
def test_multigraph_all_algorithms(directed):
    u, v, w, n = _multigraph(3, directed=directed)
    g = sp.from_arrays(u, v, w, directed=directed, n=n)
    o = cpu_ref.build_csr(u, v, w, directed, n)
    np.testing.assert_array_equal(g.adj, o.adj)
    np.testing.assert_array_equal(g.rev_eid, o.reid)
    dist, _, _ = cpu_ref.sssp(o, 0)
    np.testing.assert_array_equal(sp.run(corpus.SSSP, g, {"src": 0}).env.node_props["dist"], dist)
    # pull form: reverse slots carry the first forward slot's weight (rweff)
    np.testing.assert_array_equal(sp.run(corpus.SSSP_PULL, g, {"src": 0}).env.node_props["dist"],
                                  dist)
    rank = cpu_ref.pagerank(o, cap=10 ** 6)[0]
    r = sp.run(corpus.PR, g, PR_ARGS, max_iters=10 ** 6, deterministic=True)
    assert r.env.node_props["rank"].tobytes() == rank.tobytes()
    bc = cpu_ref.bc(o, [0, 5, 7, 5])[0]
    r = sp.run(corpus.BC, g, {"sourceSet": [0, 5, 7, 5]}, deterministic=True)
    assert r.env.node_props["bc"].tobytes() == bc.tobytes()
    assert sp.run(corpus.TC, g, {}).env.scalars["triangle_count"] == cpu_ref.tc(o)


def test_sssp_negative_weights_dag():
    u, v, w, n = _multigraph(5, neg=True)
    g = sp.from_arrays(u, v, w, directed=True, n=n)
    o = cpu_ref.build_csr(u, v, w, True, n)
    dist, _, rc = cpu_ref.sssp(o, int(u[0]))
    assert rc == 0
    r = sp.run(corpus.SSSP, g, {"src": int(u[0])})
    np.testing.assert_array_equal(r.env.node_props["dist"], dist)


def test_sssp_negative_cycle_nonconvergence():
    g = sp.from_edges([(0, 1, 1), (1, 2, -3), (2, 0, 1)])
    with pytest.raises(NonConvergenceError) as ei:
        sp.run(corpus.SSSP, g, {"src": 0})
    assert ei.value.flag == "finished" and ei.value.cap == 2 * 3 + 16
    with pytest.raises(NonConvergenceError) as ei:
        sp.run(corpus.SSSP, g, {"src": 0}, max_iters=5)
    assert ei.value.cap == 5


def test_int_max_semantics():
    """A candidate >= INT_MAX never wins (interp.py:11-14)."""
    g = sp.from_edges([(0, 1, 2_000_000_000), (1, 2, 2_000_000_000), (0, 3, 5)])
    d = sp.run(corpus.SSSP, g, {"src": 0}).env.node_props["dist"]
    assert d.tolist() == [0, 2_000_000_000, 2147483647, 5]


def test_spec_known_answers():
    # SPEC.md:271-275
    d = sp.run(corpus.SSSP, sp.from_edges([(0, 1, 4), (1, 2, 3)]), {"src": 0})
    assert d.env.node_props["dist"].tolist() == [0, 4, 7]
    iso = sp.from_edges([(1, 2, 5)], n=4)
    assert sp.run(corpus.SSSP, iso, {"src": 0}).env.node_props["dist"].tolist() == \
        [0, 2147483647, 2147483647, 2147483647]
    c4 = sp.from_edges([(0, 1), (1, 2), (2, 3), (3, 0)])
    r = sp.run(corpus.PR, c4, PR_ARGS)
    assert np.allclose(r.env.node_props["rank"], 0.25, atol=1e-9)
    k3 = sp.from_edges([(0, 1), (0, 2), (1, 2)], directed=False)
    k4 = sp.from_edges([(a, b) for a in range(4) for b in range(a + 1, 4)], directed=False)
    assert sp.run(corpus.TC, k3, {}).env.scalars["triangle_count"] == 1
    assert sp.run(corpus.TC, k4, {}).env.scalars["triangle_count"] == 4
    p3 = sp.from_edges([(0, 1), (1, 2)], directed=False)
    r = sp.run(corpus.BC, p3, {"sourceSet": [0, 1, 2]}, deterministic=True)
    assert r.env.node_props["bc"].tolist() == [0.0, 1.0, 0.0]


def test_empty_and_degenerate():
    g = sp.from_edges([])
    assert g.n == 0 and g.m == 0
    r = sp.run(corpus.PR, g, PR_ARGS)
    assert r.env.scalars["iter"] == 1 and r.env.scalars["diff"] == 0.0
    assert sp.run(corpus.TC, g, {}).env.scalars["triangle_count"] == 0
    with pytest.raises(ExecError):
        sp.run(corpus.SSSP, g, {"src": 0})
    g1 = sp.from_edges([], n=5)
    r = sp.run(corpus.BC, g1, {"sourceSet": []})
    assert list(r.env.node_props) == ["bc"] and not r.env.node_props["bc"].any()
    r = sp.run(corpus.SSSP, g1, {"src": 4})
    assert r.env.node_props["dist"].tolist() == [2147483647] * 4 + [0]
    with pytest.raises(ExecError, match="missing argument 'src'"):
        sp.run(corpus.SSSP, g1, {})
    with pytest.raises(ExecError, match="set argument 'sourceSet' id 9 out of range"):
        sp.run(corpus.BC, g1, {"sourceSet": [1, 9]})


def test_iteration_hook_called_each_iteration():
    g = sp.from_edges([(i, i + 1, 1) for i in range(20)])
    seen = []
    r = sp.run(corpus.PR, g, PR_ARGS, on_fixedpoint_iteration=lambda f, k, ex: seen.append((f, k)))
    assert seen == [("converged", k) for k in range(1, r.fixedpoint_iterations["converged"] + 1)]
    seen.clear()
    r = sp.run(corpus.SSSP, g, {"src": 0}, on_fixedpoint_iteration=lambda f, k, ex: seen.append(k))
    assert seen == list(range(1, r.fixedpoint_iterations["finished"] + 1))

    def boom(f, k, ex):
        raise KeyboardInterrupt("stop")
    with pytest.raises(KeyboardInterrupt):
        sp.run(corpus.SSSP, g, {"src": 0}, on_fixedpoint_iteration=boom)


def test_weight_range_and_io(tmp_path):
    g = sp.from_edges([(0, 1, 3), (1, 2, 1), (2, 0, 9)])
    assert (sp.min_wt(g), sp.max_wt(g)) == (1, 9)
    p = tmp_path / "g.txt"
    sp.write_edge_list(g, str(p))
    g2 = sp.load_edge_list(str(p))
    np.testing.assert_array_equal(g2.adj, g.adj)
    np.testing.assert_array_equal(g2.weights, g.weights)


@pytest.mark.parametrize("n,p,seed", [(600, 0.8, 1), (900, 0.45, 2)])
def test_tc_dense_rows_cta_path(n, p, seed):
    """Upper rows longer than the warp path (> 256 after degree ordering)
    go through the CTA kernel; dense random graphs exercise it, with
    parallel edges sprinkled in (multiplicity products)."""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(len(iu)) < p
    u, v = iu[keep], ju[keep]
    dup = rng.random(len(u)) < 0.01
    u = np.concatenate([u, u[dup]])
    v = np.concatenate([v, v[dup]])
    w = np.ones(len(u), dtype=np.int64)
    g = sp.from_arrays(u, v, w, directed=False, n=n)
    o = cpu_ref.build_csr(u, v, w, False, n)
    assert sp.run(corpus.TC, g, {}).env.scalars["triangle_count"] == cpu_ref.tc(o, nthreads=8)


TC_FORMS = [{"SP_TC_WARP_MAX": "16", "SP_TC_HUB": "0"},
            {"SP_TC_WARP_MAX": "16", "SP_TC_HASH_MAX": "32", "SP_TC_HUB": "0"},
            {"SP_TC_WARP_MAX": "16", "SP_TC_HASH_MAX": "32", "SP_TC_BIG_MAX": "64",
             "SP_TC_HUB": "0"},
            {"SP_TC_WARP_MAX": "16"},
            {"SP_TC_WARP_MAX": "16", "SP_TC_HUB": "2"},
            # every hub-rank row to k_tc_big / none of them
            {"SP_TC_WARP_MAX": "16", "SP_TC_HUB_MIN": "0"},
            {"SP_TC_HUB_MIN": "1000000"}]


@pytest.mark.parametrize("form", TC_FORMS, ids=["hashed", "staged", "global", "hub", "hub16",
                                                "hub_all", "hub_none"])
@pytest.mark.parametrize("graph", ["dense_dup", "rmat_sym"])
def test_tc_big_row_forms(graph, form, monkeypatch):
    """k_tc_big's three row forms -- shared hash table, staged A with a
    filter + binary search, and binary search in global memory -- are
    normally reached only by rows longer than 256 / 8 K / 48 K; lowered
    thresholds route small graphs through each form, against the oracle
    (parallel edges included: multiplicity products)."""
    for k, val in form.items():
        monkeypatch.setenv(k, val)
    if graph == "dense_dup":
        rng = np.random.default_rng(9)
        n = 500
        iu, ju = np.triu_indices(n, 1)
        keep = rng.random(len(iu)) < 0.3
        u, v = iu[keep], ju[keep]
        dup = rng.random(len(u)) < 0.02
        u = np.concatenate([u, u[dup]])
        v = np.concatenate([v, v[dup]])
        w = np.ones(len(u), dtype=np.int64)
    else:
        u, v, w, n = gen.rmat(13, 16, seed=4, undirected=True)
    g = sp.from_arrays(u, v, w, directed=False, n=n)
    o = cpu_ref.build_csr(u, v, w, False, n)
    assert sp.run(corpus.TC, g, {}).env.scalars["triangle_count"] == cpu_ref.tc(o, nthreads=8)


@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("pinned", [False, True])
def test_from_csr_pipelined_reverse(weighted, pinned, monkeypatch):
    """A large directed host CSR (>= 8 M slots) is uploaded in pieces with
    the reverse CSR built piecewise (per-piece stable sorts + one scatter):
    identical arrays to the one-sort build of the same graph, and the same
    PageRank bits."""
    import torch
    gd = sp.generate("rmat", 20, 16, seed=6)  # directed, m ~ 16 M
    off = np.array(gd.offsets)
    adj = np.array(gd.adj)
    w = np.array(gd.weights) if weighted else None
    if pinned:
        off = torch.from_numpy(off).pin_memory().numpy()
        adj = torch.from_numpy(adj).pin_memory().numpy()
        if weighted:
            w = torch.from_numpy(w).pin_memory().numpy()
    g = sp.from_csr(off, adj, w, directed=True)
    monkeypatch.setenv("SP_UPLOAD_PLAIN", "1")
    gp = sp.from_csr(off, adj, w, directed=True)
    for a, b in ((g, gd), (gp, gd)):
        np.testing.assert_array_equal(a.rev_offsets, b.rev_offsets)
        np.testing.assert_array_equal(a.rev_adj, b.rev_adj)
        np.testing.assert_array_equal(a.adj, b.adj)
    if weighted:
        np.testing.assert_array_equal(g.weights, gd.weights)
    r1 = sp.run(corpus.PR, g, PR_ARGS)
    r2 = sp.run(corpus.PR, gd, PR_ARGS)
    assert r1.env.node_props["rank"].tobytes() == r2.env.node_props["rank"].tobytes()
    if weighted:  # w_eff and the reverse weights come from the uploaded arrays
        for prog in (corpus.SSSP, corpus.SSSP_PULL):
            np.testing.assert_array_equal(sp.run(prog, g, {"src": 0}).env.node_props["dist"],
                                          sp.run(prog, gd, {"src": 0}).env.node_props["dist"])
    for x in (g, gp, gd):
        x.close()


@pytest.mark.parametrize("case", CASES)
def test_native_loader_builds_reference_csr(case, tmp_path):
    """load_edge_list through the native parser (mixed \\n / \\r\\n / \\r line
    ends, comments, blank lines, tabs) builds the reference's CSR arrays."""
    z = load_golden(case)
    u, v, w = z["u"], z["v"], z["w"]
    if len(u) == 0 or int(max(u.max(), v.max())) + 1 != int(z["n"]):
        pytest.skip("n is not 1 + max id for this case")
    ends = ["\n", "\r\n", "\r"]
    lines = ["# generated from the golden edge list", ""]
    for i in range(len(u)):
        sep = "\t" if i % 3 == 0 else " "
        lines.append(f"{u[i]}{sep}{v[i]} {w[i]}" if i % 5 else f"  {u[i]} {v[i]}  {w[i]} ")
    text = "".join(ln + ends[i % 3] for i, ln in enumerate(lines))
    p = tmp_path / "g.txt"
    p.write_bytes(text.encode())
    g = sp.load_edge_list(str(p), directed=bool(z["directed"]))
    np.testing.assert_array_equal(g.offsets, z["csr_off"])
    np.testing.assert_array_equal(g.adj, z["csr_adj"])
    np.testing.assert_array_equal(g.weights, z["csr_w"])
    np.testing.assert_array_equal(g.rev_adj, z["csr_radj"])


def test_native_loader_large_file_matches_arrays(tmp_path):
    """A multi-MiB file (parsed by several host threads) gives the same graph
    as from_arrays on the same edges."""
    u, v, w, n = gen.rmat(15, 16, seed=9)
    text = "\n".join(f"{a} {b} {c}" for a, b, c in zip(u.tolist(), v.tolist(), w.tolist()))
    p = tmp_path / "big.txt"
    p.write_text(text + "\n")
    g = sp.load_edge_list(str(p))
    h = sp.from_arrays(u, v, w, directed=True)
    np.testing.assert_array_equal(g.offsets, h.offsets)
    np.testing.assert_array_equal(g.adj, h.adj)
    np.testing.assert_array_equal(g.weights, h.weights)


def test_concurrent_calls_on_one_graph():
    """A graph handle is immutable and safe for concurrent readers
    (SPEC.md:239): four host threads run all four programs on the same
    graph at once and get the single-threaded results."""
    import threading
    u, v, w, n = gen.rmat(12, 16, seed=21, undirected=True)
    g = sp.from_arrays(u, v, w, directed=False, n=n)
    want = {
        "sssp": sp.run(corpus.SSSP, g, {"src": 1}).env.node_props["dist"],
        "pr": sp.run(corpus.PR, g, {"damping": 0.85, "epsilon": 1e-6,
                                    "maxIter": 100}).env.node_props["rank"],
        "bc": sp.run(corpus.BC, g, {"sourceSet": [1, 2, 3]}).env.node_props["bc"],
        "tc": sp.run(corpus.TC, g, {}).env.scalars["triangle_count"],
    }
    got, errs = {}, []

    def work(key):
        try:
            for _ in range(3):
                if key == "sssp":
                    got[key] = sp.run(corpus.SSSP, g, {"src": 1}).env.node_props["dist"]
                elif key == "pr":
                    got[key] = sp.run(corpus.PR, g, {"damping": 0.85, "epsilon": 1e-6,
                                                     "maxIter": 100}).env.node_props["rank"]
                elif key == "bc":
                    got[key] = sp.run(corpus.BC, g, {"sourceSet": [1, 2, 3]}).env.node_props["bc"]
                else:
                    got[key] = sp.run(corpus.TC, g, {}).env.scalars["triangle_count"]
        except Exception as e:  # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=work, args=(k,)) for k in want]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    assert np.array_equal(got["sssp"], want["sssp"])
    assert got["pr"].tobytes() == want["pr"].tobytes()  # deterministic run to run
    assert got["bc"].tobytes() == want["bc"].tobytes()
    assert got["tc"] == want["tc"]


@pytest.mark.parametrize("kind,p0,p1,und", [("rmat", 14, 16, False), ("rmat", 18, 16, False),
                                            ("grid", 64, 64, True)])
def test_device_loop_equals_host_loop(kind, p0, p1, und, monkeypatch):
    """The conditional-graph fixedPoint loops (PR, SSSP) give bit-identical
    results to the host-driven loop over the same kernels (SP_HOSTLOOP=1)."""
    g, _ = _pair(kind, p0, p1, 5, und)
    args = {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
    dev_pr = sp.run(corpus.PR, g, args)
    dev_ss = sp.run(corpus.SSSP, g, {"src": 0})
    monkeypatch.setenv("SP_HOSTLOOP", "1")
    host_pr = sp.run(corpus.PR, g, args)
    host_ss = sp.run(corpus.SSSP, g, {"src": 0})
    assert dev_pr.env.node_props["rank"].tobytes() == host_pr.env.node_props["rank"].tobytes()
    assert dev_pr.env.scalars == host_pr.env.scalars
    assert np.array_equal(dev_ss.env.node_props["dist"], host_ss.env.node_props["dist"])


class _TridentLikeGraph:
    """The attribute surface of trident.graph.CsrGraph (graph.py:18-36):
    Python lists, as the reference builds them."""

    def __init__(self, z):
        self.offsets = [int(x) for x in z["csr_off"]]
        self.adj = [int(x) for x in z["csr_adj"]]
        self.weights = [int(x) for x in z["csr_w"]]
        self.directed = bool(z["directed"])

    def num_nodes(self):
        return len(self.offsets) - 1


@pytest.mark.parametrize("case", ["fx_rand200_a_d", "fx_rand200_b_u", "syn_rmat10_d"])
def test_run_adopts_reference_graph_objects(case):
    """run() on a reference-style CsrGraph object: uploaded once (cached per
    object), results equal the reference's golden values."""
    from paper_2305_03317_b200 import graph as spg
    z = load_golden(case)
    tg = _TridentLikeGraph(z)
    r = sp.run(corpus.SSSP, tg, {"src": int(z["sssp_srcs"][0])})
    np.testing.assert_array_equal(r.env.node_props["dist"], z["sssp_dist"][0])
    assert spg.device_graph(tg) is spg.device_graph(tg)  # one upload per object
    if int(z["pr_err_cap"]) < 0:  # the reference converged within its cap
        r = sp.run(corpus.PR, tg, {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100},
                   deterministic=True)
        assert r.env.node_props["rank"].tobytes() == z["pr_rank"].tobytes()
    assert sp.run(corpus.TC, tg, {}).env.scalars["triangle_count"] == int(z["tc"])


@pytest.mark.parametrize("case", CASES)
def test_reduction_program(case, graphs):
    """reduction.sp (the generic forall / neighbour-reduction shape):
    prop = 1 everywhere, accum = number of CSR slots (the reference's
    result, checked against the golden CSR)."""
    z, g = graphs(case)
    r = sp.run(corpus.REDUCTION, g, {})
    assert r.env.scalars == {"accum": len(z["csr_adj"])}
    assert r.env.node_props["prop"].tolist() == [1] * int(z["n"])


@pytest.mark.parametrize("directed", [True, False])
@pytest.mark.parametrize("reverse", [0, 1])
def test_neighbor_sum_generic(directed, reverse):
    """The generic neighbour reduction on an arbitrary int64 property,
    over g.neighbors (reverse=0) or g.nodesTo (reverse=1), vs numpy."""
    import ctypes as C
    from paper_2305_03317_b200 import _lib
    u, v, w, n = gen.rmat(12, 16, seed=31, undirected=not directed)
    g = sp.from_arrays(u, v, w, directed=directed, n=n)
    prop = np.random.default_rng(3).integers(-10 ** 12, 10 ** 12, n).astype(np.int64)
    per = np.empty(n, dtype=np.int64)
    tot = C.c_int64()
    rc = _lib.lib().sp_neighbor_sum(g.handle, prop.ctypes.data_as(C.c_void_p), _lib.SP_MEM_HOST,
                                    reverse, per.ctypes.data_as(C.c_void_p), C.byref(tot), None)
    assert rc == 0
    off = np.asarray(g.rev_offsets if reverse else g.offsets)
    col = np.asarray(g.rev_adj if reverse else g.adj)
    rows = np.repeat(np.arange(n), np.diff(off))
    want = np.zeros(n, dtype=np.int64)
    np.add.at(want, rows, prop[col])
    np.testing.assert_array_equal(per, want)
    assert tot.value == int(want.sum())


@pytest.mark.parametrize("case", ["multi300_u_7", "multi300_d_0", "rmat9_u_123"])
def test_assign_random_weights_device_graph(case):
    """assign_random_weights on a device graph gives the weights the
    reference assigned (tests/golden/weights, made by the reference) and a
    graph whose w_eff/SSSP follow them."""
    import os
    from conftest import REPO
    z = np.load(os.path.join(REPO, "tests", "golden", "weights", case + ".npz"))
    g = sp.from_csr(z["off"], z["adj"], None, directed=bool(z["directed"]))
    g2 = sp.assign_random_weights(g, int(z["lo"]), int(z["hi"]), int(z["seed"]))
    np.testing.assert_array_equal(g2.weights, z["w"])
    np.testing.assert_array_equal(g2.adj, z["adj"])
    o = cpu_ref.Csr(g2.n, g2.m, g2.directed, np.asarray(g2.offsets), np.asarray(g2.adj),
                    np.asarray(g2.weights), None, None, None, None)
    weff = np.zeros(g2.m, np.int32)
    cpu_ref.lib().cr_weff(g2.n, cpu_ref._ptr(o.off), cpu_ref._ptr(o.adj),
                          cpu_ref._ptr(np.ascontiguousarray(o.w)), cpu_ref._ptr(weff))
    np.testing.assert_array_equal(g2.effective_weights, weff)


@pytest.mark.parametrize("case", ["fx_rand200_a_u", "fx_k5_d", "fx_grid5x5_u"])
def test_as_lists_matches_reference_layout(case, graphs):
    """as_lists=True: node props are Python lists of Python scalars equal
    (==) to the reference's final_env lists (interp.py:259-266)."""
    z, g = graphs(case)
    r = sp.run(corpus.SSSP, g, {"src": int(z["sssp_srcs"][0])}, as_lists=True)
    d = r.env.node_props["dist"]
    assert isinstance(d, list) and all(type(x) is int for x in d)
    assert d == z["sssp_dist"][0].tolist()
    assert r.env.node_props["modified"] == [False] * g.n
    r = sp.run(corpus.PR, g, PR_ARGS, deterministic=True, as_lists=True)
    assert r.env.node_props["rank"] == z["pr_rank"].tolist()
    assert r.env.node_props["rank_nxt"] == z["pr_rank_nxt"].tolist()
    assert all(type(x) is float for x in r.env.node_props["rank"])
    r = sp.run(corpus.BC, g, {"sourceSet": z["bc_srcs"].tolist()}, deterministic=True,
               as_lists=True)
    assert r.env.node_props["bc"] == z["bc"].tolist()
    with pytest.raises(ValueError):
        sp.run(corpus.PR, g, PR_ARGS, as_lists=True, device_outputs=True)


def test_from_csr_rejects_bad_input():
    """from_csr validates its input before any kernel indexes by it."""
    from paper_2305_03317_b200.errors import ArgError
    off = np.array([0, 2, 3, 3], np.int64)
    adj = np.array([1, 2, 0], np.int32)
    g = sp.from_csr(off, adj, None, directed=True)
    assert g.m == 3
    with pytest.raises(ArgError):  # weights shorter than adj
        sp.from_csr(off, adj, np.array([1, 2], np.int32))
    with pytest.raises(ArgError):  # last offset != len(adj)
        sp.from_csr(np.array([0, 2, 3, 4], np.int64), adj)
    with pytest.raises(ArgError):  # rows not monotone (device check)
        sp.from_csr(np.array([0, 3, 1, 3], np.int64), adj)
    with pytest.raises(ArgError):  # id out of range (device check)
        sp.from_csr(off, np.array([1, 7, 0], np.int32))
    with pytest.raises(ArgError):
        sp.from_csr(off, np.array([1, -1, 0], np.int32), directed=False)
    with pytest.raises(ArgError):  # float weights are not truncated
        sp.from_csr(off, adj, np.array([1.5, 2.0, 3.0]))


def test_from_csr_rejects_bad_ids_pipelined():
    """The large-graph upload path (reverse CSR built while the adjacency
    crosses PCIe) flags an out-of-range id without writing out of bounds."""
    from paper_2305_03317_b200.errors import ArgError
    rng = np.random.default_rng(5)
    n, m = 1 << 16, 1 << 23
    adj = np.sort(rng.integers(0, n, m, dtype=np.int32).reshape(n, -1), axis=1).ravel()
    off = np.arange(0, m + 1, m // n, dtype=np.int64)
    g = sp.from_csr(off, adj, None, directed=True)
    assert g.m == m
    g.close()
    bad = adj.copy()
    bad[m // 2] = n + 5
    with pytest.raises(ArgError):
        sp.from_csr(off, bad, None, directed=True)
    bad[m // 2] = -3
    with pytest.raises(ArgError):
        sp.from_csr(off, bad, None, directed=True)


def test_preprocessing_times_reported():
    """sp_graph_prep_ms: a lazily built per-graph structure reports its build
    time once built (the TC upper CSR on the first TC call; the pull-sweep
    reverse weights on a forced direction-optimising SSSP run) and nothing
    before; structures built during the upload (w_eff of an edge-list
    graph) are not reported."""
    g, _ = _pair("rmat", 14, 16, 5, True)
    assert g.preprocessing_ms() == {}
    sp.run(corpus.TC, g, {})
    pre = g.preprocessing_ms()
    assert set(pre) == {"tc_upper"} and pre["tc_upper"] > 0
    sp.run(corpus.TC, g, {})
    assert g.preprocessing_ms()["tc_upper"] == pre["tc_upper"]  # built once
    d, _ = _pair("rmat", 12, 16, 5, False)
    sp.run(corpus.SSSP_PULL, d, {"src": 0})
    assert d.preprocessing_ms().get("rweff", 0) > 0
    gr, _ = _pair("grid", 64, 64, 5, True)  # thin: ELL rows, then 2-hop shortcut rows
    sp.run(corpus.SSSP, gr, {"src": 0})
    pre = gr.preprocessing_ms()
    assert pre.get("ell", 0) > 0 and pre.get("ell2", 0) > 0


def test_pagerank_cluster_hot_set_subprocess():
    """The 2-CTA cluster hot set (k_pr_units_hot2: half of a 40 K-source hot
    set per CTA, the other half read through distributed shared memory;
    SP_PR_HOT_MAX is read once per process, so this runs in a child
    process): ranks within 1e-12 of the oracle and its iteration count on
    RMAT-20, whose top 40 K sources qualify."""
    import os
    import subprocess
    import sys
    code = r'''
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2305_03317_b200 as sp
from paper_2305_03317_b200 import corpus, gen
from oracle import cpu_ref
u, v, w, n = gen.rmat(20, 16, seed=7)
g = sp.from_arrays(u, v, w, directed=True, n=n)
o = cpu_ref.build_csr(u, v, w, True, n)
args = {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
for _ in range(3):  # the hot set is built on the graph's second fast call
    r = sp.run(corpus.PR, g, args)
rank, it, diff, its, rc = cpu_ref.pagerank(o, 0.85, 1e-6, 100)
assert r.env.scalars["iter"] == it, (r.env.scalars["iter"], it)
np.testing.assert_allclose(r.env.node_props["rank"], rank, rtol=1e-12, atol=0)
print("ok", r.stats["kernel_launches"])
'''
    env = dict(os.environ, SP_PR_HOT_MAX="40960", SP_PR_REL="0", SP_PR_HOT_VERBOSE="1")
    p = subprocess.run([sys.executable, "-c", code], cwd=os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    assert p.stdout.startswith("ok")
    assert "top 4095" in p.stderr  # the split (> 20 K) hot set was built
