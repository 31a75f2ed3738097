"""Multi-rank host logic of paper_2305_03317_b200.parallel on gloo
(world_size 2 and 3, CPU): sharding, exchange and convergence are checked
against the single-process oracle -- never against trident.bsp.simulate,
whose SSSP supersteps are wrong at nranks > 1."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import REPO  # noqa: F401  (sys.path set up)
from oracle import cpu_ref
from paper_2305_03317_b200 import corpus, gen, parallel


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graph(kind, directed):
    if kind == "rmat":
        u, v, w, n = gen.rmat(7, 8, seed=3, undirected=not directed)
    elif kind == "grid":
        u, v, w, n = gen.grid(6, 7, seed=5)
        directed = False
    else:  # multigraph with parallel edges and self-loops
        rng = np.random.default_rng(11)
        n = 60
        u = rng.integers(0, n, 500)
        v = rng.integers(0, n, 500)
        w = rng.integers(1, 20, 500)
    return cpu_ref.build_csr(u, v, w, directed, n)


def _worker(rank, world, port, kind, directed, q, exchange="auto"):
    import torch.distributed as dist
    from oracle_backend import OracleBackend
    os.environ["SP_SSSP_EXCHANGE"] = exchange
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = _graph(kind, directed)
        be = OracleBackend()
        out = {}
        r = parallel.run_sharded(corpus.SSSP, g, {"src": 0}, backend=be)
        out["dist"] = r.env.node_props["dist"]
        r = parallel.run_sharded(corpus.SSSP, g, {"src": 0}, backend=be, local_fixpoint=True)
        out["dist_lf"] = r.env.node_props["dist"]
        args = {"damping": 0.85, "epsilon": 1e-6, "maxIter": 100}
        r = parallel.run_sharded(corpus.PR, g, args, backend=be)
        out["rank"] = r.env.node_props["rank"]
        out["iter"] = r.env.scalars["iter"]
        srcs = [0, 5, 3, 5, 17, 1, 2]
        r = parallel.run_sharded(corpus.BC, g, {"sourceSet": srcs}, backend=be)
        out["bc"] = r.env.node_props["bc"]
        out["sigma"] = r.env.node_props["sigma"]
        out["delta"] = r.env.node_props["delta"]
        r = parallel.run_sharded(corpus.TC, g, {}, backend=be)
        out["tc"] = r.env.scalars["triangle_count"]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind,directed", [("rmat", True), ("rmat", False), ("grid", False),
                                           ("multi", True), ("multi", False)])
def test_sharded_matches_single_process_oracle(world, kind, directed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, directed, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = _graph(kind, directed)
    d_ref = cpu_ref.sssp(g, 0)[0]
    rank_ref, it_ref, *_ = cpu_ref.pagerank(g)
    srcs = [0, 5, 3, 5, 17, 1, 2]
    bc_ref, sg_ref, dl_ref = cpu_ref.bc(g, srcs)
    tc_ref = cpu_ref.tc(g)
    for r in range(world):
        o = res[r]
        assert np.array_equal(o["dist"], d_ref)          # bit-exact
        assert np.array_equal(o["dist_lf"], d_ref)       # local fixpoint: same dist
        assert o["rank"].tobytes() == rank_ref.tobytes()  # same left folds per vertex
        assert o["iter"] == it_ref
        scale = max(1.0, float(np.abs(bc_ref).max()))
        assert float(np.abs(o["bc"] - bc_ref).max()) <= 1e-12 * scale  # source order changes
        assert np.array_equal(o["sigma"], sg_ref) and np.array_equal(o["delta"], dl_ref)
        assert o["tc"] == tc_ref


def test_tc_ranges_partition():
    off = np.array([0, 5, 5, 9, 40, 41, 41, 60])
    for world in (1, 2, 3, 8):
        rs = parallel.tc_ranges(off, world)
        assert rs[0][0] == 0 and rs[-1][1] == len(off) - 1
        for (a, b), (c, d) in zip(rs, rs[1:]):
            assert b == c and a <= b


def _trace_worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle_backend import OracleBackend
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # path10 with unit weights: the reference's bsp.simulate loses
        # dist[6..9] at nranks=2; run_sharded must not
        u = list(range(9))
        v = list(range(1, 10))
        g = cpu_ref.build_csr(u, v, [1] * 9, True, 10)
        sim = parallel.simulate(corpus.SSSP, g, world, {"src": 0}, backend=OracleBackend())
        q.put((rank, sim.result.env.node_props["dist"], parallel.format_trace_tsv(sim),
               [(s.index, s.finished, dict(s.local_updates), dict(s.msgs_out))
                for s in sim.supersteps]))
    finally:
        dist.destroy_process_group()


def test_simulate_trace_and_f4_fix():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_trace_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, rest) for r, *rest in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        d, tsv, steps = res[r]
        assert d.tolist() == list(range(10))  # every vertex reached (F4 fixed)
        lines = tsv.strip().split("\n")
        assert lines[0] == "superstep\trank\tlocal_updates\tmsgs_out\tfinished"
        assert len(lines) == 1 + 2 * len(steps)
        assert [s[1] for s in steps] == [False] * (len(steps) - 1) + [True]
        # the path crosses from rank 0's block into rank 1's exactly once:
        # one aggregated Min message, sent by rank 0
        assert sum(s[3][0] for s in steps) == 1 and sum(s[3][1] for s in steps) == 0
        # every vertex but the source is lowered once, by its owner or via
        # that message
        assert sum(s[2][0] + s[2][1] for s in steps) + 1 == 9
    assert res[0][1] == res[1][1]


def _sssp_worker(rank, world, port, exchange, q):
    import torch.distributed as dist
    from oracle_backend import OracleBackend
    from paper_2305_03317_b200.errors import NonConvergenceError
    os.environ["SP_SSSP_EXCHANGE"] = exchange
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        be = OracleBackend()
        out = {}
        for kind, directed in (("rmat", True), ("grid", False), ("multi", True)):
            g = _graph(kind, directed)
            r = parallel.run_sharded(corpus.SSSP, g, {"src": 0}, backend=be)
            k = r.fixedpoint_iterations["finished"]
            # the cap is tested after convergence: max_iters == k converges
            r2 = parallel.run_sharded(corpus.SSSP, g, {"src": 0}, max_iters=k, backend=be)
            try:
                parallel.run_sharded(corpus.SSSP, g, {"src": 0}, max_iters=k - 1, backend=be)
                capped = None
            except NonConvergenceError as e:
                capped = (e.flag, e.cap)
            lf = parallel.run_sharded(corpus.SSSP, g, {"src": 0}, backend=be,
                                      local_fixpoint=True, trace=True)
            out[kind] = (r.env.node_props["dist"], k, r2.env.node_props["dist"],
                         r2.fixedpoint_iterations["finished"], capped,
                         lf.env.node_props["dist"], lf.fixedpoint_iterations["finished"],
                         r.stats["dense_supersteps"], r.stats["messages"])
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["sparse", "dense"])
def test_sharded_sssp_exchange_forms_and_cap(exchange):
    """Both exchange forms give the oracle's dist; max_iters == k converges
    and k - 1 raises NonConvergenceError('finished', k - 1) (the cap is
    tested after the exchange); local fixpoints need no more
    supersteps than single passes."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_sssp_worker, args=(r, world, port, exchange, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for kind, directed in (("rmat", True), ("grid", False), ("multi", True)):
        d_ref = cpu_ref.sssp(_graph(kind, directed), 0)[0]
        for r in range(world):
            d, k, d2, k2, capped, dlf, klf, dense, msgs = res[r][kind]
            assert np.array_equal(d, d_ref) and np.array_equal(d2, d_ref)
            assert np.array_equal(dlf, d_ref)
            assert k2 == k and k >= 1
            assert capped == ("finished", k - 1)
            assert klf <= k
            if exchange == "dense":
                assert dense == k
            else:
                assert dense == 0
        assert len({res[r][kind][1] for r in range(world)}) == 1  # same superstep count
