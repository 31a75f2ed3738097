"""parallel.run_sharded with the native per-rank backend on the GPU.

One GPU is available, so two ranks share cuda:0 over gloo (NCCL refuses two
ranks on one device); this drives the native block kernels
(sp_sssp_shard_*: owner-computes SSSP with the exchange fused into the
relaxation over peer memory -- remote atomicMin into the owner's dist and
its inbox, CUDA IPC between the two processes -- and with aggregated
messages in both exchange forms, sp_pagerank_shard_* (planned once, stream-ordered steps, the
contrib exchange as peer stores fused into the step -- CUDA IPC between the
two processes -- and as an all-gather), sp_tc ranges, sp_bc source shares) through the real sharding/exchange logic and checks the results
against the single-process CPU oracle."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import REPO  # noqa: F401
from oracle import cpu_ref
from paper_2305_03317_b200 import corpus, gen

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _edges(kind):
    if kind == "rmat_d":
        return gen.rmat(12, 16, seed=4) + (True,)
    if kind == "rmat_u":
        return gen.rmat(12, 8, seed=5, undirected=True) + (False,)
    u, v, w, n = gen.grid(40, 50, seed=6)
    return u, v, w, n, False


def _worker(rank, world, port, kind, q):
    import torch
    import torch.distributed as dist

    import paper_2305_03317_b200 as sp
    from paper_2305_03317_b200 import parallel
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        u, v, w, n, directed = _edges(kind)
        g = sp.from_arrays(u, v, w, directed=directed, n=n)
        be = parallel.NativeBackend(0)
        out = {}
        r = parallel.run_sharded(corpus.SSSP, g, {"src": 0}, backend=be)
        out["dist"], out["sssp_exchange"] = r.env.node_props["dist"], r.stats["exchange"]
        for ex in ("sparse", "dense"):
            os.environ["SP_SSSP_EXCHANGE"] = ex
            r = parallel.run_sharded(corpus.SSSP, g, {"src": 0}, backend=be)
            out["dist_" + ex] = r.env.node_props["dist"]
            out["k_" + ex] = r.fixedpoint_iterations["finished"]
        os.environ["SP_SSSP_EXCHANGE"] = "auto"
        sim = parallel.simulate(corpus.SSSP, g, 2, {"src": 0}, backend=be, local_fixpoint=True)
        out["dist_lf"] = sim.result.env.node_props["dist"]
        out["trace"] = parallel.format_trace_tsv(sim)
        out["steps"] = [(s.finished, dict(s.local_updates), dict(s.msgs_out))
                        for s in sim.supersteps]
        out["k_lf"] = sim.result.fixedpoint_iterations["finished"]
        r = parallel.run_sharded(corpus.PR, g, {"damping": 0.85, "epsilon": 1e-6,
                                                "maxIter": 100}, backend=be,
                                 deterministic=True)
        out["rank"], out["iter"] = r.env.node_props["rank"], r.env.scalars["iter"]
        r = parallel.run_sharded(corpus.PR, g, {"damping": 0.85, "epsilon": 1e-6,
                                                "maxIter": 100}, backend=be)
        out["rank_fast"] = r.env.node_props["rank"]
        # the same two runs with the all-gather exchange instead of the
        # peer stores fused into the step (CUDA IPC between the two
        # processes here; NVLink between GPUs): identical results
        os.environ["SP_PR_EXCHANGE"] = "nccl"
        r = parallel.run_sharded(corpus.PR, g, {"damping": 0.85, "epsilon": 1e-6,
                                                "maxIter": 100}, backend=be, deterministic=True)
        out["rank_gather"], out["iter_gather"] = r.env.node_props["rank"], r.env.scalars["iter"]
        r = parallel.run_sharded(corpus.PR, g, {"damping": 0.85, "epsilon": 1e-6,
                                                "maxIter": 100}, backend=be)
        out["rank_fast_gather"] = r.env.node_props["rank"]
        os.environ["SP_PR_EXCHANGE"] = "p2p"
        srcs = list(range(0, 40, 3))
        r = parallel.run_sharded(corpus.BC, g, {"sourceSet": srcs}, backend=be)
        out["bc"] = r.env.node_props["bc"]
        out["tc"] = parallel.run_sharded(corpus.TC, g, {}, backend=be).env.scalars[
            "triangle_count"]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["rmat_d", "rmat_u", "grid"])
def test_native_sharded_two_ranks(kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    u, v, w, n, directed = _edges(kind)
    o = cpu_ref.build_csr(u, v, w, directed, n)
    d_ref = cpu_ref.sssp(o, 0)[0]
    rank_ref, it_ref, *_ = cpu_ref.pagerank(o)
    bc_ref = cpu_ref.bc(o, list(range(0, 40, 3)))[0]
    tc_ref = cpu_ref.tc(o)
    for r in range(2):
        x = res[r]
        assert np.array_equal(x["dist"], d_ref)
        assert x["sssp_exchange"] == "peer"  # fused into the relaxation (CUDA IPC here)
        for key in ("dist_sparse", "dist_dense", "dist_lf"):
            assert np.array_equal(x[key], d_ref), key
        assert x["k_sparse"] == x["k_dense"]  # same supersteps, either exchange form
        assert x["k_lf"] <= x["k_sparse"]
        # native simulate trace: bsp.py's TSV layout, one line per rank per
        # superstep, finished only on the last; every vertex reached from 0
        # is lowered once at least, by its owner or by an applied message
        lines = x["trace"].strip().split("\n")
        assert lines[0] == "superstep\trank\tlocal_updates\tmsgs_out\tfinished"
        assert len(lines) == 1 + 2 * len(x["steps"])
        assert [s[0] for s in x["steps"]] == [False] * (len(x["steps"]) - 1) + [True]
        if len(x["steps"]) > 1:
            assert sum(s[2][0] + s[2][1] for s in x["steps"]) > 0  # messages crossed
        reached = int((d_ref < 2147483647).sum())
        assert sum(s[1][0] + s[1][1] for s in x["steps"]) + \
            sum(s[2][0] + s[2][1] for s in x["steps"]) >= reached - 1
        assert x["rank"].tobytes() == rank_ref.tobytes() and x["iter"] == it_ref
        assert np.abs(x["rank_fast"] - rank_ref).max() <= 1e-12 * np.abs(rank_ref).max()
        assert x["rank_gather"].tobytes() == rank_ref.tobytes() and x["iter_gather"] == it_ref
        assert x["rank_fast_gather"].tobytes() == x["rank_fast"].tobytes()
        assert np.abs(x["bc"] - bc_ref).max() <= 1e-9 * max(1.0, np.abs(bc_ref).max())
        assert x["tc"] == tc_ref
