"""Multi-GPU runs of the corpus programs: one process per GPU over
``torch.distributed`` (NCCL on the GPUs; any backend for the host logic).

``run_sharded(tp, g, args, ...)`` returns the same ``RunResult`` as
``interp.run`` on every rank.  Each program shards the way SURVEY.md 8e lays
out (the reference models multi-rank execution in-process in
trident/bsp.py; its ownership rule is graph.py:226-249):

* BC  -- sources round-robin over ranks in list order, graph replicated;
         one ``all_reduce(sum)`` of the bc array at the end; sigma/delta of
         the last source come from the rank that ran it (broadcast).  No
         data-path collective.
* TC  -- vertex ranges balanced by a sum-of-squared-degree work proxy, graph
         replicated; one integer ``all_reduce(sum)`` (exact).
* PR  -- block partition, planned once per run; per iteration a local pull
         over the owned block whose epilogue also stores every contrib it
         computes straight into every rank's contrib array for the next
         iteration (peer memory: CUDA IPC, NVLink between GPUs; two arrays
         alternate by iteration parity) -- the reference's remote-read
         snapshot (bsp.py:182-185/287-288) without a separate collective --
         then ``all_reduce(max)`` of diff (the scalar merge, bsp.py:322-330),
         which also orders every rank's stores before the next step.  With
         SP_PR_EXCHANGE=nccl, or where peer mapping fails, an ``all_gather``
         of the owned slices after the step.  One host read per iteration.
* SSSP -- owner-computes over the block partition: per superstep each rank
         relaxes its owned frontier (one pass, or to a local fixpoint);
         remote improvements leave as ONE aggregated (vertex, local min)
         message per vertex (bsp.py:45-72), grouped by owner and exchanged
         with one ``all_to_all_single`` -- or, when the messages would
         outweigh the distance array, a MIN ``reduce_scatter``; owners apply
         them (bsp.py:350-368), then ``all_reduce(sum)`` of the next
         frontier sizes decides convergence -- evaluated AFTER the exchange,
         which is exactly what bsp.py:393-417 gets wrong.

The per-rank compute is a backend object; ``NativeBackend`` drives
libstarplat_b200.so on this rank's GPU.  The tests substitute a CPU backend
(tests/oracle_backend.py) to run this module's host logic on gloo.
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib, corpus
from .errors import errors_for
from .graph import block_partition, device_graph
from .interp import PropertyEnv, RunResult, check_args, default_iteration_cap


class NativeBackend:
    """Per-rank compute on a CUDA device through the C ABI (no fallback)."""

    def __init__(self, device: int):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.index = device
        _lib.require_device(device)
        self.L = _lib.lib()
        self.last_stats = {}  # counters of the last native call (sp_stats)

    def _fence(self):
        # the native calls run on their own streams (and sync them before
        # returning); torch's copies and collectives run on torch's current
        # stream, so that work must be complete before a native call reads it
        self.torch.cuda.current_stream(self.device).synchronize()

    def _chk(self, rc, what):
        if rc != _lib.SP_OK:
            raise RuntimeError(f"{what} failed ({rc}): {_lib.last_error()}")

    def graph(self, g):
        return device_graph(g, self.index)

    def offsets(self, g) -> np.ndarray:
        return np.asarray(g.offsets)

    # -- BC
    def bc(self, g, srcs, deterministic):
        t = self.torch
        n = g.n
        bc = t.zeros(max(1, n), dtype=t.float64, device=self.device)[:n]
        sg = t.zeros(max(1, n), dtype=t.float64, device=self.device)[:n]
        dl = t.zeros(max(1, n), dtype=t.float64, device=self.device)[:n]
        self._fence()
        if len(srcs):
            s = np.asarray(srcs, dtype=np.int32)
            flags = _lib.SP_FLAG_DETERMINISTIC if deterministic else 0
            st = _lib.Stats()
            rc = self.L.sp_bc(g.handle, s.ctypes.data_as(C.c_void_p), len(s), flags,
                              C.c_void_p(bc.data_ptr()), C.c_void_p(sg.data_ptr()),
                              C.c_void_p(dl.data_ptr()), _lib.SP_MEM_DEVICE, C.byref(st))
            self._chk(rc, "sp_bc")
            self.last_stats = st.as_dict()
        else:
            self.last_stats = {}
        return bc, sg, dl

    # -- TC
    def tc(self, g, v0, v1) -> int:
        self._fence()
        cnt = C.c_uint64()
        st = _lib.Stats()
        self._chk(self.L.sp_tc(g.handle, int(v0), int(v1), C.byref(cnt), C.byref(st)), "sp_tc")
        self.last_stats = st.as_dict()
        return int(cnt.value)

    # -- PR
    def pr_init(self, g, v0, v1):
        t = self.torch
        nb = max(1, v1 - v0)
        rank = t.empty(nb, dtype=t.float64, device=self.device)
        contrib = t.empty(nb, dtype=t.float64, device=self.device)
        self._fence()
        self._chk(self.L.sp_pagerank_block_init(g.handle, int(v0), int(v1),
                                                C.c_void_p(rank.data_ptr()),
                                                C.c_void_p(contrib.data_ptr())),
                  "sp_pagerank_block_init")
        return rank, contrib

    def pr_shard(self, g, v0, v1, damping, deterministic):
        return _NativePrShard(self, g, v0, v1, damping, deterministic)

    # -- SSSP (owner-computes shard, one handle per run)
    def sssp_shard(self, g, src, v0, v1, per, world, p2p=None):
        """p2p = (group, me): the exchange fused into the relaxation over
        peer-mapped dist arrays and inboxes (raises RuntimeError if the peer
        mapping fails)."""
        return _NativeShard(self, g, src, v0, v1, per, world, p2p)

    def to_host(self, x):
        return x.cpu().numpy()


class _NativePrShard:
    """sp_pagerank_shard_* planned once per run; every step is enqueued on
    torch's current stream (no host synchronisation: the exchange
    collectives that follow are ordered after it on the device)."""

    def __init__(self, be, g, v0, v1, damping, det):
        self.be = be
        self.h = C.c_void_p()
        flags = _lib.SP_FLAG_DETERMINISTIC if det else 0
        stream = be.torch.cuda.current_stream(be.device).cuda_stream
        be._fence()
        be._chk(be.L.sp_pagerank_shard_create(g.handle, int(v0), int(v1), float(damping), flags,
                                              C.c_void_p(stream), C.byref(self.h)),
                "sp_pagerank_shard_create")

    def step(self, contrib_full, rank, contrib, diff):
        self.be._chk(self.be.L.sp_pagerank_shard_step(
            self.h, C.c_void_p(contrib_full.data_ptr()), C.c_void_p(rank.data_ptr()),
            C.c_void_p(contrib.data_ptr()), C.c_void_p(diff.data_ptr())),
            "sp_pagerank_shard_step")

    # -- the contrib exchange fused into the step (peer stores over NVLink)
    def peer_setup(self, n, world, me, group):
        """Map every rank's two contrib arrays (one per iteration parity) into
        this process (CUDA IPC) and hand them to the shard; returns this
        rank's own two arrays as device pointers wrapped for reading."""
        dist = _dist()
        L, dev = self.be.L, self.be.index
        self.own, self.opened = [], []
        handles = []
        for _ in range(2):
            ptr, hnd = C.c_void_p(), (C.c_char * 64)()
            self.be._chk(L.sp_peer_alloc(dev, max(8, 8 * n), C.byref(ptr), hnd),
                         "sp_peer_alloc")
            self.own.append(ptr.value)
            handles.append(bytes(hnd))
        allh = [None] * world
        dist.all_gather_object(allh, handles, group=group)
        table = (C.c_void_p * (2 * world))()
        for s in range(2):
            for q in range(world):
                if q == me:
                    table[s * world + q] = self.own[s]
                else:
                    p = C.c_void_p()
                    hb = (C.c_char * 64).from_buffer_copy(allh[q][s])
                    self.be._chk(L.sp_peer_open(dev, hb, C.byref(p)), "sp_peer_open")
                    self.opened.append(p.value)
                    table[s * world + q] = p.value
        self.be._chk(L.sp_pagerank_shard_peers(self.h, 2, world, table),
                     "sp_pagerank_shard_peers")
        return self.own

    def step_peers(self, contrib_in_ptr, rank, contrib, diff, parity):
        self.be._chk(self.be.L.sp_pagerank_shard_step_peers(
            self.h, C.c_void_p(contrib_in_ptr), C.c_void_p(rank.data_ptr()),
            C.c_void_p(contrib.data_ptr()), C.c_void_p(diff.data_ptr()), int(parity)),
            "sp_pagerank_shard_step_peers")

    def close(self):
        if self.h:
            self.be.L.sp_pagerank_shard_destroy(self.h)
            self.h = C.c_void_p()
        for p in getattr(self, "opened", []):
            self.be.L.sp_peer_free(C.c_void_p(p), 1)
        for p in getattr(self, "own", []):
            self.be.L.sp_peer_free(C.c_void_p(p), 0)
        self.opened, self.own = [], []


class _DevArray:
    """A torch-visible view of a raw device pointer (__cuda_array_interface__)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


class _NativeShard:
    """sp_sssp_shard_* on this rank's GPU: dist (padded to per * world for a
    reduce-scatter) and the message send buffer are torch tensors.  With p2p
    = (group, me), dist, the inbox and its tail are peer-mapped buffers
    (sp_peer_alloc) shared with every rank, and the exchange is fused into
    the relaxation (sp_sssp_shard_peers / _collect)."""

    def __init__(self, be, g, src, v0, v1, per, world, p2p=None):
        t = be.torch
        self.be, self.g, self.world, self.per = be, g, world, per
        self.own, self.opened = [], []
        self.fused = p2p is not None
        self.h = C.c_void_p()
        L, dev = be.L, be.index
        if self.fused:
            group, me = p2p
            handles = []
            for nbytes in (4 * per * world, 4 * max(1, g.n), 8):  # dist, inbox, tail
                ptr, hnd = C.c_void_p(), (C.c_char * 64)()
                be._chk(L.sp_peer_alloc(dev, max(8, nbytes), C.byref(ptr), hnd), "sp_peer_alloc")
                self.own.append(ptr.value)
                handles.append(bytes(hnd))
            self.dist = t.as_tensor(_DevArray(self.own[0], per * world, "<i4"), device=be.device)
            self.dist.fill_(2147483647)
        else:
            self.dist = t.full((per * world,), 2147483647, dtype=t.int32, device=be.device)
        self.send = t.empty(max(1, g.n), dtype=t.int64, device=be.device)
        be._fence()
        be._chk(be.L.sp_sssp_shard_create(g.handle, int(v0), int(v1), int(src), int(world),
                                          C.c_void_p(self.dist.data_ptr()), C.byref(self.h)),
                "sp_sssp_shard_create")
        if self.fused:
            allh = [None] * world
            _dist().all_gather_object(allh, handles, group=group)
            tabs = [(C.c_void_p * world)() for _ in range(3)]
            for q in range(world):
                for i in range(3):
                    if q == me:
                        tabs[i][q] = self.own[i]
                    else:
                        ptr = C.c_void_p()
                        hb = (C.c_char * 64).from_buffer_copy(allh[q][i])
                        be._chk(L.sp_peer_open(dev, hb, C.byref(ptr)), "sp_peer_open")
                        self.opened.append(ptr.value)
                        tabs[i][q] = ptr.value
            be._chk(L.sp_sssp_shard_peers(self.h, int(per), tabs[0], tabs[1], tabs[2],
                                          C.c_void_p(self.own[1]), C.c_void_p(self.own[2])),
                    "sp_sssp_shard_peers")

    def collect(self) -> int:
        f = C.c_int64()
        self.be._chk(self.be.L.sp_sssp_shard_collect(self.h, C.byref(f)), "sp_sssp_shard_collect")
        return int(f.value)

    def relax(self, max_rounds):
        """-> (per-owner message counts, info[4]: owned expanded, slots
        relaxed, rounds, frontier left); raises OverflowError."""
        counts = np.zeros(self.world, dtype=np.int64)
        info = np.zeros(4, dtype=np.int64)
        self.be._fence()
        rc = self.be.L.sp_sssp_shard_relax(self.h, int(max_rounds), int(self.per),
                                           C.c_void_p(self.send.data_ptr()),
                                           counts.ctypes.data_as(C.c_void_p),
                                           info.ctypes.data_as(C.c_void_p))
        if rc == _lib.SP_ERR_OVERFLOW:
            raise OverflowError(_lib.last_error())
        self.be._chk(rc, "sp_sssp_shard_relax")
        return counts, info

    def apply(self, msgs=None, k=0, block=None) -> int:
        self.be._fence()
        f = C.c_int64()
        self.be._chk(self.be.L.sp_sssp_shard_apply(
            self.h, C.c_void_p(msgs.data_ptr()) if msgs is not None and k else None, int(k),
            C.c_void_p(block.data_ptr()) if block is not None else None, C.byref(f)),
            "sp_sssp_shard_apply")
        return int(f.value)

    def result(self):
        return self.be.to_host(self.dist[: self.g.n])

    def close(self):
        if self.h:
            self.be.L.sp_sssp_shard_destroy(self.h)
            self.h = C.c_void_p()
        for p in self.opened:
            self.be.L.sp_peer_free(C.c_void_p(p), 1)
        for p in self.own:
            self.be.L.sp_peer_free(C.c_void_p(p), 0)
        self.opened, self.own = [], []


def _dist():
    import torch.distributed as dist
    if not dist.is_initialized():
        raise RuntimeError("run_sharded needs an initialised torch.distributed process group")
    return dist


def _all_gather_flat(full, part, group):
    dist = _dist()
    if dist.get_backend(group) == "gloo":  # no all_gather_into_tensor on gloo
        chunks = list(full.chunk(dist.get_world_size(group)))
        dist.all_gather(chunks, part, group=group)
    else:
        dist.all_gather_into_tensor(full, part, group=group)


# ---------------------------------------------------------------------------
# superstep trace (the reference's bsp.Superstep / SimResult / TSV, bsp.py:75-103)


@dataclass
class Superstep:
    """One superstep of a sharded run, per rank (global rank -> count).

    local_updates: owned vertices whose property changed in the step (SSSP
    dist drops, PR ranks written, BC/TC: vertices processed); msgs_out: the
    values this rank contributed to the exchange after aggregation -- SSSP:
    remote vertices whose distance it lowered (one aggregated Min message
    per vertex, bsp.py:45-72), PR: its contrib slice (all-gather), BC: its
    bc partial (all-reduce), TC: its count."""
    index: int
    label: str
    local_updates: dict = field(default_factory=dict)
    msgs_out: dict = field(default_factory=dict)
    exchanged: int = 0
    finished: bool = False


@dataclass
class SimResult:
    result: RunResult
    supersteps: list


def format_trace_tsv(sim) -> str:
    """bsp.format_trace_tsv's layout (bsp.py:96-103)."""
    lines = ["superstep\trank\tlocal_updates\tmsgs_out\tfinished"]
    for step in sim.supersteps:
        for rank in sorted(step.local_updates):
            lines.append(f"{step.index}\t{rank}\t{step.local_updates[rank]}"
                         f"\t{step.msgs_out[rank]}"
                         f"\t{'true' if step.finished else 'false'}")
    return "\n".join(lines) + "\n"


class _Tracer:
    def __init__(self, enabled, be, group):
        self.on = enabled
        self.be = be
        self.group = group
        self.steps: list[Superstep] = []

    def record(self, label, local_updates, msgs_out, finished=False):
        if not self.on:
            return
        dist = _dist()
        t = self.be.torch.tensor([int(local_updates), int(msgs_out)],
                                 dtype=self.be.torch.int64, device=self.be.device)
        parts = [self.be.torch.zeros_like(t) for _ in range(dist.get_world_size(self.group))]
        dist.all_gather(parts, t, group=self.group)
        ranks = [dist.get_global_rank(self.group, r) if self.group is not None else r
                 for r in range(len(parts))]
        lu = {rk: int(p[0].item()) for rk, p in zip(ranks, parts)}
        mo = {rk: int(p[1].item()) for rk, p in zip(ranks, parts)}
        self.steps.append(Superstep(len(self.steps), label, lu, mo, sum(mo.values()),
                                    bool(finished)))

    def finish_last(self):
        if self.on and self.steps:
            self.steps[-1].finished = True


def simulate(tp, g, nranks: int, args: dict, function: str | None = None,
             max_iters: int | None = None, *, backend=None, group=None,
             deterministic: bool = False, local_fixpoint: bool = False) -> SimResult:
    """bsp.simulate's surface (bsp.py:452-465) over real ranks: nranks must
    equal the process group's size (one rank per GPU); returns the run's
    result and its superstep trace (convergence evaluated after the
    exchange, unlike bsp.py:393-417 -- SURVEY F4).  local_fixpoint: SSSP
    ranks relax their owned frontier to a local fixpoint before each
    exchange (bsp.py:297-306)."""
    dist = _dist()
    if nranks != dist.get_world_size(group):
        raise ValueError(f"simulate: nranks={nranks} but the process group has "
                         f"{dist.get_world_size(group)} ranks (one rank per GPU)")
    r = run_sharded(tp, g, args, function, max_iters, backend=backend, group=group,
                    deterministic=deterministic, trace=True, local_fixpoint=local_fixpoint)
    return SimResult(result=r, supersteps=r.supersteps)


def tc_ranges(offsets: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous vertex ranges with about equal sum of squared degrees (the
    per-vertex intersection work grows with deg^2); covers [0, n) exactly."""
    deg = np.diff(np.asarray(offsets, dtype=np.int64)).astype(np.float64)
    n = len(deg)
    w = np.cumsum(deg * deg + 1.0)
    tot = w[-1] if n else 0.0
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(w, tot * r / world, side="left")) if n else 0)
    cuts.append(n)
    for i in range(1, len(cuts)):  # monotone even for degenerate inputs
        cuts[i] = max(cuts[i], cuts[i - 1])
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


def run_sharded(tp, g, args: dict, function: str | None = None,
                max_iters: int | None = None, *, backend=None, group=None,
                deterministic: bool = False, trace: bool = False,
                local_fixpoint: bool = False) -> RunResult:
    """Run a corpus program over all ranks of ``group`` (default: the world).
    Every rank must call it with the same graph and arguments.  trace=True
    records the superstep trace in ``result.supersteps`` (one extra small
    all-gather per superstep).  local_fixpoint (SSSP): relax the owned
    frontier to a local fixpoint between exchanges (bsp.py:297-306) --
    fewer supersteps, same dist."""
    dist = _dist()
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    if backend is None:
        import torch
        backend = NativeBackend(torch.cuda.current_device())
    E = errors_for(tp)
    prog = corpus.identify(tp, function)
    dg = backend.graph(g)
    bound = check_args(prog, dg, args, E)
    cap = max_iters if max_iters is not None else default_iteration_cap(dg.n)
    t0 = time.perf_counter()
    fn = {"sssp": _sssp, "sssp_pull": _sssp, "pr": _pr, "bc": _bc, "tc": _tc}[prog.key]
    tr = _Tracer(trace, backend, group)
    kw = {"local_fixpoint": local_fixpoint} if fn is _sssp else {}
    env, fpi, stats = fn(backend, dg, bound, cap, world, me, group, deterministic, E, prog, tr,
                         **kw)
    r = RunResult(env=env, fixedpoint_iterations=fpi,
                  wall_seconds=time.perf_counter() - t0, stats=stats)
    r.supersteps = tr.steps if trace else None
    return r


def _reduce_scatter_min(out, full, group):
    dist = _dist()
    if dist.get_backend(group) == "gloo":  # no reduce_scatter on gloo
        t = full.clone()
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        me = dist.get_rank(group)
        out.copy_(t[me * out.numel():(me + 1) * out.numel()])
    else:
        dist.reduce_scatter_tensor(out, full, op=dist.ReduceOp.MIN, group=group)


def _sum_stats(be, keys, group):
    """Counters of this rank's last native call, summed over the ranks."""
    dist = _dist()
    st = getattr(be, "last_stats", {}) or {}
    t = be.torch.tensor([float(st.get(k, 0)) for k in keys], dtype=be.torch.float64,
                        device=be.device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return {k: int(v) for k, v in zip(keys, t.tolist())}


def _bc(be, g, bound, cap, world, me, group, det, E, prog, tr):
    dist = _dist()
    srcs = bound["sourceSet"]
    mine = srcs[me::world]
    bc, sg, dl = be.bc(g, mine, det)
    tr.record("bc sources", len(mine), g.n if mine else 0, finished=True)
    dist.all_reduce(bc, op=dist.ReduceOp.SUM, group=group)
    env = PropertyEnv()
    env.node_props = {"bc": be.to_host(bc)}
    if srcs:
        owner = (len(srcs) - 1) % world  # ran the last source of the list
        glob = dist.get_global_rank(group, owner) if group is not None else owner
        dist.broadcast(sg, src=glob, group=group)
        dist.broadcast(dl, src=glob, group=group)
        env.node_props.update(sigma=be.to_host(sg), delta=be.to_host(dl))
    stats = _sum_stats(be, ("edges_visited", "vertices_visited", "model_bytes"), group)
    stats["sources_local"] = len(mine)
    return env, {}, stats


def _tc(be, g, bound, cap, world, me, group, det, E, prog, tr):
    dist = _dist()
    v0, v1 = tc_ranges(be.offsets(g), world)[me]
    part = be.tc(g, v0, v1)
    tr.record("tc range", v1 - v0, 1, finished=True)
    t = be.torch.tensor([part], dtype=be.torch.int64, device=be.device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    env = PropertyEnv(scalars={"triangle_count": int(t.item())})
    stats = _sum_stats(be, ("edges_visited", "model_bytes"), group)
    stats.update(range=(v0, v1), local_count=part)
    return env, {}, stats


def _pr(be, g, bound, cap, world, me, group, det, E, prog, tr):
    dist = _dist()
    torch = be.torch
    parts = block_partition(g, world)
    per = parts[0].size
    rr = parts[me].real_range()
    v0, v1 = rr.start, rr.stop
    rank_l, contrib_l = be.pr_init(g, v0, v1)
    slice_l = torch.zeros(per, dtype=torch.float64, device=be.device)
    full = torch.zeros(per * world, dtype=torch.float64, device=be.device)

    def gather():
        slice_l.zero_()
        if v1 > v0:
            slice_l[: v1 - v0] = contrib_l[: v1 - v0]
        _all_gather_flat(full, slice_l, group)

    gather()
    it = 0
    iters = 0
    diff = 0.0
    dt = torch.zeros(1, dtype=torch.float64, device=be.device)
    sh = be.pr_shard(g, v0, v1, bound["damping"], det)  # planned once per run
    # the contrib exchange: fused into the step as peer stores (each rank's
    # epilogue writes its contribs straight into every rank's array for the
    # next iteration, NVLink on a multi-GPU box) or, SP_PR_EXCHANGE=nccl /
    # backends without peer mapping, an all-gather after the step
    p2p = (world > 1 and hasattr(sh, "peer_setup")
           and os.environ.get("SP_PR_EXCHANGE", "p2p") != "nccl")
    if p2p:  # iteration 1 reads the initial all-gather (`full`), then sets 1, 0, 1, ...
        try:
            arrays = sh.peer_setup(g.n, world, me, group)
            ok = 1
        except RuntimeError:  # e.g. no peer access / IPC between these processes
            ok = 0
        okt = torch.tensor([ok], dtype=torch.int32, device=be.device)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN, group=group)  # every rank or none
        if not int(okt.item()):
            p2p = False
            sh.close()
            sh = be.pr_shard(g, v0, v1, bound["damping"], det)
    try:
        while True:
            # the step, the max-reduce of diff and the contrib exchange are
            # all queued on the device; the convergence test is the
            # iteration's one host read
            if p2p:
                # reads set it % 2, stores into every rank's set (it + 1) % 2;
                # the diff all-reduce orders every rank's stores before any
                # rank's next step
                sh.step_peers(arrays[it % 2] if it else full.data_ptr(), rank_l, contrib_l,
                              dt, (it + 1) % 2)
                dist.all_reduce(dt, op=dist.ReduceOp.MAX, group=group)
            else:
                sh.step(full, rank_l, contrib_l, dt)
                dist.all_reduce(dt, op=dist.ReduceOp.MAX, group=group)
                gather()
            diff = float(dt.item())
            it += 1
            iters += 1
            done = diff < bound["epsilon"] or it >= bound["maxIter"]  # pr.sp:10
            tr.record("fixedPoint converged", v1 - v0, v1 - v0, finished=done)
            if done:
                break
            if iters >= cap:
                raise E.NonConvergenceError(prog.flag, cap)
    finally:
        sh.close()
    # ranks back to every rank (owned slices, padded to per)
    rl = torch.zeros(per, dtype=torch.float64, device=be.device)
    if v1 > v0:
        rl[: v1 - v0] = rank_l[: v1 - v0]
    rfull = torch.zeros(per * world, dtype=torch.float64, device=be.device)
    _all_gather_flat(rfull, rl, group)
    rank = be.to_host(rfull)[: g.n].copy()
    env = PropertyEnv(node_props={"rank": rank, "rank_nxt": rank.copy()},
                      scalars={"iter": it, "diff": diff, "converged": True})
    return env, {"converged": iters}, {"block": (v0, v1)}


def _sssp(be, g, bound, cap, world, me, group, det, E, prog, tr, local_fixpoint=False):
    """Owner-computes supersteps: local relaxation (one pass, or passes to a
    local fixpoint, bsp.py:297-306), aggregated min-messages exchanged with
    one all-to-all (sparse supersteps) or a MIN reduce-scatter of the dist
    arrays (dense ones), owner apply, then ONE all-reduce of the frontier
    sizes: fixedPoint finishes when no rank has a frontier after the
    exchange, and the cap is tested only after that
    (bsp.py:402-415)."""
    dist = _dist()
    torch = be.torch
    parts = block_partition(g, world)
    per = parts[0].size
    rr = parts[me].real_range()
    v0, v1 = rr.start, rr.stop
    n = g.n
    # the exchange fused into the relaxation over peer memory (NVLink between
    # GPUs) unless SP_SSSP_EXCHANGE forces a message form or the mapping
    # fails on any rank (decided collectively)
    mode = os.environ.get("SP_SSSP_EXCHANGE", "auto")
    sh = None
    if world > 1 and mode in ("auto", "p2p") and hasattr(be, "sssp_shard") and \
            isinstance(be, NativeBackend):
        try:
            sh = be.sssp_shard(g, bound["src"], v0, v1, per, world, p2p=(group, me))
            ok = 1
        except RuntimeError:
            ok = 0
        okt = torch.tensor([ok], dtype=torch.int32, device=be.device)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN, group=group)
        if not int(okt.item()) and sh is not None:
            sh.close()
            sh = None
        elif not int(okt.item()):
            sh = None
    if sh is None:
        sh = be.sssp_shard(g, bound["src"], v0, v1, per, world)
    fused = getattr(sh, "fused", False)
    try:
        steps = relaxed = sent_total = 0
        dense_steps = 0
        while True:
            try:
                counts, info = sh.relax(cap if local_fixpoint else 1)
                bad = 0
            except OverflowError:
                counts, info, bad = np.zeros(world, dtype=np.int64), np.zeros(4, np.int64), 1
            relaxed += int(info[1])
            if fused:  # messages already in the owners' inboxes
                okt = torch.tensor([bad], dtype=torch.int64, device=be.device)
                dist.all_reduce(okt, op=dist.ReduceOp.MAX, group=group)  # + every relax done
                if int(okt.item()):
                    raise E.ExecError("SSSP distance left the int32 range (negative weights)")
                sent_total += int(counts.sum())
                f = sh.collect()
                steps += 1
                ft = torch.tensor([f], dtype=torch.int64, device=be.device)
                dist.all_reduce(ft, op=dist.ReduceOp.SUM, group=group)
                done = int(ft.item()) == 0
                tr.record("fixedPoint finished", int(info[0]), int(counts.sum()), finished=done)
                if done:
                    break
                if steps >= cap:
                    raise E.NonConvergenceError(prog.flag, cap)
                continue
            # every rank's per-owner counts (+ overflow flag): the send and
            # receive splits of the all-to-all and the global message volume
            row = torch.tensor(list(counts) + [bad], dtype=torch.int64, device=be.device)
            allc = [torch.zeros_like(row) for _ in range(world)]
            dist.all_gather(allc, row, group=group)
            M = torch.stack(allc).cpu().numpy()
            if M[:, world].any():
                raise E.ExecError("SSSP distance left the int32 range (negative weights)")
            total = int(M[:, :world].sum())
            sent_total += int(counts.sum())
            # message forms (tests force each with SP_SSSP_EXCHANGE)
            dense = mode == "dense" or (mode in ("auto", "p2p") and 8 * total > 4 * per * world)
            if dense:  # a MIN reduce-scatter of the dist arrays moves fewer bytes
                dense_steps += 1
                blk = torch.empty(per, dtype=torch.int32, device=be.device)
                _reduce_scatter_min(blk, sh.dist, group)
                f = sh.apply(block=blk[: v1 - v0] if v1 > v0 else blk)
            elif total:
                send_splits = [int(x) for x in M[me, :world]]
                recv_splits = [int(x) for x in M[:, me]]
                recv = torch.empty(max(1, sum(recv_splits)), dtype=torch.int64, device=be.device)
                dist.all_to_all_single(recv[: sum(recv_splits)], sh.send[: sum(send_splits)],
                                       recv_splits, send_splits, group=group)
                f = sh.apply(recv, sum(recv_splits))
            else:
                f = sh.apply()
            steps += 1
            ft = torch.tensor([f], dtype=torch.int64, device=be.device)
            dist.all_reduce(ft, op=dist.ReduceOp.SUM, group=group)
            done = int(ft.item()) == 0
            tr.record("fixedPoint finished", int(info[0]), int(counts.sum()), finished=done)
            if done:
                break
            if steps >= cap:
                raise E.NonConvergenceError(prog.flag, cap)
        # owned blocks back to every rank
        mine = torch.full((per,), 2147483647, dtype=torch.int32, device=be.device)
        mine[: v1 - v0] = sh.dist[v0:v1]
        full = torch.empty(per * world, dtype=torch.int32, device=be.device)
        _all_gather_flat(full, mine, group)
        d = be.to_host(full)[:n].copy()
    finally:
        sh.close()
    env = PropertyEnv(node_props={"dist": d, "modified": np.zeros(n, dtype=bool),
                                  "modified_nxt": np.zeros(n, dtype=bool)},
                      scalars={"finished": True})
    return env, {"finished": steps}, {"relaxed": relaxed, "block": (v0, v1),
                                      "messages": sent_total, "dense_supersteps": dense_steps,
                                      "exchange": "peer" if fused else "messages"}
