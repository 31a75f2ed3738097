"""Device-resident CSR graphs: the drop-in for trident/graph.py.

Same entry points and argument meaning as the reference --
``from_edges`` (graph.py:101-116), ``load_edge_list`` (119-151),
``assign_random_weights`` (154-190), ``Partition`` / ``block_partition`` /
``owner_of`` (193-249), ``min_wt`` / ``max_wt`` (252-261),
``write_edge_list`` (264-272) -- but the CSR is built ON THE GPU by
libstarplat_b200.so (stable radix sort, reverse CSR, w_eff) and stays
resident there: uploaded once, never copied back for the algorithms
(the reference's transfer plan H2D_ONCE, trident/sema.py:773-774).

``CsrGraph`` keeps the reference's attribute names; the arrays
(``offsets``, ``adj``, ``weights``, ``rev_offsets``, ``rev_adj``,
``rev_eid``) are NumPy views downloaded lazily on first access -- host
inspection only, never on the hot path.  A reference ``trident`` CsrGraph
can be handed to ``run`` directly; ``device_graph`` uploads it once and
caches the device copy for the object's lifetime.
"""

from __future__ import annotations

import ctypes as C
import random
import threading
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import (ArgError, BackendError, EmptyGraphError, FormatError,
                     GraphIoError, RangeError)

_I32_MIN, _I32_MAX = -(2 ** 31), 2 ** 31 - 1


def _check(rc: int, what: str):
    if rc == _lib.SP_OK:
        return
    msg = _lib.last_error()
    if rc == _lib.SP_ERR_ARG:
        raise ArgError(f"{what}: {msg}")
    if rc == _lib.SP_ERR_UNSUPPORTED:
        raise ArgError(f"{what}: unsupported input: {msg}")
    if rc == _lib.SP_ERR_OOM:
        raise MemoryError(f"{what}: device out of memory: {msg}")
    raise BackendError(f"{what} failed ({rc}): {msg}")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class CsrGraph:
    """Forward + reverse CSR with edge weights, resident on one GPU.

    Mirrors trident/graph.py:18-65 (fields n, m, offsets, adj, weights,
    rev_offsets, rev_adj, rev_eid, directed and the accessor methods).
    Immutable and safe for concurrent readers.
    """

    def __init__(self, handle: C.c_void_p, device: int = 0):
        self._h = handle
        self.device = device
        n = C.c_int64()
        m = C.c_int64()
        d = C.c_int()
        _check(_lib.lib().sp_graph_info(handle, C.byref(n), C.byref(m), C.byref(d)),
               "sp_graph_info")
        self.n = int(n.value)
        self.m = int(m.value)
        self.directed = bool(d.value)
        self._cache: dict[int, np.ndarray] = {}
        self._lock = threading.Lock()
        self._finalizer = weakref.finalize(self, _destroy, handle)

    # -- native handle ----------------------------------------------------
    @property
    def handle(self) -> C.c_void_p:
        if self._h is None:
            raise ValueError("graph has been closed")
        return self._h

    def close(self) -> None:
        """Free the device arrays now (otherwise at garbage collection)."""
        if self._h is not None:
            self._finalizer()
            self._h = None

    def preprocessing_ms(self) -> dict:
        """Device time (ms) of each one-time per-graph structure built so far
        by the first call that needed it (degree-ordered upper CSR for TC,
        w_eff, PR hot-source encoding / relabelled layout, ...); structures
        not built (or built during the upload) are omitted.  No reference
        counterpart: a measurement aid (sp_graph_prep_ms)."""
        out = {}
        ms = C.c_double(-1.0)
        for kind, name in enumerate(_lib.PREP_KINDS):
            _check(_lib.lib().sp_graph_prep_ms(self.handle, kind, C.byref(ms)),
                   "sp_graph_prep_ms")
            if ms.value >= 0:
                out[name] = ms.value
        return out

    # -- lazily downloaded host views (graph.py:28-36) ----------------------
    def _array(self, which: int, dtype, count: int) -> np.ndarray:
        with self._lock:
            a = self._cache.get(which)
            if a is None:
                a = np.empty(count, dtype=dtype)
                if count:
                    _check(_lib.lib().sp_graph_download(self.handle, which, _ptr(a)),
                           "sp_graph_download")
                a.setflags(write=False)
                self._cache[which] = a
            return a

    @property
    def offsets(self) -> np.ndarray:
        return self._array(_lib.SP_ARR_OFFSETS, np.int64, self.n + 1)

    @property
    def adj(self) -> np.ndarray:
        return self._array(_lib.SP_ARR_ADJ, np.int32, self.m)

    @property
    def weights(self) -> np.ndarray:
        return self._array(_lib.SP_ARR_WEIGHTS, np.int32, self.m)

    @property
    def rev_offsets(self) -> np.ndarray:
        return self._array(_lib.SP_ARR_REV_OFFSETS, np.int64, self.n + 1)

    @property
    def rev_adj(self) -> np.ndarray:
        return self._array(_lib.SP_ARR_REV_ADJ, np.int32, self.m)

    @property
    def rev_eid(self) -> np.ndarray:
        return self._array(_lib.SP_ARR_REV_EID, np.int64, self.m)

    @property
    def effective_weights(self) -> np.ndarray:
        """w_eff[e]: weight of the first slot u->v (get_edge semantics)."""
        return self._array(_lib.SP_ARR_WEFF, np.int32, self.m)

    # -- accessors (graph.py:38-65) -----------------------------------------
    def degree(self, v: int) -> int:
        o = self.offsets
        return int(o[v + 1] - o[v])

    def in_degree(self, v: int) -> int:
        o = self.rev_offsets
        return int(o[v + 1] - o[v])

    def neighbors(self, v: int) -> list[int]:
        o = self.offsets
        return self.adj[o[v]:o[v + 1]].tolist()

    def in_neighbors(self, v: int) -> list[int]:
        o = self.rev_offsets
        return self.rev_adj[o[v]:o[v + 1]].tolist()

    def out_edges(self, v: int) -> range:
        o = self.offsets
        return range(int(o[v]), int(o[v + 1]))

    def in_slots(self, v: int) -> range:
        o = self.rev_offsets
        return range(int(o[v]), int(o[v + 1]))

    def find_edge(self, u: int, v: int) -> int | None:
        """First forward edge index for u->v, or None (graph.py:56-62)."""
        o = self.offsets
        lo, hi = int(o[u]), int(o[u + 1])
        k = lo + int(np.searchsorted(self.adj[lo:hi], v, side="left"))
        if k < hi and int(self.adj[k]) == v:
            return k
        return None

    def has_edge(self, u: int, v: int) -> bool:
        return self.find_edge(u, v) is not None

    def __repr__(self):
        return (f"CsrGraph(n={self.n}, m={self.m}, directed={self.directed}, "
                f"device=cuda:{self.device})")


def _destroy(handle):
    try:
        _lib.lib().sp_graph_destroy(handle)
    except Exception:  # interpreter shutdown
        pass


def _new_handle(fn, *args, what: str) -> C.c_void_p:
    h = C.c_void_p()
    _check(fn(*args, C.byref(h)), what)
    return h


# ---------------------------------------------------------------------------
# construction


def _as_i32(a, what: str) -> np.ndarray:
    """int32 copy/view of an integer array; values outside int32 and
    non-integral values are rejected (never truncated or wrapped)."""
    a = np.asarray(a)
    if a.dtype == np.int32:  # already in range: no O(m) host scan
        return np.ascontiguousarray(a)
    if a.size and a.dtype.kind == "f":
        if not np.all(np.isfinite(a)) or not np.all(a == np.floor(a)):
            raise ArgError(f"{what} must be integers (got non-integral {a.dtype} values)")
    elif a.size and a.dtype.kind not in "iub":
        raise ArgError(f"{what} must be integers (got dtype {a.dtype})")
    if a.size and a.dtype.kind in "iuf":
        lo, hi = a.min(), a.max()
        if lo < _I32_MIN or hi > _I32_MAX:
            raise ArgError(f"{what} outside the int32 range [{lo}, {hi}] "
                           "(unsupported by the B200 backend)")
    return np.ascontiguousarray(a, dtype=np.int32)


def from_arrays(u, v, w=None, directed: bool = True, default_weight: int = 1,
                n: int | None = None, device: int = 0, _nonneg: bool = False) -> CsrGraph:
    """Array form of ``from_edges``: edge i is (u[i], v[i], w[i])."""
    u = _as_i32(u, "vertex id")
    v = _as_i32(v, "vertex id")
    if len(u) != len(v):
        raise ArgError("u and v differ in length")
    if w is None:
        w = np.full(len(u), default_weight, dtype=np.int64)
    w = _as_i32(w, "edge weight")
    if len(u) and not _nonneg and (int(u.min()) < 0 or int(v.min()) < 0):
        raise ArgError("negative vertex id in edge list")
    _lib.require_device(device)
    L = _lib.lib()
    h = _new_handle(L.sp_graph_from_edges, _ptr(u), _ptr(v), _ptr(w), len(u),
                    -1 if n is None else int(n), int(bool(directed)),
                    _lib.SP_MEM_HOST, device, what="sp_graph_from_edges")
    return CsrGraph(h, device)


def from_edges(edges, directed: bool = True, default_weight: int = 1,
               n: int | None = None, device: int = 0) -> CsrGraph:
    """Build a graph from (u, v[, w]) tuples; n defaults to 1 + max id
    (graph.py:101-116).  Slot order, stable (src, dst) sort, undirected
    mirroring of non-loop edges and the reverse CSR match the reference."""
    edges = list(edges)
    u = np.fromiter((t[0] for t in edges), dtype=np.int64, count=len(edges))
    v = np.fromiter((t[1] for t in edges), dtype=np.int64, count=len(edges))
    w = np.fromiter((t[2] if len(t) == 3 else default_weight for t in edges),
                    dtype=np.int64, count=len(edges))
    return from_arrays(u, v, w, directed=directed, n=n, device=device)


def load_edge_list(path: str, directed: bool = True,
                   default_weight: int = 1, device: int = 0) -> CsrGraph:
    """Whitespace-separated ``u v [w]`` edge list (graph.py:119-151): 0-based
    ids, ``#`` and blank lines skipped, duplicates kept; raises GraphIoError /
    FormatError(lineno) exactly where the reference does.  The text is parsed
    by the native multithreaded loader (sp_graph_from_edge_text); non-ASCII
    text or values outside int32 take the reference's Python parsing path."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise GraphIoError(f"cannot read graph file {path!r}: {e}") from e
    if _I32_MIN <= int(default_weight) <= _I32_MAX:
        L = _lib.lib()
        info = (C.c_int64 * 8)()
        blk = C.POINTER(C.c_int32)()
        rc = L.sp_parse_edge_text(data, len(data), int(default_weight), 0, C.byref(blk), info)
        if rc == _lib.SP_OK:
            try:
                ne, stride = int(info[6]), int(info[7])
                a = np.ctypeslib.as_array(blk, shape=(3 * stride,))
                return from_arrays(a[:ne], a[stride:stride + ne], a[2 * stride:2 * stride + ne],
                                   directed=directed, device=device, _nonneg=True)
            finally:
                L.sp_free_host(blk)
        if rc == _lib.SP_ERR_ARG and info[0] in (1, 2, 3):
            _raise_format_error(data, int(info[0]), int(info[1]))
        if rc != _lib.SP_ERR_UNSUPPORTED:
            _check(rc, "sp_parse_edge_text")
    return _load_edge_list_py(_py_lines(data), directed, default_weight, device)


def _py_lines(data: bytes) -> list[str]:
    """The lines f.readlines() yields in text mode (universal newlines)."""
    text = data.decode("utf-8").replace("\r\n", "\n").replace("\r", "\n")
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    return lines


def _raise_format_error(data: bytes, kind: int, lineno: int):
    """The reference's FormatError for line `lineno` (messages built from
    the line text exactly as graph.py:134-148 does)."""
    stripped = _py_lines(data)[lineno - 1].strip()
    if kind == 1:
        raise FormatError(lineno, f"expected 2 or 3 fields, got {len(stripped.split())}")
    if kind == 2:
        raise FormatError(lineno, f"non-integer field in {stripped!r}")
    raise FormatError(lineno, f"negative vertex id in {stripped!r}")


def _load_edge_list_py(lines, directed, default_weight, device) -> CsrGraph:
    us: list[int] = []
    vs: list[int] = []
    ws: list[int] = []
    for lineno, line in enumerate(lines, start=1):
        s = line.strip()
        if not s or s.startswith("#"):
            continue
        fields = s.split()
        if len(fields) not in (2, 3):
            raise FormatError(lineno, f"expected 2 or 3 fields, got {len(fields)}")
        try:
            a = int(fields[0])
            b = int(fields[1])
            c = int(fields[2]) if len(fields) == 3 else default_weight
        except ValueError:
            raise FormatError(lineno, f"non-integer field in {s!r}") from None
        if a < 0 or b < 0:
            raise FormatError(lineno, f"negative vertex id in {s!r}")
        us.append(a)
        vs.append(b)
        ws.append(c)
    return from_arrays(_ints(us, "vertex id"), _ints(vs, "vertex id"),
                       _ints(ws, "edge weight"), directed=directed, device=device)


def _ints(vals: list[int], what: str) -> np.ndarray:
    """int64 array of Python ints; values the backend cannot hold raise the
    same ArgError as _as_i32."""
    if vals and (min(vals) < _I32_MIN or max(vals) > _I32_MAX):
        raise ArgError(f"{what} outside the int32 range [{min(vals)}, {max(vals)}] "
                       "(unsupported by the B200 backend)")
    return np.array(vals, dtype=np.int64)


def from_csr(offsets, adj, weights=None, directed: bool = True,
             device: int = 0) -> CsrGraph:
    """Wrap an existing forward CSR (rows already in reference order, e.g. a
    trident CsrGraph's lists); the reverse CSR and w_eff are built on the
    device.  weights=None: an unweighted graph (every slot weight 1, filled
    on the device; nothing is uploaded for it)."""
    off = np.ascontiguousarray(np.asarray(offsets), dtype=np.int64)
    adj = _as_i32(adj, "vertex id")
    w = None if weights is None else _as_i32(weights, "edge weight")
    n = len(off) - 1
    # O(1) shape checks here; row monotonicity and 0 <= adj < n are checked
    # on the device before any kernel indexes by them (sp_graph_from_csr)
    if n < 0:
        raise ArgError("offsets must hold n + 1 >= 1 entries")
    if int(off[0]) != 0 or int(off[-1]) != len(adj):
        raise ArgError(f"offsets must start at 0 and end at len(adj) = {len(adj)} "
                       f"(got {int(off[0])} .. {int(off[-1])})")
    if w is not None and len(w) != len(adj):
        raise ArgError(f"weights ({len(w)}) and adj ({len(adj)}) differ in length")
    _lib.require_device(device)
    h = _new_handle(_lib.lib().sp_graph_from_csr, _ptr(off), _ptr(adj),
                    None if w is None else _ptr(w), n, len(adj), int(bool(directed)),
                    _lib.SP_MEM_HOST, device, what="sp_graph_from_csr")
    return CsrGraph(h, device)


def generate(kind: str, p0: int, p1: int, seed: int = 1,
             undirected: bool = False, device: int = 0) -> CsrGraph:
    """Seeded synthetic graph generated on the device, bit-identical to
    ``paper_2305_03317_b200.gen`` (kind: 'rmat' (scale, edge factor),
    'uniform' (n, candidate edges), 'grid' (rows, cols))."""
    k = {"rmat": _lib.SP_GEN_RMAT, "uniform": _lib.SP_GEN_UNIFORM,
         "grid": _lib.SP_GEN_GRID}[kind]
    _lib.require_device(device)
    h = _new_handle(_lib.lib().sp_graph_generate, k, int(p0), int(p1), int(seed),
                    int(bool(undirected)), device, what="sp_graph_generate")
    return CsrGraph(h, device)


# ---------------------------------------------------------------------------
# reference-graph adoption

_adopted: dict[int, tuple] = {}
_adopt_lock = threading.Lock()


def device_graph(g, device: int | None = None) -> CsrGraph:
    """The device-resident form of ``g`` on ``device``: ``g`` itself for a
    CsrGraph of this package on that device (a graph on another device is
    an error: its arrays live in that GPU's memory), else a one-time upload
    of a reference ``trident`` CsrGraph, cached per (object, device) while
    the source object lives."""
    if isinstance(g, CsrGraph):
        if device is not None and g.device != device:
            raise ArgError(f"graph lives on cuda:{g.device}, not cuda:{device}")
        return g
    if device is None:
        device = 0
    key = (id(g), device)
    with _adopt_lock:
        ent = _adopted.get(key)
        if ent is not None and ent[0]() is g:
            return ent[1]
    dg = from_csr(g.offsets, g.adj, g.weights, directed=getattr(g, "directed", True),
                  device=device)
    with _adopt_lock:
        try:
            ref = weakref.ref(g, lambda _r, k=key: _adopted.pop(k, None))
        except TypeError:  # not weak-referenceable: no caching
            return dg
        _adopted[key] = (ref, dg)
    return dg


# ---------------------------------------------------------------------------
# utilities of trident/graph.py that are not on the device path


def random_weights(offsets, adj, directed: bool, lo: int, hi: int, seed: int) -> np.ndarray:
    """The weight array ``assign_random_weights`` gives a CSR (host only):
    Python's Mersenne Twister seeded with ``seed``, ``randint(lo, hi)`` per
    slot in slot order when directed (graph.py:163-167); when undirected one
    draw per canonical (u <= v) slot in CSR order, mirrored onto the k-th
    reverse copy of the same pair by position (graph.py:168-187)."""
    if lo > hi:
        raise RangeError(f"lo ({lo}) exceeds hi ({hi})")
    rng = random.Random(seed)
    off = np.asarray(offsets).tolist()
    adj = np.asarray(adj).tolist()
    m = len(adj)
    if directed:
        return np.fromiter((rng.randint(lo, hi) for _ in range(m)), dtype=np.int64, count=m)
    w = [0] * m
    pending: dict[tuple[int, int], list[int]] = {}
    for x in range(len(off) - 1):
        for e in range(off[x], off[x + 1]):
            y = adj[e]
            if x <= y:
                val = rng.randint(lo, hi)
                w[e] = val
                if x != y:
                    pending.setdefault((y, x), []).append(val)
    seen: dict[tuple[int, int], int] = {}
    for x in range(len(off) - 1):
        for e in range(off[x], off[x + 1]):
            y = adj[e]
            if x > y:
                k = seen.get((x, y), 0)
                seen[(x, y)] = k + 1
                w[e] = pending[(x, y)][k]
    return np.asarray(w, dtype=np.int64)


def assign_random_weights(g: CsrGraph, lo: int, hi: int, seed: int) -> CsrGraph:
    """i.i.d. uniform integer weights in [lo, hi] (graph.py:154-190; see
    ``random_weights`` for the draw order).  Returns a new device graph."""
    w = random_weights(g.offsets, g.adj, g.directed, lo, hi, seed)
    return from_csr(g.offsets, g.adj, w, directed=g.directed, device=g.device)


@dataclass(frozen=True)
class Partition:
    """One rank's contiguous block of the padded vertex range
    (graph.py:193-223); a rank is one GPU here."""

    rank: int
    nranks: int
    local_begin: int
    local_end: int
    n: int
    padded: int = field(default=0)

    @property
    def size(self) -> int:
        return self.local_end - self.local_begin

    def owns(self, v: int) -> bool:
        return self.local_begin <= v < self.local_end

    def real_range(self) -> range:
        return range(min(self.local_begin, self.n), min(self.local_end, self.n))

    def to_local(self, v: int) -> int:
        if not self.owns(v):
            raise ArgError(f"vertex {v} not owned by rank {self.rank}")
        return v - self.local_begin

    def to_global(self, lv: int) -> int:
        if not 0 <= lv < self.size:
            raise ArgError(f"local id {lv} out of range on rank {self.rank}")
        return lv + self.local_begin


def block_partition(g, nranks: int) -> list[Partition]:
    """ceil(n/k) vertices per rank over the id space padded to a multiple of
    k; padding only at the tail (graph.py:226-244)."""
    if nranks < 1:
        raise ArgError(f"nranks must be >= 1, got {nranks}")
    n = g.n
    per = -(-n // nranks) if n else 0
    parts = []
    for r in range(nranks):
        b, e = r * per, (r + 1) * per
        parts.append(Partition(rank=r, nranks=nranks, local_begin=b, local_end=e,
                               n=n, padded=max(0, e - max(n, b))))
    return parts


def owner_of(v: int, nranks: int, n: int) -> int:
    """Rank owning vertex v under block_partition (graph.py:247-249)."""
    return v // (-(-n // nranks))


def min_wt(g: CsrGraph) -> int:
    if g.m == 0:
        raise EmptyGraphError("minWt on a graph with no edges")
    lo = C.c_int32()
    _check(_lib.lib().sp_graph_weight_range(g.handle, C.byref(lo), None),
           "sp_graph_weight_range")
    return int(lo.value)


def max_wt(g: CsrGraph) -> int:
    if g.m == 0:
        raise EmptyGraphError("maxWt on a graph with no edges")
    hi = C.c_int32()
    _check(_lib.lib().sp_graph_weight_range(g.handle, None, C.byref(hi)),
           "sp_graph_weight_range")
    return int(hi.value)


def write_edge_list(g: CsrGraph, path: str) -> None:
    """``u v w`` per stored slot, each undirected edge once (graph.py:264-272)."""
    off = g.offsets
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(off))
    adj = g.adj.astype(np.int64)
    w = g.weights.astype(np.int64)
    keep = np.ones(g.m, bool) if g.directed else adj >= src
    with open(path, "w", encoding="utf-8") as f:
        for a, b, c in zip(src[keep].tolist(), adj[keep].tolist(), w[keep].tolist()):
            f.write(f"{a} {b} {c}\n")
