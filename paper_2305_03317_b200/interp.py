"""``run``: the drop-in for trident.interp.run on the corpus programs.

Signature, argument checking, iteration cap, result layout and exceptions
follow trident/interp.py:
  run(tp, g, args, function=None, max_iters=None, on_fixedpoint_iteration=None)
    -> RunResult(env=PropertyEnv(node_props, edge_props, scalars),
                 fixedpoint_iterations, wall_seconds, return_value)
The program is identified (corpus.identify), the arguments are checked and
coerced exactly like check_args (interp.py:91-129), and the work runs on the
GPU through libstarplat_b200.so.  Property arrays come back as NumPy arrays
(same values as the reference's lists), or as the reference's Python lists
with ``as_lists=True``.

Differences, all documented in DESIGN.md:
  * SSSP's fixedPoint iteration count comes from the parallel frontier order,
    not the interpreter's in-place order, and may differ (dist never does).
  * PR/BC fold hub rows (in-degree > 4096 / 8192) with a fixed-shape tree
    unless ``deterministic=True`` (then every fold is the reference's left
    fold, bit for bit).
  * The iteration hook receives a small context object, not the
    interpreter's Executor.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib, corpus
from .errors import BackendError, errors_for
from .graph import CsrGraph, device_graph


def default_iteration_cap(n: int) -> int:
    """interp.py:36-37."""
    return 2 * n + 16


@dataclass
class PropertyEnv:
    node_props: dict = field(default_factory=dict)
    edge_props: dict = field(default_factory=dict)
    scalars: dict = field(default_factory=dict)


@dataclass
class RunResult:
    env: PropertyEnv
    fixedpoint_iterations: dict = field(default_factory=dict)
    wall_seconds: float = 0.0
    return_value: object = None
    stats: dict | None = None  # backend counters (device ms, edges visited, ...)


@dataclass
class HookContext:
    """Third argument of on_fixedpoint_iteration (the reference passes its
    Executor, interp.py:411-412)."""

    program: str
    graph: CsrGraph
    flag: str
    iterations: int


def _coerce(kind: str, value):
    """interp.py:75-82 for the formal kinds the corpus uses."""
    if kind in ("double", "float"):
        return float(value)
    if kind == "bool":
        return bool(value)
    return int(value)


def check_args(prog: corpus.Program, g: CsrGraph, args: dict, E) -> dict:
    """interp.py:91-129 restricted to the corpus formals."""
    bound = {}
    for name, kind in prog.params:
        if kind == "Graph":
            continue
        if name not in args:
            raise E.ExecError(f"missing argument '{name}'")
        v = args[name]
        if kind == "node":
            vid = int(v)
            if not 0 <= vid < g.n:
                raise E.ExecError(f"node argument '{name}'={vid} out of range")
            bound[name] = vid
        elif kind == "SetN":
            ids = [int(x) for x in v]
            for vid in ids:
                if not 0 <= vid < g.n:
                    raise E.ExecError(f"set argument '{name}' id {vid} out of range")
            bound[name] = ids
        else:
            bound[name] = _coerce(kind, v)
    return bound


def _raise_for(rc: int, E, flag: str | None, cap: int, hook_exc):
    if rc == _lib.SP_OK:
        return
    if hook_exc is not None:
        raise hook_exc
    msg = _lib.last_error()
    if rc == _lib.SP_ERR_NONCONV:
        raise E.NonConvergenceError(flag, cap)
    if rc in (_lib.SP_ERR_ARG, _lib.SP_ERR_OVERFLOW, _lib.SP_ERR_UNSUPPORTED):
        raise E.ExecError(msg)
    if rc == _lib.SP_ERR_OOM:
        raise MemoryError(f"device out of memory: {msg}")
    raise BackendError(f"native call failed ({rc}): {msg}")


class _Hook:
    """Adapts on_fixedpoint_iteration to the C callback."""

    def __init__(self, fn, prog, g):
        self.fn, self.prog, self.g = fn, prog, g
        self.exc = None
        self.cb = _lib.ITER_CB(self._call) if fn is not None else _lib.ITER_CB()

    def _call(self, iters, _user):
        try:
            self.fn(self.prog.flag, int(iters),
                    HookContext(self.prog.key, self.g, self.prog.flag, int(iters)))
            return 0
        except BaseException as e:  # surfaced after the native call returns
            self.exc = e
            return 1


def _i64(x: int) -> int:
    return max(-(2 ** 63), min(2 ** 63 - 1, int(x)))


_PINNED_MIN = 1 << 16  # results at least this long land in pinned host memory


def _torch():
    try:
        import torch  # plumbing only: pinned host / device buffers
        return torch
    except ImportError:  # pragma: no cover
        return None


def _host_array(n: int, dtype) -> np.ndarray:
    """NumPy result array; large ones are backed by torch's cached pinned
    host memory so the device-to-host copy runs at full PCIe speed (the
    array keeps its pinned storage alive)."""
    torch = _torch()
    if n >= _PINNED_MIN and torch is not None and torch.cuda.is_available():
        td = {np.float64: torch.float64, np.int32: torch.int32}[dtype]
        return torch.empty(n, dtype=td, pin_memory=True).numpy()
    return np.empty(n, dtype=dtype)


def _host_copy(a: np.ndarray) -> np.ndarray:
    """A copy of a result array (multi-threaded for large ones)."""
    torch = _torch()
    if len(a) >= _PINNED_MIN and torch is not None:
        out = _host_array(len(a), a.dtype.type)
        torch.from_numpy(out).copy_(torch.from_numpy(a))
        return out
    return a.copy()


def _out(n: int, dtype, dev: int | None):
    """Result buffer: a NumPy array (host) or a torch CUDA tensor (device)."""
    if dev is None:
        return _host_array(n, dtype), _lib.SP_MEM_HOST
    import torch  # plumbing only: device memory for results that stay in HBM
    t = torch.empty(max(1, n), dtype={np.float64: torch.float64,
                                      np.int32: torch.int32}[dtype],
                    device=torch.device("cuda", dev))[:n]
    return t, _lib.SP_MEM_DEVICE


def _ptr(buf):
    return C.c_void_p(buf.data_ptr()) if hasattr(buf, "data_ptr") else \
        buf.ctypes.data_as(C.c_void_p)


def run(tp, g, args: dict, function: str | None = None,
        max_iters: int | None = None, on_fixedpoint_iteration=None, *,
        deterministic: bool = False, device_outputs: bool = False,
        as_lists: bool = False) -> RunResult:
    """Run a corpus program on the GPU.  ``tp`` is a reference TypedProgram
    (recognised structurally), a ``corpus.Program`` or a corpus key.

    ``device_outputs=True`` leaves the property arrays in HBM (torch CUDA
    tensors on the graph's device) instead of copying them to NumPy.
    ``as_lists=True`` returns every node property as a Python list of
    Python ints / floats / bools, exactly the reference's ``final_env``
    layout (interp.py:259-266), for callers that compare with ``==``,
    mutate or JSON-serialise the lists."""
    if as_lists and device_outputs:
        raise ValueError("as_lists and device_outputs are mutually exclusive")
    E = errors_for(tp)
    prog = corpus.identify(tp, function)
    dg = device_graph(g)
    bound = check_args(prog, dg, args, E)
    cap = _i64(max_iters if max_iters is not None else default_iteration_cap(dg.n))
    L = _lib.lib()
    st = _lib.Stats()
    hook = _Hook(on_fixedpoint_iteration, prog, dg)
    flags = _lib.SP_FLAG_DETERMINISTIC if deterministic else 0
    n = dg.n
    odev = dg.device if device_outputs else None
    t0 = time.perf_counter()
    env = PropertyEnv()
    fpi: dict = {}
    if prog.key in ("sssp", "sssp_pull"):
        dist, mem = _out(n, np.int32, odev)
        iters = C.c_int64()
        fn = L.sp_sssp_pull if prog.key == "sssp_pull" else L.sp_sssp
        rc = fn(dg.handle, bound["src"], cap, _ptr(dist), mem, C.byref(iters),
                hook.cb, None, C.byref(st))
        _raise_for(rc, E, prog.flag, cap, hook.exc)
        env.node_props = {"dist": dist, "modified": np.zeros(n, dtype=bool),
                          "modified_nxt": np.zeros(n, dtype=bool)}
        if odev is not None:
            env.node_props["modified"] = env.node_props["modified_nxt"] = None
        env.scalars = {"finished": True}
        fpi = {"finished": int(iters.value)}
    elif prog.key == "pr":
        rank, mem = _out(n, np.float64, odev)
        it, its = C.c_int64(), C.c_int64()
        diff = C.c_double()
        rc = L.sp_pagerank(dg.handle, bound["damping"], bound["epsilon"],
                           _i64(bound["maxIter"]), cap, flags, _ptr(rank), mem,
                           C.byref(it), C.byref(diff), C.byref(its), hook.cb, None,
                           C.byref(st))
        _raise_for(rc, E, prog.flag, cap, hook.exc)
        # rank_nxt == rank at exit (pr.sp:25-27 copies it back every iteration)
        env.node_props = {"rank": rank,
                          "rank_nxt": rank if odev is not None else _host_copy(rank)}
        env.scalars = {"iter": int(it.value), "diff": float(diff.value),
                       "converged": True}
        fpi = {"converged": int(its.value)}
    elif prog.key == "bc":
        srcs = np.asarray(bound["sourceSet"], dtype=np.int32)
        bc, mem = _out(n, np.float64, odev)
        sigma, _ = _out(n, np.float64, odev)
        delta, _ = _out(n, np.float64, odev)
        rc = L.sp_bc(dg.handle, srcs.ctypes.data_as(C.c_void_p), len(srcs), flags,
                     _ptr(bc), _ptr(sigma), _ptr(delta), mem, C.byref(st))
        _raise_for(rc, E, None, cap, None)
        env.node_props = {"bc": bc}
        if len(srcs):  # sigma/delta are attached inside the source loop (bc.sp:5-7)
            env.node_props.update(sigma=sigma, delta=delta)
    elif prog.key == "reduction":
        # reduction.sp:2-10: prop = 1 everywhere; accum += nbr.prop over every
        # (v, nbr) slot (the inner `count` is local, not in the result)
        tot = C.c_int64()
        rc = L.sp_neighbor_sum(dg.handle, None, _lib.SP_MEM_HOST, 0, None, C.byref(tot),
                               C.byref(st))
        _raise_for(rc, E, None, cap, None)
        env.node_props = {"prop": np.ones(n, dtype=np.int64)}
        env.scalars = {"accum": int(tot.value)}
    elif prog.key == "forall":  # the generic neighbour-reduction shape (forall.py)
        from . import forall
        props, scalars, fst = forall.execute(prog, dg)
        env.node_props = props
        env.scalars = scalars
        st.kernel_launches = fst["kernel_launches"]
        st.device_ms = fst["device_ms"]
        st.edges_visited = fst["edges_visited"]
    elif prog.key == "tc":
        cnt = C.c_uint64()
        rc = L.sp_tc(dg.handle, 0, n, C.byref(cnt), C.byref(st))
        _raise_for(rc, E, None, cap, None)
        env.scalars = {"triangle_count": int(cnt.value)}
    else:  # pragma: no cover
        raise E.ExecError(f"unhandled program {prog.key}")
    if as_lists:
        env.node_props = {k: np.asarray(a).tolist() for k, a in env.node_props.items()}
    wall = time.perf_counter() - t0
    return RunResult(env=env, fixedpoint_iterations=fpi, wall_seconds=wall,
                     return_value=None, stats=st.as_dict())
