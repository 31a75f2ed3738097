"""ctypes wrapper of the CPU oracle (oracle/cpu_ref.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg, always as the checker or
the timed CPU baseline, never by the product package.

Every function restates trident.interp.run semantics for one corpus program
(see the file:line citations in cpu_ref.c) and is pinned bit-for-bit to the
Python reference by tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcpu_ref.so")

_lib = None

_i64 = C.c_int64
_i32 = C.c_int32
_p = C.c_void_p


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.cr_count_slots.restype = _i64
        L.cr_count_slots.argtypes = [_i64, _p, _p, C.c_int]
        L.cr_build_csr.restype = C.c_int
        L.cr_build_csr.argtypes = [_i64, _i64, _p, _p, _p, C.c_int,
                                   _p, _p, _p, _p, _p, _p]
        L.cr_weff.restype = None
        L.cr_weff.argtypes = [_i64, _p, _p, _p, _p]
        L.cr_sssp.restype = C.c_int
        L.cr_sssp.argtypes = [_i64, _p, _p, _p, _i32, _i64, _p, _p]
        L.cr_sssp_dijkstra.argtypes = [_i64, _p, _p, _p, _i32, _p]
        L.cr_pagerank.restype = C.c_int
        L.cr_pagerank.argtypes = [_i64, _p, _p, _p, C.c_double, C.c_double,
                                  _i64, _i64, _p, _p, _p, _p, C.c_int]
        L.cr_bc.restype = None
        L.cr_bc.argtypes = [_i64, _p, _p, _p, _p, _p, _i64, _p, _p, _p, C.c_int]
        L.cr_tc.restype = C.c_uint64
        L.cr_tc.argtypes = [_i64, _p, _p, C.c_int]
        L.cr_num_threads.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class Csr:
    n: int
    m: int
    directed: bool
    off: np.ndarray
    adj: np.ndarray
    w: np.ndarray
    roff: np.ndarray
    radj: np.ndarray
    reid: np.ndarray
    weff: np.ndarray


def build_csr(u, v, w, directed: bool, n: int | None = None) -> Csr:
    """trident.graph.from_edges restated (graph.py:101-116)."""
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.int32)
    ne = len(u)
    maxid = int(max(u.max(), v.max())) if ne else -1
    nn = max(n if n is not None else 0, maxid + 1)
    L = lib()
    m = int(L.cr_count_slots(ne, _ptr(u), _ptr(v), int(directed)))
    off = np.zeros(nn + 1, np.int64)
    adj = np.zeros(m, np.int32)
    wt = np.zeros(m, np.int32)
    roff = np.zeros(nn + 1, np.int64)
    radj = np.zeros(m, np.int32)
    reid = np.zeros(m, np.int64)
    rc = L.cr_build_csr(nn, ne, _ptr(u), _ptr(v), _ptr(w), int(directed),
                        _ptr(off), _ptr(adj), _ptr(wt), _ptr(roff),
                        _ptr(radj), _ptr(reid))
    if rc != 0:
        raise MemoryError("cr_build_csr failed")
    weff = np.zeros(m, np.int32)
    L.cr_weff(nn, _ptr(off), _ptr(adj), _ptr(wt), _ptr(weff))
    return Csr(nn, m, directed, off, adj, wt, roff, radj, reid, weff)


def sssp(g: Csr, src: int, cap: int | None = None):
    """Returns (dist int32[n], fixedpoint iterations, rc)."""
    cap = 2 * g.n + 16 if cap is None else cap
    dist = np.zeros(g.n, np.int32)
    it = np.zeros(1, np.int64)
    rc = lib().cr_sssp(g.n, _ptr(g.off), _ptr(g.adj), _ptr(g.weff), src, cap,
                       _ptr(dist), _ptr(it))
    return dist, int(it[0]), rc


def sssp_dijkstra(g: Csr, src: int):
    """Exact distances by Dijkstra (trident/oracles.py:23-40) over w_eff;
    equal to sssp()'s for non-negative weights.  Returns (dist, rc)."""
    dist = np.zeros(g.n, np.int32)
    rc = lib().cr_sssp_dijkstra(g.n, _ptr(g.off), _ptr(g.adj), _ptr(g.weff), src, _ptr(dist))
    return dist, rc


def pagerank(g: Csr, damping=0.85, eps=1e-6, max_iter=100,
             cap: int | None = None, nthreads: int = 1):
    """Returns (rank f64[n], iter, diff, fixedpoint iterations, rc)."""
    cap = 2 * g.n + 16 if cap is None else cap
    rank = np.zeros(g.n, np.float64)
    it = np.zeros(1, np.int64)
    its = np.zeros(1, np.int64)
    diff = np.zeros(1, np.float64)
    rc = lib().cr_pagerank(g.n, _ptr(g.off), _ptr(g.roff), _ptr(g.radj),
                           float(damping), float(eps), int(max_iter), cap,
                           _ptr(rank), _ptr(it), _ptr(diff), _ptr(its),
                           nthreads)
    return rank, int(it[0]), float(diff[0]), int(its[0]), rc


def bc(g: Csr, sources, nthreads: int = 1):
    """Returns (bc, sigma_last, delta_last) f64[n]."""
    s = np.ascontiguousarray(np.asarray(sources, dtype=np.int32))
    b = np.zeros(g.n, np.float64)
    sg = np.zeros(g.n, np.float64)
    dl = np.zeros(g.n, np.float64)
    lib().cr_bc(g.n, _ptr(g.off), _ptr(g.adj), _ptr(g.roff), _ptr(g.radj),
                _ptr(s), len(s), _ptr(b), _ptr(sg), _ptr(dl), nthreads)
    return b, sg, dl


def tc(g: Csr, nthreads: int = 1) -> int:
    return int(lib().cr_tc(g.n, _ptr(g.off), _ptr(g.adj), nthreads))


def num_threads() -> int:
    return int(lib().cr_num_threads())
