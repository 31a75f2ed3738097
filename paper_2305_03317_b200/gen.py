"""Seeded synthetic graph generators (host replica of the device generators).

The BASELINE configs name RMAT (a/b/c/d = .57/.19/.19/.05),
uniform-random and 2-D grid graphs with weights U[1,100].
Every random draw is a pure function of (seed, counter) through splitmix64,
so the same edge list can be produced here in NumPy (small scales, fed to
the CPU oracle and the Python reference) and on the GPU by
``csrc/sp_gen.cu`` (full scales), bit for bit.  The fixture generator the
reference ships (pkg/tools/gen_fixtures.py:37-78) is the pattern: seeded,
byte-reproducible, dedupe + drop self-loops.

Pipeline of every generator: candidate pairs -> (canonicalise for undirected)
-> drop self-loops -> sort + unique on the 64-bit key (u << 32 | v) -> weight
from a hash of the (canonical) pair.  Output is three int32 arrays (u, v, w)
in ascending key order, the edge-list input of ``graph.from_arrays``.
"""

from __future__ import annotations

import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# 16-bit RMAT thresholds: round(p * 65536), cumulative.
RMAT_A, RMAT_B, RMAT_C = 0.57, 0.19, 0.19


def rmat_thresholds(a=RMAT_A, b=RMAT_B, c=RMAT_C):
    ta = int(round(a * 65536))
    tb = ta + int(round(b * 65536))
    tc = tb + int(round(c * 65536))
    return ta, tb, tc


def splitmix64(x):
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _seed_key(seed: int) -> np.uint64:
    return splitmix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF))[()]


def pair_weights(u: np.ndarray, v: np.ndarray, seed: int,
                 lo: int = 1, hi: int = 100) -> np.ndarray:
    """w = lo + hash(seed, u<<32|v) % (hi-lo+1); u,v are the canonical pair."""
    span = np.uint64(hi - lo + 1)
    key = (u.astype(np.uint64) << np.uint64(32)) | v.astype(np.uint64)
    h = splitmix64(key ^ _seed_key(seed ^ 0x5EED))
    return (np.int64(lo) + (h % span).astype(np.int64)).astype(np.int32)


def _dedupe(u: np.ndarray, v: np.ndarray, undirected: bool):
    u = u.astype(np.uint64)
    v = v.astype(np.uint64)
    if undirected:
        u, v = np.minimum(u, v), np.maximum(u, v)
    keep = u != v
    key = (u[keep] << np.uint64(32)) | v[keep]
    key = np.unique(key)
    return ((key >> np.uint64(32)).astype(np.int32),
            (key & np.uint64(0xFFFFFFFF)).astype(np.int32))


def rmat_pairs(scale: int, edge_factor: int, seed: int):
    """Raw RMAT candidate pairs (before dedupe), edge i uses hash words
    splitmix64(seedkey ^ (i << 4 | g)) for level groups g of 4 levels."""
    ne = edge_factor << scale
    ta, tb, tc = rmat_thresholds()
    i = np.arange(ne, dtype=np.uint64)
    sk = _seed_key(seed)
    u = np.zeros(ne, dtype=np.uint64)
    v = np.zeros(ne, dtype=np.uint64)
    ngroups = (scale + 3) // 4
    for g in range(ngroups):
        h = splitmix64(sk ^ ((i << np.uint64(4)) | np.uint64(g)))
        for j in range(4):
            lvl = g * 4 + j
            if lvl >= scale:
                break
            r = (h >> np.uint64(16 * j)) & np.uint64(0xFFFF)
            bu = (r >= np.uint64(tb)).astype(np.uint64)
            bv = (((r >= np.uint64(ta)) & (r < np.uint64(tb))) |
                  (r >= np.uint64(tc))).astype(np.uint64)
            sh = np.uint64(scale - 1 - lvl)
            u |= bu << sh
            v |= bv << sh
    return u, v


def rmat(scale: int, edge_factor: int = 16, seed: int = 1,
         undirected: bool = False, weight_seed: int | None = None):
    """RMAT edge list: (u, v, w) int32, deduplicated, no self-loops,
    no relabelling (vertex 0 is the hub)."""
    u, v = rmat_pairs(scale, edge_factor, seed)
    u, v = _dedupe(u, v, undirected)
    w = pair_weights(u, v, seed if weight_seed is None else weight_seed)
    return u, v, w, 1 << scale


def uniform(n: int, nedges: int, seed: int = 1, undirected: bool = True,
            weight_seed: int | None = None):
    """Uniform-random pairs via multiply-shift range reduction of one hash."""
    i = np.arange(nedges, dtype=np.uint64)
    h = splitmix64(_seed_key(seed) ^ i)
    nn = np.uint64(n)
    lo32 = np.uint64(0xFFFFFFFF)
    with np.errstate(over="ignore"):
        u = ((h >> np.uint64(32)) * nn) >> np.uint64(32)
        v = ((h & lo32) * nn) >> np.uint64(32)
    u, v = _dedupe(u, v, undirected)
    w = pair_weights(u, v, seed if weight_seed is None else weight_seed)
    return u, v, w, n


def grid(rows: int, cols: int, seed: int = 1):
    """4-neighbour grid, right and down edges per cell in row-major order
    (pkg/tools/gen_fixtures.py:68-78 order), undirected, hashed weights."""
    r, c = np.meshgrid(np.arange(rows, dtype=np.int64),
                       np.arange(cols, dtype=np.int64), indexing="ij")
    vid = (r * cols + c).ravel()
    right = (c + 1 < cols).ravel()
    down = (r + 1 < rows).ravel()
    # interleave (right, down) per cell, keeping only existing edges
    uu = np.stack([vid, vid], axis=1).ravel()
    vv = np.stack([vid + 1, vid + cols], axis=1).ravel()
    ok = np.stack([right, down], axis=1).ravel()
    u = uu[ok].astype(np.int32)
    v = vv[ok].astype(np.int32)
    w = pair_weights(u, v, seed)
    return u, v, w, rows * cols
