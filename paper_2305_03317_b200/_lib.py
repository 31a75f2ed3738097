"""ctypes binding of libstarplat_b200.so (include/starplat_b200.h).

The library is built in-tree (``python -c "import __graft_entry__ as g;
g.build()"`` or ``make -C paper_2305_03317_b200/csrc``).  There is no CPU
fallback: if the library or a CUDA device is missing, every entry point
raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# SP_LIB: an alternative build of the same library (diagnostic variants)
LIB_PATH = os.environ.get("SP_LIB") or os.path.join(HERE, "libstarplat_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "starplat_b200.h")

ABI_VERSION = 8  # must equal SP_ABI_VERSION in include/starplat_b200.h

SP_OK = 0
SP_ERR_ARG = -1
SP_ERR_NONCONV = -2
SP_ERR_CUDA = -3
SP_ERR_OOM = -4
SP_ERR_OVERFLOW = -5
SP_ERR_UNSUPPORTED = -6
SP_ERR_ABORTED = -7

SP_MEM_HOST = 0
SP_MEM_DEVICE = 1
SP_FLAG_DETERMINISTIC = 1

SP_ARR_OFFSETS, SP_ARR_ADJ, SP_ARR_WEIGHTS, SP_ARR_REV_OFFSETS, \
    SP_ARR_REV_ADJ, SP_ARR_REV_EID, SP_ARR_WEFF = range(7)
SP_GEN_RMAT, SP_GEN_UNIFORM, SP_GEN_GRID = range(3)
SP_REDUCE_SUM_I64, SP_REDUCE_MIN_F64, SP_REDUCE_MAX_F64 = range(3)
PREP_KINDS = ("tc_upper", "weff", "rweff", "pr_hot", "pr_rel", "ell", "ell2")  # SP_PREP_* order


class Stats(C.Structure):
    _fields_ = [("iterations", C.c_int64),
                ("edges_visited", C.c_int64),
                ("vertices_visited", C.c_int64),
                ("kernel_launches", C.c_int64),
                ("device_ms", C.c_double),
                ("main_kernel_ms", C.c_double),
                ("main_kernel_launches", C.c_int64),
                ("model_bytes", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


ITER_CB = C.CFUNCTYPE(C.c_int, C.c_int64, C.c_void_p)

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_int = C.c_int
_u = C.c_uint
_d = C.c_double

# name -> (restype, argtypes); exactly the symbols include/starplat_b200.h declares
SIGNATURES = {
    "sp_abi_version": (_int, []),
    "sp_last_error": (C.c_char_p, []),
    "sp_device_count": (_int, []),
    "sp_graph_from_edges": (_int, [_p, _p, _p, _i64, _i64, _int, _int, _int, _p]),
    "sp_graph_from_csr": (_int, [_p, _p, _p, _i64, _i64, _int, _int, _int, _p]),
    "sp_graph_generate": (_int, [_int, _i64, _i64, _i64, _int, _int, _p]),
    "sp_parse_edge_text": (_int, [C.c_char_p, _i64, _i64, _int, _p, _p]),
    "sp_free_host": (None, [_p]),
    "sp_graph_info": (_int, [_p, _p, _p, _p]),
    "sp_graph_download": (_int, [_p, _int, _p]),
    "sp_graph_weight_range": (_int, [_p, _p, _p]),
    "sp_graph_prep_ms": (_int, [_p, _int, _p]),
    "sp_graph_destroy": (None, [_p]),
    "sp_sssp": (_int, [_p, _i32, _i64, _p, _int, _p, ITER_CB, _p, _p]),
    "sp_sssp_pull": (_int, [_p, _i32, _i64, _p, _int, _p, ITER_CB, _p, _p]),
    "sp_sssp_shard_create": (_int, [_p, _i64, _i64, _i32, _int, _p, _p]),
    "sp_sssp_shard_relax": (_int, [_p, _i64, _i64, _p, _p, _p]),
    "sp_sssp_shard_apply": (_int, [_p, _p, _i64, _p, _p]),
    "sp_sssp_shard_destroy": (None, [_p]),
    "sp_sssp_shard_peers": (_int, [_p, _i64, _p, _p, _p, _p, _p]),
    "sp_sssp_shard_collect": (_int, [_p, _p]),
    "sp_pagerank": (_int, [_p, _d, _d, _i64, _i64, _u, _p, _int, _p, _p, _p,
                           ITER_CB, _p, _p]),
    "sp_pagerank_block_init": (_int, [_p, _i64, _i64, _p, _p]),
    "sp_pagerank_shard_create": (_int, [_p, _i64, _i64, _d, _u, _p, _p]),
    "sp_pagerank_shard_step": (_int, [_p, _p, _p, _p, _p]),
    "sp_pagerank_shard_destroy": (None, [_p]),
    "sp_pagerank_shard_peers": (_int, [_p, _int, _int, _p]),
    "sp_pagerank_shard_step_peers": (_int, [_p, _p, _p, _p, _p, _int]),
    "sp_peer_alloc": (_int, [_int, _i64, _p, _p]),
    "sp_peer_open": (_int, [_int, _p, _p]),
    "sp_peer_free": (None, [_p, _int]),
    "sp_bc": (_int, [_p, _p, _i64, _u, _p, _p, _p, _int, _p]),
    "sp_tc": (_int, [_p, _i64, _i64, _p, _p]),
    "sp_neighbor_sum": (_int, [_p, _p, _int, _int, _p, _p, _p]),
    "sp_neighbor_reduce": (_int, [_p, _int, _int, _i64, _d, _p, _int, _p, _p, _p]),
}

_lib = None
_lock = threading.Lock()


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load the native library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissing(
                    f"{LIB_PATH} not built; run `make -C {HERE}/csrc` "
                    "(no CPU fallback exists)")
            L = C.CDLL(LIB_PATH)
            L.sp_abi_version.restype = C.c_int
            if L.sp_abi_version() != ABI_VERSION:
                raise LibraryMissing(
                    f"{LIB_PATH} has ABI {L.sp_abi_version()}, expected {ABI_VERSION}; rebuild it")
            for name, (res, args) in SIGNATURES.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def last_error() -> str:
    msg = lib().sp_last_error()
    return msg.decode(errors="replace") if msg else ""


def device_count() -> int:
    return int(lib().sp_device_count())


def require_device(device: int = 0):
    n = device_count()
    if n <= device:
        raise RuntimeError(
            f"no CUDA device {device} visible (found {n}); the B200 backend has "
            "no CPU fallback")
