"""B200-native (sm_100a) backend for the StarPlat corpus graph programs.

Drop-in for the hot path of the reference package ``trident``:
graph load -> device CSR (``graph``) -> SSSP / PageRank / BC / TC
(``interp.run``), executed by hand-written CUDA kernels in
libstarplat_b200.so (C ABI: include/starplat_b200.h).  No CPU fallback.
"""

from . import corpus, errors, gen  # noqa: F401
from .graph import (CsrGraph, Partition, assign_random_weights,  # noqa: F401
                    block_partition, device_graph, from_arrays, from_csr,
                    from_edges, generate, load_edge_list, max_wt, min_wt,
                    owner_of, write_edge_list)
from .interp import PropertyEnv, RunResult, default_iteration_cap, run  # noqa: F401

__all__ = ["CsrGraph", "Partition", "assign_random_weights", "block_partition",
           "device_graph", "from_arrays", "from_csr", "from_edges", "generate",
           "load_edge_list", "max_wt", "min_wt", "owner_of", "write_edge_list",
           "PropertyEnv", "RunResult", "default_iteration_cap", "run",
           "corpus", "errors", "gen"]
