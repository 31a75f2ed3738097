/*
 * starplat_b200.h -- C ABI of the B200 (sm_100a) graph-kernel backend.
 *
 * This is the drop-in boundary behind the reference's Python entry points.
 * The reference (trident, pure Python) has no FFI of its own; each entry
 * point below replaces one Python function of the hot path, cited as
 * trident/<file>:<line> (relative to /root/reference/pkg/src).  The Python
 * host layer (paper_2305_03317_b200/) binds these with ctypes and keeps the
 * reference's signatures, argument checks and exception types.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Vertex ids int32, edge ids / offsets
 *     int64, weights int32, properties int32 / double.
 *   - `mem` says where a caller buffer lives: SP_MEM_HOST (pageable or
 *     pinned host memory; copied inside the call) or SP_MEM_DEVICE (a device
 *     pointer on the graph's device, e.g. a torch tensor's data_ptr()).
 *   - Return SP_OK (0) or a negative SP_ERR_*; sp_last_error() gives a
 *     thread-local message.  No call falls back to the CPU.
 *   - A graph handle is immutable after creation and safe for concurrent
 *     readers; every algorithm call uses its own stream and
 *     scratch (stream-ordered allocations).
 */
#ifndef STARPLAT_B200_H
#define STARPLAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_ABI_VERSION 8

enum sp_status {
    SP_OK = 0,
    SP_ERR_ARG = -1,          /* bad argument -> ExecError (interp.py:98-128) */
    SP_ERR_NONCONV = -2,      /* fixedPoint cap -> NonConvergenceError (errors.py:85-92) */
    SP_ERR_CUDA = -3,         /* CUDA runtime failure -> RuntimeError */
    SP_ERR_OOM = -4,          /* device allocation failed */
    SP_ERR_OVERFLOW = -5,     /* an int32 distance would leave int32 range */
    SP_ERR_UNSUPPORTED = -6,  /* input outside the backend's domain (e.g. n >= 2^31) */
    SP_ERR_ABORTED = -7       /* iteration callback asked to stop */
};

enum sp_mem { SP_MEM_HOST = 0, SP_MEM_DEVICE = 1 };

/* Algorithm flags. */
#define SP_FLAG_DETERMINISTIC 1u /* bit-exact left folds everywhere (PR, BC) */

/* Arrays a graph handle can hand back (sp_graph_download). */
enum sp_array {
    SP_ARR_OFFSETS = 0,     /* int64[n+1]  CsrGraph.offsets     graph.py:30 */
    SP_ARR_ADJ = 1,         /* int32[m]    CsrGraph.adj         graph.py:31 */
    SP_ARR_WEIGHTS = 2,     /* int32[m]    CsrGraph.weights     graph.py:32 */
    SP_ARR_REV_OFFSETS = 3, /* int64[n+1]  CsrGraph.rev_offsets graph.py:33 */
    SP_ARR_REV_ADJ = 4,     /* int32[m]    CsrGraph.rev_adj     graph.py:34 */
    SP_ARR_REV_EID = 5,     /* int64[m]    CsrGraph.rev_eid     graph.py:35 */
    SP_ARR_WEFF = 6         /* int32[m]    weight of the first slot u->v (get_edge) */
};

enum sp_gen_kind { SP_GEN_RMAT = 0, SP_GEN_UNIFORM = 1, SP_GEN_GRID = 2 };

typedef struct sp_graph sp_graph;

/* Optional per-call counters (NULL to skip). */
typedef struct sp_stats {
    int64_t iterations;        /* fixedPoint iterations / BFS levels summed   */
    int64_t edges_visited;     /* SSSP: relaxations R; PR: iters*m; BC: sum m_s; TC: pairs */
    int64_t vertices_visited;  /* SSSP: frontier sum F; PR: iters*n; BC: sum n_s */
    int64_t kernel_launches;   /* kernels this call launched                  */
    double device_ms;          /* device time of the call (CUDA events)       */
    double main_kernel_ms;     /* summed device time of the dominant kernel   */
    int64_t main_kernel_launches;
    int64_t model_bytes;       /* algorithmic bytes of the call per SURVEY 8d (0 = n/a) */
} sp_stats;

/* fixedPoint iteration callback, mirrors interp.py:138,411-412
 * (on_fixedpoint_iteration(flag, iters, executor)); return nonzero to abort. */
typedef int (*sp_iter_cb)(int64_t iters, void *user);

/* ---- runtime ---------------------------------------------------------- */
int sp_abi_version(void);
const char *sp_last_error(void);
int sp_device_count(void);

/* ---- graph core: replaces trident/graph.py ----------------------------- */

/* from_edges (graph.py:101-116): one slot per edge plus the mirror for
 * undirected non-loop edges, n = max(n, 1 + max id), forward CSR stably
 * sorted by (src, dst) (graph.py:70-81), reverse CSR by (dst, src, eid)
 * (graph.py:84-96).  Built on the device; uploaded once, never copied back. */
int sp_graph_from_edges(const int32_t *u, const int32_t *v, const int32_t *w,
                        int64_t nedges, int64_t n, int directed, int mem,
                        int device, sp_graph **out);

/* CsrGraph(...) (graph.py:18-36) from an existing forward CSR whose rows are
 * already in reference order; the reverse CSR is rebuilt on the device.
 * weights == NULL: unweighted input, every slot gets weight 1 (the
 * reference's default_weight) on the device, nothing is copied for it. */
int sp_graph_from_csr(const int64_t *offsets, const int32_t *adj,
                      const int32_t *weights, int64_t n, int64_t m,
                      int directed, int mem, int device, sp_graph **out);

/* Seeded synthetic graphs generated on the device, bit-identical to
 * paper_2305_03317_b200/gen.py (pattern: pkg/tools/gen_fixtures.py:37-78).
 *   SP_GEN_RMAT:    p0 = scale, p1 = edge factor
 *   SP_GEN_UNIFORM: p0 = n,     p1 = candidate edges
 *   SP_GEN_GRID:    p0 = rows,  p1 = cols (always undirected)            */
int sp_graph_generate(int kind, int64_t p0, int64_t p1, int64_t seed,
                      int undirected, int device, sp_graph **out);

/* Text parsing of load_edge_list (graph.py:119-151), host only: `u v [w]`
 * lines (\n, \r\n or \r terminated), '#' and blank lines skipped,
 * duplicates kept, parsed on all host threads (nthreads <= 0: all).  On
 * success *uvw is a malloc'd block [u | v | w] (stride info[7], info[6]
 * edges) for sp_graph_from_edges; free it with sp_free_host.  info[8]:
 * [0] error kind (1 field count, 2 non-integer field, 3 negative vertex id;
 * returned with SP_ERR_ARG for the first failing line = the line the
 * reference raises FormatError on), [1] that line number, [2..3] vertex id
 * min/max, [4..5] weight min/max.  SP_ERR_UNSUPPORTED: non-ASCII text or
 * values outside int32 (the host layer then parses with the reference's own
 * Python semantics). */
int sp_parse_edge_text(const char *buf, int64_t len, int64_t default_weight,
                       int nthreads, int32_t **uvw, int64_t *info);
void sp_free_host(void *p);

int sp_graph_info(const sp_graph *g, int64_t *n, int64_t *m, int *directed);
int sp_graph_download(const sp_graph *g, int which, void *host_dst);
/* min_wt / max_wt (graph.py:252-261); SP_ERR_ARG when m == 0. */
int sp_graph_weight_range(const sp_graph *g, int32_t *wmin, int32_t *wmax);
/* One-time per-graph preprocessing that the first call needing it builds
 * and caches on the handle (no reference counterpart: the interpreter keeps
 * no derived structures).  *ms = device time of that build (CUDA events on
 * the building call's stream), -1 when it was not built (or was built
 * during the upload, untimed).  Waits for the build to finish. */
#define SP_PREP_TC_UPPER 0 /* degree-ordered upper CSR (sp_tc)               */
#define SP_PREP_WEFF     1 /* first-slot weights w_eff (sp_sssp)            */
#define SP_PREP_RWEFF    2 /* reverse-slot w_eff (pull sweeps)              */
#define SP_PREP_PR_HOT   3 /* PR hot-source encoding of radj                */
#define SP_PREP_PR_REL   4 /* PR relabelled (out-degree rank) layout        */
#define SP_PREP_ELL      5 /* ELL rows of bounded-degree graphs (async SSSP) */
#define SP_PREP_ELL2     6 /* 2-hop shortcut rows (async SSSP, out-degree <= 4) */
int sp_graph_prep_ms(const sp_graph *g, int kind, double *ms);
void sp_graph_destroy(sp_graph *g);

/* ---- executor: replaces trident/interp.py:579-589 on the corpus -------- */

/* corpus/programs/sssp.sp (and sssp_pull.sp: same dist).  dist[n] int32
 * (INT_MAX = unreachable, syntax.py:114).  cap = fixedPoint cap
 * (interp.py:36-37,143,415-416).  iters = fixedPoint iterations. */
int sp_sssp(sp_graph *g, int32_t src, int64_t cap, int32_t *dist, int mem,
            int64_t *iters, sp_iter_cb cb, void *user, sp_stats *st);

/* corpus/programs/sssp_pull.sp (sssp_pull.sp:9-14): the pull form --
 * every vertex takes the minimum over its frontier in-neighbours (reverse
 * CSR, w_eff of the first forward slot u -> v), exact min, no atomics on
 * dist -- for large frontiers, push steps for small ones (direction
 * optimisation).  Same dist as sp_sssp (the unique relaxation fixpoint). */
int sp_sssp_pull(sp_graph *g, int32_t src, int64_t cap, int32_t *dist, int mem,
                 int64_t *iters, sp_iter_cb cb, void *user, sp_stats *st);

/* Owner-computes SSSP shards for multi-GPU runs (graph.py:226-249 block
 * ownership; replaces the BSP superstep of bsp.py:290-335,393-417 for
 * sssp.sp, with convergence evaluated after the exchange).
 * A shard owns dist[v] for v in [v0, v1) of the caller's device array
 * dist (>= n entries, updated in place; the other entries are this rank's
 * candidates for remote vertices).  Per superstep:
 *   sp_sssp_shard_relax: up to max_rounds passes over the owned frontier
 *     (max_rounds > 1: the reference's local fixpoint, bsp.py:297-306);
 *     owned winners form the next local frontier, remote winners are sent
 *     as ONE message per vertex with the local minimum (aggregate_messages,
 *     bsp.py:45-72): send[] (device, capacity n) receives packed
 *     (vid << 32 | uint32 dist) grouped by owner rank (owner = vid / per),
 *     counts[world] (host) the group sizes.  info[4] (host, may be NULL):
 *     owned vertices lowered (Min wins, deduped per pass), slots relaxed,
 *     rounds run, owned frontier left.  SP_ERR_OVERFLOW: a distance left the int32 range.
 *   sp_sssp_shard_apply: the owner's strict min of received messages
 *     (bsp.py:350-368) -- msgs[k] packed as above -- or, when block != NULL,
 *     of block[v - v0] (a MIN reduce-scatter of every rank's dist array);
 *     *frontier = the owned frontier of the next superstep.  The run has
 *     converged when the frontiers of all ranks are empty. */
typedef struct sp_sssp_shard sp_sssp_shard;
int sp_sssp_shard_create(sp_graph *g, int64_t v0, int64_t v1, int32_t src, int world,
                         int32_t *dist, sp_sssp_shard **out);
int sp_sssp_shard_relax(sp_sssp_shard *h, int64_t max_rounds, int64_t per,
                        int64_t *send, int64_t *counts, int64_t *info);
int sp_sssp_shard_apply(sp_sssp_shard *h, const int64_t *msgs, int64_t k,
                        const int32_t *block, int64_t *frontier);
void sp_sssp_shard_destroy(sp_sssp_shard *h);
/* The exchange fused into the relaxation (instead of messages + an
 * all-to-all): with every rank's dist array, inbox (capacity n) and inbox
 * tail mapped into this process (sp_peer_alloc / sp_peer_open; over NVLink
 * between GPUs; indices = ranks, owner = v / per), sp_sssp_shard_relax
 * lowers a remote vertex's dist in its owner's array directly and, once per
 * superstep, appends the vertex to the owner's inbox -- counts come back 0.
 * After every rank's relax has completed (the caller's barrier),
 * sp_sssp_shard_collect appends this rank's inbox to its frontier, resets
 * the tail and returns the next frontier size. */
int sp_sssp_shard_peers(sp_sssp_shard *h, int64_t per, int32_t *const *peer_dist,
                        int32_t *const *peer_inbox, unsigned long long *const *peer_tail,
                        int32_t *inbox, unsigned long long *tail);
int sp_sssp_shard_collect(sp_sssp_shard *h, int64_t *frontier);

/* corpus/programs/pr.sp.  rank[n] = final ranks (== rank_nxt at exit);
 * iter / diff = the program's scalars; iters = fixedPoint iterations. */
int sp_pagerank(sp_graph *g, double damping, double epsilon, int64_t max_iter,
                int64_t cap, unsigned flags, double *rank, int mem,
                int64_t *iter, double *diff, int64_t *iters, sp_iter_cb cb,
                void *user, sp_stats *st);

/* Vertex-block PageRank shards for block-partitioned multi-GPU runs
 * (graph.py:226-249 ownership; replaces the BSP remote-read superstep of
 * bsp.py:182-185,287-288 for pr.sp).  sp_pagerank_block_init writes the
 * block's initial rank[v - v0] = 1/n and contrib_out[v - v0] = rank/outdeg.
 * A shard is planned once per run (slot/row bounds of the block, unit
 * index, scratch, hot sources); sp_pagerank_shard_step computes rank for
 * v in [v0, v1) from the full contrib_in[n] array, writes
 * contrib_out[v - v0] = rank/outdeg and the block's max |delta| into the
 * device double *diff.  stream != NULL: every step is enqueued on that
 * cudaStream_t (the caller's, e.g. torch's current stream) and returns
 * without synchronising; NULL: the library's stream, synchronised.  All
 * pointers are device pointers. */
typedef struct sp_pagerank_shard sp_pagerank_shard;
int sp_pagerank_block_init(sp_graph *g, int64_t v0, int64_t v1,
                           double *rank_local, double *contrib_out);
int sp_pagerank_shard_create(sp_graph *g, int64_t v0, int64_t v1, double damping,
                             unsigned flags, void *stream, sp_pagerank_shard **out);
int sp_pagerank_shard_step(sp_pagerank_shard *h, const double *contrib_in,
                           double *rank_local, double *contrib_out, double *diff);
void sp_pagerank_shard_destroy(sp_pagerank_shard *h);
/* The contrib exchange fused into the step (instead of an all-gather):
 * sp_pagerank_shard_peers gives the shard nsets x npeers device pointers
 * (set s, peer q: rank q's contrib array for the iterations of parity s,
 * global indices; mapped with sp_peer_open); sp_pagerank_shard_step_peers
 * then also stores every contrib it computes at peers[set][q][v] from the
 * producing kernel -- over NVLink for other GPUs.  The caller orders the
 * steps (e.g. the diff all-reduce of each iteration) and alternates sets so
 * a store never lands in an array a slower rank still reads. */
int sp_pagerank_shard_peers(sp_pagerank_shard *h, int nsets, int npeers,
                            double *const *peers);
int sp_pagerank_shard_step_peers(sp_pagerank_shard *h, const double *contrib_in,
                                 double *rank_local, double *contrib_out, double *diff,
                                 int set);

/* Peer-mapped device buffers (CUDA IPC): sp_peer_alloc allocates `bytes` on
 * `device` and writes its 64-byte IPC handle; another process maps it with
 * sp_peer_open (peer access over NVLink / the same GPU); sp_peer_free
 * unmaps (opened = 1) or frees (opened = 0). */
int sp_peer_alloc(int device, int64_t bytes, void **ptr, void *handle);
int sp_peer_open(int device, const void *handle, void **ptr);
void sp_peer_free(void *ptr, int opened);

/* corpus/programs/bc.sp over srcs in list order (duplicates re-run).
 * bc[n] accumulated; sigma/delta[n] of the LAST source (may be NULL). */
int sp_bc(sp_graph *g, const int32_t *srcs, int64_t nsrc, unsigned flags,
          double *bc, double *sigma, double *delta, int mem, sp_stats *st);

/* corpus/programs/tc.sp (tc.sp:3-13); exact, with multiplicity: every
 * triangle a-b-c contributes m_ab * m_bc * m_ac (slot multiplicities).
 * [v0, v1) selects a share of the triangles for sharded runs, so that the
 * shares of any partition of [0, n) sum to the whole count: undirected
 * graphs -- triangles whose lowest-ranked vertex (rank = (degree, id)) lies
 * in [v0, v1); directed graphs -- the program's middle vertex v in [v0, v1). */
int sp_tc(sp_graph *g, int64_t v0, int64_t v1, uint64_t *count, sp_stats *st);

/* Generic forall/reduction (corpus/programs/reduction.sp:5-10 and the
 * programs of its shape the host layer recognises, paper_2305_03317_b200/
 * forall.py): for every v, reduce a per-slot term over N(v) (reverse = 0,
 * g.neighbors) or over nodesTo(v) (reverse = 1); exact in any order.
 *   SP_REDUCE_SUM_I64: term = prop[u] (int64 node property) or, prop ==
 *     NULL, the constant iterm; per_vertex / total are int64.
 *   SP_REDUCE_MIN_F64 / SP_REDUCE_MAX_F64: term = the constant dterm;
 *     per_vertex / total are double, +inf / -inf for no slot.
 * per_vertex[n] (may be NULL) gets the row results, *total their reduction.
 * sp_neighbor_sum is the SUM form with iterm = 1. */
enum sp_reduce_op { SP_REDUCE_SUM_I64 = 0, SP_REDUCE_MIN_F64 = 1, SP_REDUCE_MAX_F64 = 2 };
int sp_neighbor_sum(sp_graph *g, const int64_t *prop, int mem, int reverse,
                    int64_t *per_vertex, int64_t *total, sp_stats *st);
int sp_neighbor_reduce(sp_graph *g, int op, int reverse, int64_t iterm, double dterm,
                       const int64_t *prop, int mem, void *per_vertex, void *total,
                       sp_stats *st);

#ifdef __cplusplus
}
#endif
#endif /* STARPLAT_B200_H */
