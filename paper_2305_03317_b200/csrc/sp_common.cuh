// sp_common.cuh -- shared runtime plumbing for the sm_100a graph backend.
#pragma once

#include <cuda_runtime.h>

#include <mutex>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/starplat_b200.h"

namespace sp {

constexpr int kIntMax = 2147483647;
constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs (queried at runtime too)

void set_error(const char *fmt, ...);
int cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define SP_CUDA(call)                                                        \
    do {                                                                     \
        cudaError_t _e = (call);                                             \
        if (_e != cudaSuccess)                                               \
            return ::sp::cuda_fail(_e, #call, __FILE__, __LINE__);           \
    } while (0)

#define SP_CHECK(cond, code, ...)                                            \
    do {                                                                     \
        if (!(cond)) {                                                       \
            ::sp::set_error(__VA_ARGS__);                                    \
            return (code);                                                   \
        }                                                                    \
    } while (0)

#define SP_TRY(call)                                                         \
    do {                                                                     \
        int _rc = (call);                                                    \
        if (_rc != SP_OK)                                                    \
            return _rc;                                                      \
    } while (0)

int num_sms(int device);

// Stream-ordered scratch allocation (cudaMallocAsync from the device's
// default pool, release threshold raised so repeated calls reuse memory).
int scratch_alloc(void **p, size_t bytes, cudaStream_t s);
void scratch_free(void *p, cudaStream_t s);
constexpr int kWorkerSlots = 16;
// serialises multi-worker calls on a device (they share the worker slots)
std::mutex &worker_slots_mutex(int dev);
int resident_alloc(void **p, size_t bytes);  // graph arrays (pool, any stream)
void resident_free(void *p);
constexpr size_t kPinnedBlock = 4096;
void *pinned_get();
void pinned_put(void *p);

// RAII holder for a per-call stream + scratch list + timing events.
struct Call {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    void *bufs[32];
    int nbufs = 0;
    int64_t launches = 0;
    void *pinned = nullptr;  // kPinnedBlock bytes of pinned host memory
    bool owned = true;       // stream/events belong to this call (else thread-cached)
    bool persisting = false; // an L2 access-policy window is set on the stream
    bool external = false;   // runs on a caller's stream: no sync at the end
    // as begin(), but enqueue on the caller's stream `s` (stream-ordered: the
    // call returns without synchronising; its scratch is freed in order)
    int begin_external(int dev, cudaStream_t s);
    // Keep [base, base+bytes) in the persisting L2 set-aside for this call's
    // kernels (random-access property arrays); best effort.
    void persist(const void *base, size_t bytes);
    int begin(int dev);
    // as begin(), on the persistent stream of worker slot k (k < kWorkerSlots)
    // of the device: a multi-worker call (sp_bc) spawns its host threads per
    // call, and per-thread streams would make every call allocate its scratch
    // on fresh streams; slot streams keep the pool's blocks reusable
    int begin_worker(int dev, int k);
    // this call's pinned host block (recycled across calls)
    int host(void **p);
    template <class T>
    int host_as(T **p) {
        void *q;
        SP_TRY(host(&q));
        *p = static_cast<T *>(q);
        return SP_OK;
    }
    template <class T>
    int alloc(T **p, size_t count) {
        void *q = nullptr;
        int rc = scratch_alloc(&q, count * sizeof(T) + 16, stream);
        if (rc != SP_OK) return rc;
        bufs[nbufs++] = q;
        *p = static_cast<T *>(q);
        return SP_OK;
    }
    int finish(sp_stats *st);  // sync + elapsed into st->device_ms
    ~Call();
};

// Launch `graph` through this thread's executable cache for (key, kind)
// (see sp_runtime.cu); the caller keeps ownership of `graph`.
enum { kLoopSsspBf = 1, kLoopSsspNf = 2, kLoopPr = 3, kLoopSsspDo = 4 };
int launch_cached_graph(cudaGraph_t graph, const void *key, int kind, cudaStream_t stream);

// Per host thread: instantiated graphs that read every per-call value from
// a device argument block owned by the entry (allocated with it), keyed by
// (graph uid, kind).  A later call on the same graph only copies its
// arguments into the block and launches: no capture, no update.
struct ArgExec {
    uint64_t key = 0;
    int kind = 0;
    int device = 0;
    cudaGraphExec_t exec = nullptr;
    void *args = nullptr;  // device argument block
    size_t bytes = 0;
};
// The entry for (key, kind) with an argument block of `bytes`; *fresh says
// whether the caller must (re)build e->exec: instantiate it when null, else
// refresh it with cudaGraphExecUpdate (an entry handed over from another
// graph of the same kind and layout).
int arg_exec_get(uint64_t key, int kind, size_t bytes, int device, ArgExec **out, bool *fresh);
enum { kArgPr = 1, kArgPrHot = 2, kArgPrRel = 3 };
uint64_t next_graph_uid();

// Copy a caller buffer to/from the device according to `mem`.
int to_device(void *dst, const void *src, size_t bytes, int mem, cudaStream_t s);
int from_device(void *dst, const void *src, size_t bytes, int mem, cudaStream_t s);

}  // namespace sp

// ---- the graph handle ----------------------------------------------------
struct sp_graph {
    uint64_t uid = sp::next_graph_uid();  // never reused (keys per-thread executable caches)
    int device = 0;
    int64_t n = 0, m = 0;
    int directed = 1;
    // forward CSR (graph.py:30-32)
    int64_t *off = nullptr;
    int32_t *adj = nullptr;
    int32_t *w = nullptr;
    int32_t *weff = nullptr;  // get_edge first-slot weight
    int32_t *rweff = nullptr; // w_eff of the forward slot behind each reverse slot (pull SSSP)
    int32_t *outdeg = nullptr;
    // reverse CSR (graph.py:33-35); aliases of off/adj when undirected
    int64_t *roff = nullptr;
    int32_t *radj = nullptr;
    int64_t *reid = nullptr;
    int32_t *indeg = nullptr;
    int64_t max_outdeg = 0, max_indeg = 0;
    // non-empty reverse rows (in-degree > 0) in ascending vertex order and
    // their row ends roff[v+1]: the row index of the edge-balanced PR pull
    int32_t *nzrow = nullptr;
    int64_t *nzend = nullptr;
    int64_t nnz_rows = 0;
    int32_t *wrange = nullptr;  // [min, max] weight (device), m > 0
    int32_t wmin_h = 0, wmax_h = 0;  // the same, on the host (read at creation)
    // degree-ordered upper CSR for triangle counting (undirected graphs),
    // built lazily by the first sp_tc call: row v holds the neighbours x of v
    // with (deg x, x) > (deg v, v), ascending, duplicates kept, starting at
    // slot 8*ustart8[v] (rows padded to 32 bytes with -1), ulen[v] entries;
    // uinfo[e] = (ustart8[x], ulen[x]) of the row slot e points to
    uint32_t *ustart8 = nullptr;
    int32_t *ulen = nullptr;
    int32_t *uadj = nullptr;
    uint2 *uinfo = nullptr;
    int32_t *uorder = nullptr;  // upper-CSR row r is the vertex uorder[r] (rows = degree ranks)
    bool tc_simple = false;     // no multi-edge: every upper-slot multiplicity is 1
    int64_t tc_hub_base = 0;    // upper rows >= this rank are hub rows (k_tc_big's bitmap form)
    int tc_hub_min = 0;         // hub rows longer than this are in ubig
    int64_t m_up = -1;      // real upper slots; -1: not built
    int64_t m_up_pad = 0;   // padded slots
    int32_t *ubig = nullptr;  // vertices whose upper row exceeds the warp path
    int64_t nbig = 0, max_ulen = 0;
    int tc_warp_max = 256;  // upper rows longer than this are in ubig (k_tc_big)
    // PageRank hot sources (built by the first fast PR call): the pr_H
    // vertices of largest out-degree, and radj re-encoded so that a slot
    // whose source is hot carries (1 << 30) | hot index
    int32_t *pr_hot_ids = nullptr;
    int32_t *pr_radj_hot = nullptr;
    int pr_H = -1;  // -1: not built, 0: disabled
    int pr_fast_calls = 0;  // fast PR calls so far (the hot set is built on the second)
    // edge-balanced PR plan of the whole graph (built by the first fast call):
    // unit_row[u] = first non-empty row whose end exceeds unit u's start
    int64_t *pr_unit_row = nullptr;
    int64_t pr_nunits = -1;
    // relabelled PR layout (built by the second fast call on a skewed
    // graph): vertices ranked by out-degree (descending, ties by id), the
    // reverse CSR in rank order with each row's sources as ranks, ascending
    // and laid out so that one warp load instruction reads consecutive ranks
    // (sp_pagerank.cu); rank r's original id is rel_order[r], v's rank is
    // rel_perm[v]
    int pr_rel = -1;  // -1: not decided, 0: not used, 1: built
    int pr_runs = 0;  // fast single-GPU PR runs started on this graph
    int sssp_do_runs = 0;  // direction-optimising SSSP runs (the hot set is built on the second)
    // bounded-degree (road-like) graphs: row v's (adj, w_eff) slots at
    // ell[v * ell_d ...], padded with x = -1 -- an expansion's row is found
    // from v alone, without the dependent offsets load (asynchronous SSSP)
    int2 *ell = nullptr;
    int ell_d = 0;
    // max out-degree <= 4: each row's 1-hop and 2-hop targets (min summed
    // w_eff per target, v itself dropped; 1-hop first), kEll2 slots per row -- shortcut
    // relaxations that halve the hop chain of the asynchronous SSSP kernel
    // (the fixpoint is unchanged: every shortcut weight is a real path length)
    int2 *ell2 = nullptr;
    int ell2_slots = 0;  // kEll2 or kEll3
    int32_t *rel_perm = nullptr, *rel_radj = nullptr, *rel_outdeg = nullptr,
            *rel_indeg = nullptr, *rel_nzrow = nullptr;
    int64_t *rel_nzend = nullptr, *rel_unit_row = nullptr;
    int64_t rel_nnz = 0, rel_nunits = 0;
    int rel_H = 0;
    // one-time preprocessing timers (sp_graph_prep_ms): device events at the
    // start and end of each lazily built structure, read on demand
    cudaEvent_t prep_ev[8][2] = {};
};

// ---- device helpers --------------------------------------------------------
namespace sp {

// Build the graph's w_eff array if it was deferred (thread-safe).
// PageRank hot-source selection (sp_pagerank.cu): for graph builders that
// encode radj while writing it (slot = kPrHotBit | hot index when hot).
constexpr int kPrHotBit = 1 << 30;
int pr_hot_prepare(sp_graph *g, Call &c, const int32_t *outdeg, int64_t max_outdeg,
                   int32_t **hot_idx, int *H);
// Build the hot-source encoding of radj now if the graph qualifies (sets
// g->pr_H: > 0 built, 0 not worth it); shared by PR and the SSSP pull sweep.
int pr_hot_build(sp_graph *g, Call &c);
int ensure_weff(sp_graph *g, Call &c);
// The lazily built per-graph structures whose build time sp_graph_prep_ms
// reports (SP_PREP_* in starplat_b200.h).
enum PrepKind {
    kPrepTcUpper = 0, kPrepWeff = 1, kPrepRweff = 2, kPrepPrHot = 3, kPrepPrRel = 4,
    kPrepEll = 5, kPrepEll2 = 6, kPrepKinds = 7
};
// Records the start (end = 0) or the end (end = 1) of one build on stream s.
void prep_mark(sp_graph *g, int kind, int end, cudaStream_t s);
// Reverse-slot weights rweff[k] = w_eff[reid[k]] (undirected: w_eff itself).
int ensure_rweff(sp_graph *g, Call &c);
// The ELL form above (built once when max out-degree <= d_max; else no-op).
int ensure_ell(sp_graph *g, Call &c, int d_max);
// 2-hop row slots: a 4-regular grid row has exactly 4 + 8 targets
// (cfg5a: 12 slots 27.7 ms, 16 slots 30.7 ms -- fewer dead lanes and
// rounds); rows with more distinct targets keep the first 12 (1-hop first)
#ifndef SP_NF_ELL2_SLOTS
#define SP_NF_ELL2_SLOTS 12
#endif
constexpr int kEll2 = SP_NF_ELL2_SLOTS, kEll3 = 32;
// The shortcut form above (built once from the ELL rows when ell_d <= 4):
// hops = 2 -> kEll2 slots, hops = 3 -> kEll3 slots (1-, 2-, then 3-hop
// targets while they fit; dropping a shortcut never changes the fixpoint).
int ensure_ell2(sp_graph *g, Call &c, int hops);

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Max of non-negative doubles via their IEEE bit patterns (order-preserving).
__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long *>(addr),
              static_cast<unsigned long long>(__double_as_longlong(v)));
}

// Warp-aggregated append: lanes with `want` get consecutive slots.
__device__ __forceinline__ int64_t warp_append(bool want, unsigned long long *counter) {
    unsigned mask = __ballot_sync(0xffffffffu, want);
    if (!mask) return -1;
    int leader = __ffs(mask) - 1;
    unsigned long long base = 0;
    if ((int)lane_id() == leader) base = atomicAdd(counter, (unsigned long long)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (!want) return -1;
    return (int64_t)base + __popc(mask & ((1u << lane_id()) - 1u));
}

// Warp-aggregated append of K rounds at once: round u's lanes with
// push[u] get consecutive slots, one global atomic for the whole batch.
template <int K>
__device__ __forceinline__ void warp_append_multi(const bool (&push)[K], const int32_t (&val)[K],
                                                  unsigned long long *counter, int32_t *out,
                                                  unsigned long long cap = ~0ull) {
    unsigned m[K];
    unsigned total = 0;
#pragma unroll
    for (int u = 0; u < K; u++) {
        m[u] = __ballot_sync(0xffffffffu, push[u]);
        total += __popc(m[u]);
    }
    if (!total) return;
    unsigned long long base = 0;
    if (lane_id() == 0) base = atomicAdd(counter, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 0);
    const unsigned lt = (1u << lane_id()) - 1u;
#pragma unroll
    for (int u = 0; u < K; u++) {
        const unsigned long long at = base + __popc(m[u] & lt);
        if (push[u] && at < cap) out[at] = val[u];  // the counter still counts overflow
        base += __popc(m[u]);
    }
}

// Per-warp staging of queue appends in shared memory: entries collect in a
// warp-private buffer and go to the global queue in batches of up to kCap,
// one global atomic per batch (a single global counter shared by every warp
// serialises at one L2 slice otherwise).  `n` is warp-uniform.
template <int kCap>
struct WarpStage {
    int32_t *buf;  // kCap entries of shared memory, private to the warp
    int n = 0;

    __device__ __forceinline__ void flush(unsigned long long *counter, int32_t *out,
                                          unsigned long long cap = ~0ull) {
        if (n == 0) return;
        __syncwarp();
        unsigned long long base = 0;
        if (lane_id() == 0) base = atomicAdd(counter, (unsigned long long)n);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int i = lane_id(); i < n; i += 32)
            if (base + i < cap) out[base + i] = buf[i];  // the counter still counts overflow
        __syncwarp();
        n = 0;
    }

    template <int K>
    __device__ __forceinline__ void push(const bool (&p)[K], const int32_t (&val)[K],
                                         unsigned long long *counter, int32_t *out,
                                         unsigned long long cap = ~0ull) {
        static_assert(K * 32 <= kCap, "one push must fit an empty stage");
        unsigned m[K];
        int total = 0;
#pragma unroll
        for (int u = 0; u < K; u++) {
            m[u] = __ballot_sync(0xffffffffu, p[u]);
            total += __popc(m[u]);
        }
        if (total == 0) return;
        if (n + total > kCap) flush(counter, out, cap);
        const unsigned lt = (1u << lane_id()) - 1u;
        int at = n;
#pragma unroll
        for (int u = 0; u < K; u++) {
            if (p[u]) buf[at + __popc(m[u] & lt)] = val[u];
            at += __popc(m[u]);
        }
        n = at;
    }
};

__device__ __forceinline__ int ld_stream_i32(const int32_t *p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

inline int grid_for(int64_t work, int block, int device, int per_sm = 8) {
    int64_t g = (work + block - 1) / block;
    int64_t cap = (int64_t)num_sms(device) * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace sp
