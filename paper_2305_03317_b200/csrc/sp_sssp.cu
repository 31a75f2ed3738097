// sp_sssp.cu -- corpus/programs/sssp.sp on sm_100a.
//
// Reference semantics (trident/interp.py): fixedPoint until (finished:
// !modified) { forall v with modified: forall nbr in neighbors(v):
// <nbr.dist, nbr.modified_nxt> = <Min(nbr.dist, v.dist + w(get_edge)), True>;
// modified = modified_nxt; modified_nxt = False }.  The result is the unique
// relaxation fixpoint, so a parallel frontier Bellman-Ford produces the same
// dist bit-for-bit; only the iteration count may differ from the
// interpreter's in-place (Gauss-Seidel) order.
//
// Device layout: dist int32[n], enq int32[n] (iteration stamp of the last
// enqueue -> dedupes the next frontier, the device form of modified_nxt),
// two frontier queues int32[n] (the device form of `modified`).
// One iteration = the load-balanced expansion of sp_expand.cuh over the
// frontier (warp-flattened rows + hub chunks) with RelaxOp:
//   * relax: cand = (int64)dist[v] + w_eff[e]; a plain load of dist[x]
//     filters non-improving candidates (dist only decreases, so a stale read
//     is conservative) before the atomicMin; a winner stamps enq[x] and is
//     appended to the next frontier with one atomic per warp;
//   * the frontier size is the convergence flag (finished = size == 0):
//     one 8-byte device->host read per iteration (K5/K6 in SURVEY 2.2).
// The Bellman-Ford device loop (CUDA-graph WHILE node) keeps dist and the
// enqueue stamp in one 64-bit word per vertex instead (RelaxPackedOp): one
// atomicMin relaxes and, through the old word, dedupes the next frontier.
// Large graphs run the direction-optimising loop (push steps + edge-
// balanced pull sweeps), thin non-negative graphs the asynchronous
// near-far kernel (per-block ring queues, no barrier per hop).
// Candidates >= INT_MAX never win (interp.py:11-14).
#include <cooperative_groups.h>

#include <chrono>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "sp_expand.cuh"

using namespace sp;

namespace {

constexpr int kBlock = 256;
constexpr int64_t kDeltaMul = 16;        // near-far step = kDeltaMul x mean weight
constexpr int64_t kNearFarMaxAvgDeg = 8;  // near-far only when m <= 8 n
constexpr int kPersistBlocksPerSm = 2;    // persistent near-far grid: blocks per SM (cfg5a: 1 -> 87.8 ms, 2 -> 86.0 ms)
constexpr int kAsyncBlocksPerSm = 1;  // asynchronous near-far: blocks per SM
constexpr int kNfHops = 2;  // warp-local continuation hops (persistent near-far); cfg5a: 1-4 ~87-93 ms, 8 -> 120 ms, 16 -> 158 ms

// Relaxation of sssp.sp:11-12 for one slot; payload = dist[v] at expansion.
struct RelaxOp {
    using Payload = int;
    struct Probe {
        int w;   // w_eff[e]
        int dx;  // dist[x] (may be stale: dist only decreases, so conservative)
    };
    int32_t *__restrict__ dist;
    int32_t *__restrict__ enq;
    const int32_t *__restrict__ weff;
    unsigned long long *overflow;
    int it;
    __device__ __forceinline__ int payload(int32_t v) const { return __ldcg(dist + v); }
    __device__ __forceinline__ Probe probe(int64_t e, int32_t x) const {
        return Probe{__ldcs(weff + e), __ldcg(dist + x)};
    }
    // Not phased (sp_expand.cuh): on RMAT the phased form measured slower
    // (register spills, re-evaluated filters) -- the dense iterations are
    // bound by probe/atomic throughput, not by the atomic chain.
    __device__ __forceinline__ bool apply(int dv, int64_t, int32_t x, Probe p) const {
        const int64_t cand = (int64_t)dv + (int64_t)p.w;
        if (cand >= (int64_t)kIntMax) return false;  // never beats INT_MAX (F12)
        if (cand < (int64_t)(-2147483647 - 1)) {
            atomicAdd(overflow, 1ull);
            return false;
        }
        const int c = (int)cand;
        if (c >= p.dx) return false;  // conservative pre-filter
        const int old = atomicMin(dist + x, c);
        return c < old && atomicExch(enq + x, it) != it;
    }
};

// RelaxOp with dist and the enqueue stamp in one 64-bit word per vertex
// (high half: dist, low half: the iteration that queued it): one atomicMin
// relaxes and, through the old word, says whether x was already queued this
// iteration -- one returning atomic per improving slot instead of two in
// series.  Ordered by dist first (the stamp only breaks ties, which never
// count as improvements).
struct RelaxPackedOp {
    using Payload = int;
    using Probe = RelaxOp::Probe;
    long long *__restrict__ dq;
    const int32_t *__restrict__ weff;
    unsigned long long *overflow;
    int it;
    __device__ __forceinline__ int payload(int32_t v) const { return (int)(__ldcg(dq + v) >> 32); }
    __device__ __forceinline__ Probe probe(int64_t e, int32_t x) const {
        return Probe{__ldcs(weff + e), (int)(__ldcg(dq + x) >> 32)};
    }
    __device__ __forceinline__ bool apply(int dv, int64_t, int32_t x, Probe p) const {
        const int64_t cand = (int64_t)dv + (int64_t)p.w;
        if (cand >= (int64_t)kIntMax) return false;  // never beats INT_MAX (F12)
        if (cand < (int64_t)(-2147483647 - 1)) {
            atomicAdd(overflow, 1ull);
            return false;
        }
        const int c = (int)cand;
        if (c >= p.dx) return false;  // conservative pre-filter
        const long long w = (long long)(((unsigned long long)(unsigned)c << 32) | (unsigned)it);
        const long long old = atomicMin(dq + x, w);
        return (int)(old >> 32) > c && (unsigned)old != (unsigned)it;
    }
};

__global__ void k_init_packed(long long *dq, int64_t n, int32_t src) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x)
        dq[x] = x == src ? 0ll : (long long)(((unsigned long long)kIntMax << 32) | 0xFFFFFFFFull);
}

__global__ void k_unpack(const long long *__restrict__ dq, int64_t n, int32_t *dist) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x)
        dist[x] = (int32_t)(dq[x] >> 32);
}

__global__ void k_init(int32_t *dist, int32_t *enq, int64_t n, int32_t src, int32_t *q) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        dist[x] = x == src ? 0 : kIntMax;
        enq[x] = x == src ? 0 : -1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) q[0] = src;
}

// ---- device-side fixedPoint loop (CUDA graph with a conditional WHILE node)
// The loop state lives on the device; the body is the expansion (+ hub
// chunks) followed by a one-thread advance kernel that folds the counters
// into the totals, swaps the queues, resets the next counters and sets the
// loop condition (frontier non-empty, no overflow, below the cap).  No host
// round trip per iteration: used whenever no per-iteration callback is set.
struct SsspLoop {
    int32_t *q[2];
    ExpandCounters cnt[2];
    int cur;       // q[cur] is the frontier being expanded
    int it;        // enqueue stamp of this iteration (iters + 1)
    int64_t nq;    // |q[cur]|
    int64_t iters, relaxed, frontier_sum, cap;
    int status;    // 0 ok / converged, 1 overflow, 2 cap reached
    unsigned blocks_done;  // k_relax_loop_chunks: the last block runs the advance
};

#ifndef SP_RL_MINB
#define SP_RL_MINB 5  // RMAT-22 SSSP 1.71 -> 1.57 ms (with SP_RLC_MINB 4); 6: slower
#endif
#ifndef SP_RLC_MINB
#define SP_RLC_MINB 4
#endif
// Op: RelaxOp or RelaxPackedOp; its overflow counter and stamp are this
// iteration's (from L)
template <class Op>
__global__ void __launch_bounds__(kExpandBlock, SP_RL_MINB) k_relax_loop(
    Op op, const int64_t *__restrict__ off, const int32_t *__restrict__ adj, ChunkItem *chunks,
    SsspLoop *L, int64_t warps) {
    const int cur = L->cur;
    const int64_t nq = L->nq;
    op.overflow = &L->cnt[cur].flag;
    op.it = L->it;
    expand_body(op, off, adj, L->q[cur], nq, L->q[cur ^ 1], chunks, &L->cnt[cur],
                expand_vpw(nq, warps));
}

__device__ __forceinline__ int loop_advance(SsspLoop *L);

// Hub chunks; the last block to finish also runs the loop advance (one
// graph node per iteration fewer: ~4 us of node latency each, cfg1 runs
// 9-10 iterations of ~40 us).
template <class Op>
__global__ void __launch_bounds__(kExpandBlock, SP_RLC_MINB) k_relax_loop_chunks(
    Op op, const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
    const ChunkItem *chunks, SsspLoop *L, cudaGraphConditionalHandle h) {
    const int cur = L->cur;
    op.overflow = &L->cnt[cur].flag;
    op.it = L->it;
    expand_chunks_body(op, off, adj, chunks, L->q[cur ^ 1], &L->cnt[cur]);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();  // this block's counter updates before its arrival
        if (atomicAdd(&L->blocks_done, 1u) == gridDim.x - 1) {
            __threadfence();
            L->blocks_done = 0;
            cudaGraphSetConditional(h, loop_advance(L));
        }
    }
}

__global__ void k_loop_advance(SsspLoop *L, cudaGraphConditionalHandle h) {
    cudaGraphSetConditional(h, loop_advance(L));
}

__device__ __forceinline__ int loop_advance(SsspLoop *L) {
    const int cur = L->cur;
    const ExpandCounters c = L->cnt[cur];
    L->iters++;
    L->frontier_sum += L->nq;
    L->relaxed += (int64_t)c.scanned;
    int go = 1;
    if (c.flag) {
        L->status = 1;
        go = 0;
    } else if (c.next_size == 0) {
        go = 0;  // finished = !modified
    } else if (L->iters >= L->cap) {
        L->status = 2;
        go = 0;
    }
    L->cnt[cur ^ 1] = ExpandCounters{0, 0, 0, 0};
    L->cur = cur ^ 1;
    L->nq = (int64_t)c.next_size;
    L->it = (int)(L->iters + 1);
    return go;
}

// ---- near-far ordering (large-diameter graphs, non-negative weights) -----
// Improvements below the threshold T go to the near queue (processed next
// iteration), the others to a far pile.  When the near queue runs dry, T
// grows by delta and k_nf_split moves the far entries below T back (stale
// and already-expanded entries are dropped).  `last[v]` is the distance v
// was last expanded with: a queue entry is expanded only if dist[v] < last.
// Same fixpoint as Bellman-Ford, far fewer repeated relaxations on graphs
// whose shortest paths are many hops long (road-like grids).
struct NfLoop {
    int32_t *q[2];
    int32_t *far[2];
    ExpandCounters cnt[2];
    unsigned long long far_n[2];
    unsigned long long split_n;  // near entries appended by k_nf_split
    int cur, fcur;
    int it;
    int64_t nq;
    int64_t T, delta;
    int64_t iters, relaxed, frontier_sum, cap;
    unsigned long long fcap;  // far pile capacity
    int status;               // 0 ok, 1 overflow, 2 cap, 3 far pile overflow
    int go;                   // persistent kernel: continue
};

struct NearFarOp {
    using Payload = int;
    using Probe = RelaxOp::Probe;
    static constexpr bool kFar = true;
    static constexpr bool kPhased = true;
    int32_t *__restrict__ dist;
    int32_t *__restrict__ enq;
    int32_t *__restrict__ last;
    const int32_t *__restrict__ weff;
    unsigned long long *overflow;
    int32_t *far_q;
    unsigned long long *far_n;
    unsigned long long far_cap;
    int64_t T;
    int it;
    __device__ __forceinline__ int payload(int32_t v) const { return __ldcg(dist + v); }
    __device__ __forceinline__ bool keep(int32_t v, int dv) const {
        if (dv >= __ldcg(last + v)) return false;  // expanded at this distance already
        last[v] = dv;
        return true;
    }
    __device__ __forceinline__ Probe probe(int64_t e, int32_t x) const {
        return Probe{__ldcs(weff + e), __ldcg(dist + x)};
    }
    __device__ __forceinline__ bool go(int dv, int32_t x, Probe p, int &c) const {
        if (x < 0) return false;
        const int64_t cand = (int64_t)dv + (int64_t)p.w;
        c = (int)cand;
        return cand < (int64_t)kIntMax && cand >= (int64_t)(-2147483647 - 1) && c < p.dx;
    }
    // improvements below T go to the near queue (once per iteration), the
    // rest to the far pile.  Phased: the grid's thin frontiers are bound by
    // the atomic round trips (measured 130 -> 119 ms on cfg5a).
    __device__ __forceinline__ int apply(int dv, int64_t, int32_t x, Probe p) const {
        int c = 0;
        const bool g = go(dv, x, p, c);
        if (x >= 0 && (int64_t)dv + (int64_t)p.w < (int64_t)(-2147483647 - 1))
            atomicAdd(overflow, 1ull);
        return atom_min_if(g, dist + x, c);
    }
    __device__ __forceinline__ int settle(int old, int32_t x, int dv, Probe p) const {
        int c = 0;
        const bool near = go(dv, x, p, c) && c < old && (int64_t)c < T;
        return atom_exch_if(near, enq + x, it);
    }
    __device__ __forceinline__ int result(int old, int stamp, int32_t x, int dv, Probe p) const {
        int c = 0;
        if (!(go(dv, x, p, c) && c < old)) return 0;
        return (int64_t)c < T ? (stamp != it ? 1 : 0) : 2;
    }
};

__global__ void __launch_bounds__(kExpandBlock, 4) k_nf_expand(
    int32_t *dist, int32_t *enq, int32_t *last, const int32_t *__restrict__ weff,
    const int64_t *__restrict__ off, const int32_t *__restrict__ adj, ChunkItem *chunks, NfLoop *L,
    int64_t warps) {
    const int cur = L->cur;
    const int64_t nq = L->nq;
    if (nq == 0) return;
    NearFarOp op{dist, enq, last, weff, &L->cnt[cur].flag, L->far[L->fcur], &L->far_n[L->fcur],
                 L->fcap, L->T, L->it};
    expand_body(op, off, adj, L->q[cur], nq, L->q[cur ^ 1], chunks, &L->cnt[cur],
                expand_vpw(nq, warps));
}

__global__ void __launch_bounds__(kExpandBlock, 3) k_nf_chunks(
    int32_t *dist, int32_t *enq, int32_t *last, const int32_t *__restrict__ weff,
    const int64_t *__restrict__ off, const int32_t *__restrict__ adj, const ChunkItem *chunks,
    NfLoop *L) {
    const int cur = L->cur;
    if (L->nq == 0) return;
    NearFarOp op{dist, enq, last, weff, &L->cnt[cur].flag, L->far[L->fcur], &L->far_n[L->fcur],
                 L->fcap, L->T, L->it};
    expand_chunks_body(op, off, adj, chunks, L->q[cur ^ 1], &L->cnt[cur]);
}

// The far pile is split when the expansion produced no near entries (every
// block of k_nf_split and k_nf_advance derive the same decision from the
// finished expansion counters; T for the split is T + delta).
__device__ __forceinline__ bool nf_split_now(const NfLoop *L) {
    const ExpandCounters &c = L->cnt[L->cur];
    return c.next_size == 0 && !c.flag && L->far_n[L->fcur] <= L->fcap;
}

// Far entries below T -> near queue (if not stale / not expanded at this
// distance); the rest -> the other far pile.
__global__ void k_nf_split(const int32_t *__restrict__ dist, int32_t *enq,
                           const int32_t *__restrict__ last, NfLoop *L) {
    if (!nf_split_now(L)) return;
    const int cur = L->cur, fc = L->fcur;
    const int64_t nf = (int64_t)min(L->far_n[fc], L->fcap);
    const int32_t *src = L->far[fc];
    const int64_t T = L->T + L->delta;
    const int it = L->it;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < nf; b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = b + threadIdx.x;
        bool to_near = false, to_far = false;
        int32_t v = 0;
        if (i < nf) {
            v = src[i];
            const int d = __ldcg(dist + v);
            if ((int64_t)d < T) {
                to_near = d < __ldcg(last + v) && atomicExch(enq + v, it) != it;
            } else {
                to_far = true;
            }
        }
        const bool nb[1] = {to_near}, fb[1] = {to_far};
        const int32_t xv[1] = {v};
        warp_append_multi<1>(nb, xv, &L->split_n, L->q[cur ^ 1]);
        warp_append_multi<1>(fb, xv, &L->far_n[fc ^ 1], L->far[fc ^ 1], L->fcap);
    }
}

__global__ void k_nf_advance2(NfLoop *L, cudaGraphConditionalHandle h) {
    const int cur = L->cur;
    const ExpandCounters c = L->cnt[cur];
    const bool split = nf_split_now(L);  // same decision k_nf_split took
    L->frontier_sum += L->nq;
    L->relaxed += (int64_t)c.scanned;
    L->iters++;
    int64_t next = (int64_t)c.next_size;
    if (split) {
        L->T += L->delta;
        L->far_n[L->fcur] = 0;
        L->fcur ^= 1;
        next = (int64_t)L->split_n;
        L->split_n = 0;
    }
    int go = 1;
    const bool far_left = L->far_n[L->fcur] > 0;
    if (L->far_n[0] > L->fcap || L->far_n[1] > L->fcap) {
        L->status = 3;  // the caller falls back to plain Bellman-Ford
        go = 0;
    } else if (c.flag) {
        L->status = 1;
        go = 0;
    } else if (next == 0 && !far_left) {
        go = 0;  // nothing near, nothing far: finished
    } else if (L->iters >= L->cap) {
        L->status = 2;
        go = 0;
    }
    L->cnt[cur ^ 1] = ExpandCounters{0, 0, 0, 0};
    L->cur = cur ^ 1;
    L->nq = next;
    L->it = (int)(L->iters + 1);
    cudaGraphSetConditional(h, go);
}

__global__ void k_fill_i32(int32_t *p, int64_t n, int32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// Persistent near-far loop for thin graphs (every row <= kSplit slots): one
// cooperative launch runs all iterations, grid-wide barriers between the
// expansion, the far split and the advance (a few microseconds per
// iteration instead of one graph node launch per kernel).
__global__ void __launch_bounds__(kExpandBlock) k_nf_persistent(
    int32_t *dist, int32_t *enq, int32_t *last, const int32_t *__restrict__ weff,
    const int64_t *__restrict__ off, const int32_t *__restrict__ adj, NfLoop *L) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (;;) {
        {   // near expansion
            const int cur = L->cur;
            const int64_t nq = L->nq;
            if (nq > 0) {
                NearFarOp op{dist, enq, last, weff, &L->cnt[cur].flag, L->far[L->fcur],
                             &L->far_n[L->fcur], L->fcap, L->T, L->it};
                expand_body<NearFarOp, kNfHops>(op, off, adj, L->q[cur], nq, L->q[cur ^ 1],
                                                 nullptr, &L->cnt[cur], expand_vpw(nq, warps));
            }
        }
        grid.sync();
        if (nf_split_now(L)) {  // same decision in every block
            const int cur = L->cur, fc = L->fcur;
            const int64_t nf = (int64_t)min(L->far_n[fc], L->fcap);
            const int32_t *src = L->far[fc];
            const int64_t T = L->T + L->delta;
            const int it = L->it;
            for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < nf;
                 b += (int64_t)gridDim.x * blockDim.x) {
                const int64_t i = b + threadIdx.x;
                bool to_near = false, to_far = false;
                int32_t v = 0;
                if (i < nf) {
                    v = src[i];
                    const int d = __ldcg(dist + v);
                    if ((int64_t)d < T)
                        to_near = d < __ldcg(last + v) && atomicExch(enq + v, it) != it;
                    else
                        to_far = true;
                }
                const bool nb[1] = {to_near}, fb[1] = {to_far};
                const int32_t xv[1] = {v};
                warp_append_multi<1>(nb, xv, &L->split_n, L->q[cur ^ 1]);
                warp_append_multi<1>(fb, xv, &L->far_n[fc ^ 1], L->far[fc ^ 1], L->fcap);
            }
        }
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) {  // advance (k_nf_advance2)
            const int cur = L->cur;
            const ExpandCounters c = L->cnt[cur];
            const bool split = nf_split_now(L);
            L->frontier_sum += L->nq;
            L->relaxed += (int64_t)c.scanned;
            L->iters++;
            int64_t next = (int64_t)c.next_size;
            if (split) {
                L->T += L->delta;
                L->far_n[L->fcur] = 0;
                L->fcur ^= 1;
                next = (int64_t)L->split_n;
                L->split_n = 0;
            }
            int go = 1;
            const bool far_left = L->far_n[L->fcur] > 0;
            if (L->far_n[0] > L->fcap || L->far_n[1] > L->fcap) {
                L->status = 3;
                go = 0;
            } else if (c.flag) {
                L->status = 1;
                go = 0;
            } else if (next == 0 && !far_left) {
                go = 0;
            } else if (L->iters >= L->cap) {
                L->status = 2;
                go = 0;
            }
            L->cnt[cur ^ 1] = ExpandCounters{0, 0, 0, 0};
            L->cur = cur ^ 1;
            L->nq = next;
            L->it = (int)(L->iters + 1);
            L->go = go;
        }
        grid.sync();
        if (!L->go) break;
    }
}


// ---- asynchronous near-far (thin graphs, non-negative weights) ----------
// One cooperative launch; no grid-wide barrier per hop.  Improvements below
// the threshold T go to ring queues, the rest to a far pile.  Every block
// owns one ring -- vertex x belongs to ring (x / 16) mod #blocks -- whose
// head is a shared-memory counter of the block; its warps pop up to 32
// consecutive published entries at a time, expand them and push their near
// improvements to the owners' rings (one tail atomic per group of lanes
// with the same owner).  A shortest path thus advances one hop per
// dependent round trip instead of one per grid-wide iteration
// (k_nf_persistent: three grid barriers per iteration, 60% of its warp
// samples stalled on them; a single global ring measured 0.37 s on cfg5a,
// its warps queued on the head CAS).
//   dq[v] = dist << 1 | queued: one atomicMin both lowers the distance and
//   marks the vertex queued, and its old value says whether the winner must
//   push it (the queued bit was clear); a popper's atomicAnd clears the bit
//   and returns the distance to expand with -- so an improvement either
//   re-queues v or is seen by the popper, with no separate flag round trip.
//   `work` counts entries pushed and not yet expanded (a batch raises it by
//   its slot count before any of its pushes and returns the surplus after):
//   zero means the phase is drained.  Then (grid barriers, once per phase)
//   T grows by delta, every ring restarts at 0 (no lap: a phase that
//   overflows a ring aborts to the synchronous kernel) and the far pile is
//   split.  Expansion order does not change the fixpoint: `dist` is
//   bit-identical to Bellman-Ford's.
struct AsyncNf {
    int32_t *ring;                  // nring rings of cap entries
    unsigned long long *tails;      // ring r's tail at tails[r * kTailStride]
    unsigned long long cap;
    int nring;
    alignas(128) long long work;
    alignas(128) int32_t *far[2];
    unsigned long long far_n[2];
    unsigned long long fcap;
    int fcur;
    int go;
    int abort;
    int status;                     // 0 ok, 3 far-pile / ring overflow, 4 watchdog
    int64_t T, delta;
    int64_t phases;
    unsigned long long relaxed, expanded, batches;
    unsigned long long far_scanned, between_cycles;  // diagnostics (SP_SSSP_TRACE)
};

constexpr int kAsyncBlock = 1024;  // launch bound; the launch uses kAsyncThreads
constexpr int kAsyncThreads = 256;
constexpr unsigned kAsyncBackoff = 256;
constexpr int kTailStride = 16;    // one 128-byte line per ring tail
#ifndef SP_NF_OWN_SHIFT
#define SP_NF_OWN_SHIFT 4
#endif
// 2^4 consecutive vertices per ring chunk: cfg5a, 1-hop rows, shift 4 / 6 /
// 8 / 10 / 12 -> 39.5 / 39.6 / 42.0 / 46.0 / 39.8 ms; 2-hop shortcut rows,
// 3 / 4 / 5 / 6 / 7 / 8 -> 25.5 / 25.5 / 25.6 / 26.2 / 27.1 / 28.2 ms
constexpr int kOwnShift = SP_NF_OWN_SHIFT;
constexpr int kEllMaxDeg = 8;      // ELL rows for graphs with max out-degree <= 8
constexpr long long kAsyncWatchdog = 1ll << 35;  // cycles (~17 s): a hang becomes a fallback

__device__ __forceinline__ int async_owner(int32_t x, int nring) {
    return (int)((uint32_t)((uint32_t)x >> kOwnShift) % (uint32_t)nring);
}

__device__ __forceinline__ void async_fail(AsyncNf *A, int status) {
    A->status = status;
    A->abort = 1;
}

// Push the lanes' near entries to their owners' rings, one tail atomic per
// group of lanes with the same owner.  `work` must count an entry before its
// tail moves: the split (counted = false) raises it here; an expansion batch
// raised it by its slot count when the batch began (tok = that atomic's
// result in lane 0: every tail atomic below depends on it, so it is issued
// only after the raise was performed -- the raise itself overlapped the
// batch's loads).  Returns the entries pushed.
__device__ __forceinline__ int async_push_near(AsyncNf *A, bool near, int32_t x, unsigned lane,
                                               bool counted, unsigned long long tok = 0) {
    const unsigned m = __ballot_sync(0xffffffffu, near);
    if (!m) return 0;
    if (!counted) {
        if (lane == 0)
            atomicAdd(reinterpret_cast<unsigned long long *>(&A->work),
                      (unsigned long long)__popc(m));
        __syncwarp();
    }
    tok = __shfl_sync(0xffffffffu, tok, 0);
    if (near) {
        const int r = async_owner(x, A->nring);
        const unsigned grp = __match_any_sync(m, r);
        const int leader = __ffs(grp) - 1;
        unsigned long long pos = 0;
        if ((int)lane == leader)
            pos = atomicAdd(A->tails + (size_t)r * kTailStride + (tok == ~0ull ? 1 : 0),
                            (unsigned long long)__popc(grp));
        pos = __shfl_sync(grp, pos, leader) + __popc(grp & ((1u << lane) - 1u));
        if (pos < A->cap)
            reinterpret_cast<volatile int32_t *>(A->ring)[(size_t)r * A->cap + pos] = x;
        else
            async_fail(A, 3);  // the ring overflowed within a phase
    }
    return __popc(m);
}

__device__ __forceinline__ void async_push_far(AsyncNf *A, int fc, bool far, int32_t x,
                                               unsigned lane) {
    const unsigned m = __ballot_sync(0xffffffffu, far);
    if (!m) return;
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(&A->far_n[fc], (unsigned long long)__popc(m));
    pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(m & ((1u << lane) - 1u));
    if (far && pos < A->fcap) A->far[fc][pos] = x;  // far_n still counts an overflow
}

// Push a warp's shared list of near winners (nn entries) to their owners'
// rings, 32 at a time (one tail atomic per owner group per 32); `work`
// already counts them (tok: the batch's raise).  Returns nn.
constexpr int kNearList = 128;
__device__ __forceinline__ int async_push_list(AsyncNf *A, const int32_t *nl, int nn,
                                               unsigned lane, unsigned long long tok) {
    __syncwarp();
    for (int b = 0; b < nn; b += 32) {
        const bool has = b + (int)lane < nn;
        const int32_t x = has ? nl[b + lane] : -1;
        async_push_near(A, has, x, lane, true, tok);
    }
    __syncwarp();
    return nn;
}

// kD > 0: bounded-degree graphs in the ELL form (g->ell, kD slots per row):
// a lane loads its vertex's whole row (one or two 16-byte loads) from v
// alone, in parallel with the dequeue atomic -- no dependent offsets load
// on the hop chain.  kD == 0: CSR rows, flattened over the warp.
// shortcut rows keep their slots and atomic results in registers: a lower
// thread bound (2-hop: 512 -> <= 128 registers; 3-hop: 256)
constexpr int async_bound(int kD) { return kD == kEll3 ? 256 : kD == kEll2 ? 512 : kAsyncBlock; }
template <int kD>
__global__ void __launch_bounds__(async_bound(kD)) k_nf_async(
    unsigned long long *dq, int32_t *last, const int32_t *__restrict__ weff,
    const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
    const int2 *__restrict__ ell, AsyncNf *A, unsigned async_max_backoff) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ unsigned long long s_head;  // this block's ring: next entry to pop
    if (threadIdx.x == 0) s_head = 0;
    __syncthreads();
    const unsigned lane = lane_id();
    volatile AsyncNf *VA = A;
    volatile unsigned long long *vhead = &s_head;
    const unsigned long long cap = A->cap;
    volatile int32_t *myring = A->ring + (size_t)blockIdx.x * cap;
    unsigned long long relaxed = 0, expanded = 0, batches = 0;
    const long long t_start = clock64();
    for (;;) {
        const int64_t T = VA->T;  // fixed during a phase (written between barriers)
        const int fc = VA->fcur;
        // ---- drain the rings
        unsigned backoff = 0;
        for (;;) {
            // poll the slots after the head: the published entries are the
            // ones already written (a reserved slot still reads -1)
            const unsigned long long h = *vhead;
            const int32_t sv = h + lane < cap ? myring[h + lane] : -1;
            const unsigned pub = __ballot_sync(0xffffffffu, sv >= 0);
            const int k = __ffs(~pub) - 1 < 0 ? 32 : __ffs(~pub) - 1;  // consecutive from h
            if (k == 0) {
                long long w = 1;
                if (lane == 0) {
                    w = VA->work;
                    if (VA->abort) {
                        w = 0;
                    } else if (clock64() - t_start > kAsyncWatchdog) {
                        async_fail(A, 4);
                        w = 0;
                    }
                }
                if (__shfl_sync(0xffffffffu, w, 0) == 0) break;
                if (backoff) __nanosleep(backoff);
                backoff = min(2u * backoff + 32u, async_max_backoff);
                continue;
            }
            int won = 0;
            if (lane == 0) won = atomicCAS(&s_head, h, h + k) == h;
            if (!__shfl_sync(0xffffffffu, won, 0)) continue;  // another warp took them
            backoff = 0;
            batches++;
            int32_t v = (int)lane < k ? sv : -1;
            if (v >= 0) myring[h + lane] = -1;  // the slot is reused next phase
            if constexpr (kD >= kEll2) {
                // shortcut rows (kD slots each): a batch of k rows is up to
                // kD rounds of 32 slots, so the rounds' atomicMins are all
                // issued before any push, and the near winners of every
                // round are pushed together from a per-warp shared list --
                // one tail round trip per batch instead of one per round
                __shared__ int32_t s_near[async_bound(kD) / 32][kNearList];
                int32_t *nl = s_near[threadIdx.x >> 5];
                const int nslot = k * kD;
                const int nrounds = (nslot + 31) >> 5;
                unsigned long long tok = 0;
                if (lane == 0)  // the batch's slot bound, raised while the rows load
                    tok = atomicAdd(reinterpret_cast<unsigned long long *>(&A->work),
                                    (unsigned long long)nslot);
                // the rows' slots need only the popped ids: all rounds' loads
                // are issued before the dequeue atomics, which they overlap
                int2 s[kD];
                unsigned long long old[kD];
#pragma unroll
                for (int r = 0; r < kD; r++) {
                    s[r] = make_int2(-1, 0);
                    if (r >= nrounds) continue;  // warp-uniform
                    const int pp = r * 32 + (int)lane;
                    const int32_t vj = __shfl_sync(0xffffffffu, v, (pp / kD) & 31);
                    if (pp < nslot && vj >= 0) s[r] = __ldg(ell + (size_t)vj * kD + (pp % kD));
                }
                int dv = 0;
                bool act = false;
                if (v >= 0) {
                    const int lst = __ldcg(last + v);
                    dv = (int)(atomicAnd(dq + v, ~1ull) >> 1);
                    act = dv < lst;
                    if (act) {
                        last[v] = dv;
                        expanded++;
                    }
                }
#pragma unroll
                for (int r = 0; r < kD; r++) {
                    old[r] = ~0ull;
                    if (r >= nrounds) continue;  // warp-uniform
                    const int vl = ((r * 32 + (int)lane) / kD) & 31;
                    const int du = __shfl_sync(0xffffffffu, dv, vl);
                    const bool aj = __shfl_sync(0xffffffffu, act, vl);
                    if (!aj) s[r].x = -1;
                    const bool live = s[r].x >= 0;
                    const unsigned rm = __ballot_sync(0xffffffffu, live);
                    if (lane == 0) relaxed += __popc(rm);
                    if (live) {
                        const int64_t cd = (int64_t)du + (int64_t)s[r].y;
                        if (cd < (int64_t)kIntMax)
                            old[r] = atomicMin(dq + s[r].x, ((unsigned long long)cd << 1) |
                                                                (cd < T ? 1ull : 0ull));
                        else
                            s[r].x = -1;  // never wins (F12)
                    }
                }
                int nn = 0;  // near winners collected in nl
                long long pushed = 0;
#pragma unroll
                for (int r = 0; r < kD; r++) {
                    if (r >= nrounds) break;
                    const int vl = ((r * 32 + (int)lane) / kD) & 31;
                    const int64_t cd = (int64_t)__shfl_sync(0xffffffffu, dv, vl) + (int64_t)s[r].y;
                    const bool fin = s[r].x >= 0;
                    const bool won = fin && (long long)(old[r] >> 1) > cd;
                    const bool nb = cd < T;
                    const bool near = won && nb && (old[r] & 1ull) == 0;
                    const unsigned m = __ballot_sync(0xffffffffu, near);
                    if (m) {
                        if (nn + __popc(m) > kNearList) {  // rare: flush the list
                            pushed += async_push_list(A, nl, nn, lane, tok);
                            nn = 0;
                        }
                        if (near) nl[nn + __popc(m & ((1u << lane) - 1u))] = s[r].x;
                        nn += __popc(m);
                    }
                    async_push_far(A, fc, won && !nb, s[r].x, lane);
                }
                pushed += async_push_list(A, nl, nn, lane, tok);
                __syncwarp();
                if (lane == 0)
                    atomicAdd(reinterpret_cast<unsigned long long *>(&A->work),
                              (unsigned long long)(-(long long)(k + nslot - pushed)));
                continue;
            } else if constexpr (kD > 0) {
                // slot p of the batch (vertex p / kD, its slot p % kD) goes
                // to lane p % 32 in round p / 32: the slot loads need only
                // the popped ids, so they are issued before the dequeue
                // atomics return, and a batch's relaxations share one push
                // round per 32 slots (as the CSR path's flattening does)
                constexpr int kLog = kD == 2 ? 1 : kD == 4 ? 2 : 3;
                const int nslot = k * kD;
                int2 s[kD];
#pragma unroll
                for (int r = 0; r < kD; r++) {
                    const int pp = r * 32 + (int)lane;
                    const int32_t vj = __shfl_sync(0xffffffffu, v, (pp >> kLog) & 31);
                    s[r] = pp < nslot && vj >= 0 ? __ldg(ell + (size_t)vj * kD + (pp & (kD - 1)))
                                                 : make_int2(-1, 0);
                }
                int dv = 0;
                bool act = false;
                if (v >= 0) {
                    const int lst = __ldcg(last + v);
                    dv = (int)(atomicAnd(dq + v, ~1ull) >> 1);
                    act = dv < lst;  // not yet expanded at this distance
                    if (act) {
                        last[v] = dv;
                        expanded++;
                    }
                }
                const int64_t total = (int64_t)__popc(__ballot_sync(0xffffffffu, act)) * kD;
                unsigned long long tok = 0;
                if (lane == 0 && total)
                    tok = atomicAdd(reinterpret_cast<unsigned long long *>(&A->work),
                                    (unsigned long long)total);
                long long pushed = 0;
#pragma unroll
                for (int r = 0; r < kD; r++) {
                    if (r * 32 >= nslot) break;  // warp-uniform
                    const int pp = r * 32 + (int)lane;
                    const int du = __shfl_sync(0xffffffffu, dv, (pp >> kLog) & 31);
                    const bool aj = __shfl_sync(0xffffffffu, act, (pp >> kLog) & 31);
                    const bool live = pp < nslot && aj && s[r].x >= 0;
                    const unsigned rm = __ballot_sync(0xffffffffu, live);
                    if (lane == 0) relaxed += __popc(rm);
                    bool near = false, far = false;
                    const int64_t cand = (int64_t)du + (int64_t)s[r].y;
                    if (live && cand < (int64_t)kIntMax) {
                        const bool nb = cand < T;
                        const unsigned long long old = atomicMin(
                            dq + s[r].x, ((unsigned long long)cand << 1) | (nb ? 1ull : 0ull));
                        if ((long long)(old >> 1) > cand) {
                            if (nb) near = (old & 1ull) == 0;
                            else far = true;
                        }
                    }
                    pushed += async_push_near(A, near, s[r].x, lane, true, tok);
                    async_push_far(A, fc, far, s[r].x, lane);
                }
                __syncwarp();
                if (lane == 0)
                    atomicAdd(reinterpret_cast<unsigned long long *>(&A->work),
                              (unsigned long long)(-(long long)(k + total - pushed)));
                continue;
            }
            int dv = 0;
            int64_t beg = 0, deg = 0;
            if (v >= 0) {
                // row bounds and last[v] overlap the exchange
                beg = off[v];
                const int64_t end = off[v + 1];
                const int lst = __ldcg(last + v);
                // clear the queued bit; the distance to expand with is the
                // value at that moment (any later improvement re-queues v)
                dv = (int)(atomicAnd(dq + v, ~1ull) >> 1);
                if (dv < lst) {  // not yet expanded at this distance
                    last[v] = dv;
                    deg = end - beg;
                    expanded++;
                }
            }
            int64_t incl = deg;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)lane >= o) incl += t;
            }
            const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
            const int64_t excl = incl - deg;
            // every slot may push one entry: count them all now (the atomic
            // overlaps the slot loads), return the surplus at the end
            unsigned long long tok = 0;
            if (lane == 0) {
                relaxed += total;
                if (total)
                    tok = atomicAdd(reinterpret_cast<unsigned long long *>(&A->work),
                                    (unsigned long long)total);
            }
            long long pushed = 0;
            for (int64_t p0 = 0; p0 < total; p0 += 32) {
                const int64_t p = p0 + lane;
                int lo = 0;  // owner lane: largest with excl <= p
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int cand = lo + step;
                    const int64_t ex = __shfl_sync(0xffffffffu, excl, cand & 31);
                    if (cand < 32 && ex <= p) lo = cand;
                }
                const int64_t ex = __shfl_sync(0xffffffffu, excl, lo);
                const int64_t b0 = __shfl_sync(0xffffffffu, beg, lo);
                const int du = __shfl_sync(0xffffffffu, dv, lo);
                bool near = false, far = false;
                int32_t x = -1;
                if (p < total) {
                    const int64_t e = b0 + (p - ex);
                    x = __ldg(adj + e);
                    const int64_t cand = (int64_t)du + (int64_t)__ldg(weff + e);
                    if (cand < (int64_t)kIntMax) {
                        // one atomic lowers dist and marks x queued (near) --
                        // no pre-read of dist[x]: one round trip less per hop
                        const bool nb = cand < T;
                        const unsigned long long old =
                            atomicMin(dq + x, ((unsigned long long)cand << 1) | (nb ? 1ull : 0ull));
                        if ((long long)(old >> 1) > cand) {
                            if (nb) near = (old & 1ull) == 0;
                            else far = true;
                        }
                    }
                }
                pushed += async_push_near(A, near, x, lane, true, tok);
                async_push_far(A, fc, far, x, lane);
            }
            __syncwarp();
            if (lane == 0)  // expanded: the batch's k entries and the unused slot counts
                atomicAdd(reinterpret_cast<unsigned long long *>(&A->work),
                          (unsigned long long)(-(long long)(k + total - pushed)));
        }
        const long long t_drained = clock64();
        grid.sync();
        if (threadIdx.x == 0) {  // drained: every ring restarts at slot 0
            s_head = 0;
            A->tails[(size_t)blockIdx.x * kTailStride] = 0;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {  // next T
            const int src = A->fcur;
            const unsigned long long nf = A->far_n[src];
            int go = 1;
            A->phases++;
            A->far_scanned += nf;
            if (A->abort) {
                go = 0;
            } else if (nf > A->fcap) {
                A->status = 3;
                go = 0;
            } else if (nf == 0) {
                go = 0;
            } else {
                A->T += A->delta;
                A->fcur = src ^ 1;
                A->far_n[src ^ 1] = 0;
            }
            A->go = go;
        }
        grid.sync();
        if (!VA->go) break;
        {   // split the old pile: below the new T and dropped since the last
            // expansion -> rings (queued bit set here); the rest -> the new pile
            const int nfc = VA->fcur, src = nfc ^ 1;
            const int64_t T2 = VA->T;
            const int64_t nf = (int64_t)VA->far_n[src];
            const int32_t *pile = A->far[src];
            const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
            const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
            for (int64_t b = wid * 32; b < nf; b += nw * 32) {
                const int64_t i = b + lane;
                bool near = false, far = false;
                int32_t x = -1;
                if (i < nf) {
                    x = pile[i];
                    const int d = (int)(__ldcg(dq + x) >> 1);
                    if ((int64_t)d < T2) {
                        near = d < __ldcg(last + x) && (atomicOr(dq + x, 1ull) & 1ull) == 0;
                    } else {
                        far = true;
                    }
                }
                async_push_near(A, near, x, lane, false);
                async_push_far(A, nfc, far, x, lane);
            }
        }
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0)
            A->between_cycles += (unsigned long long)(clock64() - t_drained);
    }
    relaxed = warp_sum(relaxed);
    expanded = warp_sum(expanded);
    if (lane == 0) {
        if (relaxed) atomicAdd(&A->relaxed, relaxed);
        if (expanded) atomicAdd(&A->expanded, expanded);
        if (batches) atomicAdd(&A->batches, batches);
    }
}

__global__ void k_async_init(unsigned long long *dq, int32_t *ring, unsigned long long *tails,
                             int64_t n, int64_t ring_total, int nring, int32_t src, int src_ring,
                             unsigned long long cap) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x)
        dq[x] = x == src ? 1ull : ((unsigned long long)kIntMax << 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ring_total;
         i += (int64_t)gridDim.x * blockDim.x)
        ring[i] = i == (int64_t)src_ring * (int64_t)cap ? src : -1;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nring;
         r += (int64_t)gridDim.x * blockDim.x)
        tails[r * kTailStride] = r == src_ring ? 1 : 0;
}

__global__ void k_async_out(const unsigned long long *__restrict__ dq, int32_t *dist, int64_t n) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x)
        dist[x] = (int32_t)(dq[x] >> 1);
}

// The asynchronous near-far loop; SP_OK with out->status 3 asks the caller
// for another form (ring or far-pile overflow, or the watchdog).
int sssp_near_far_async(sp_graph *g, Call &c, int32_t *dist, int32_t src, int64_t delta,
                        SsspLoop *out, float *kernel_ms) {
    const int64_t n = g->n, m = g->m;
    const int sms = num_sms(c.device);
    const char *thr = getenv("SP_NF_ASYNC_THREADS");  // threads per block (sweeps)
    int threads = thr ? std::max(32, std::min(kAsyncBlock, atoi(thr) / 32 * 32))
                      : kAsyncThreads;
    // bounded-degree graphs: the ELL row form (SP_NF_ELL=0: CSR rows)
    const char *ee = getenv("SP_NF_ELL");
    if (!(ee && ee[0] == '0')) SP_TRY(ensure_ell(g, c, kEllMaxDeg));
    // 2-hop shortcut rows on graphs of out-degree <= 4 (SP_NF_SHORTCUT=0: off)
    // (SP_NF_SHORTCUT=3: 1- to 3-hop rows of 32 slots)
    const char *se = getenv("SP_NF_SHORTCUT");
    const bool shortcut = !(ee && ee[0] == '0') && !(se && se[0] == '0') && g->ell &&
                          g->ell_d <= 4;
    const int hops = se && se[0] == '3' ? 3 : 2;
    if (shortcut) SP_TRY(ensure_ell2(g, c, hops));
    // 2-hop rows: 320 threads per block (cfg5a, 12-slot rows, 256 / 320 /
    // 384 / 448: 27.4 / 26.9 / 27.5 / 28.9 ms; two blocks per SM: slower)
    if (!thr && shortcut && g->ell2 && g->ell2_slots == kEll2) threads = 320;
    const bool use2 = shortcut && g->ell2 &&
                      threads <= (g->ell2_slots == kEll3 ? 256 : 512);  // its launch bound
    // a shortcut row covers two hops: a phase may span a wider distance
    // band (cfg5a, 16-slot rows, delta 816 / 1632 / 2400 / 3200: 34.3 / 31.2
    // / 31.4 / 32.1 ms; 12-slot rows at 384 threads, 1632 / 2400: 27.4 /
    // 26.7 ms; 1-hop rows: 39.5 ms at 816, 39.0 at 1632)
    if (use2 && !getenv("SP_SSSP_DELTA")) delta *= 3;
    const void *kfn = use2 && g->ell2_slots == kEll3 ? (const void *)k_nf_async<kEll3>
                      : use2          ? (const void *)k_nf_async<kEll2>
                      : g->ell_d == 2 ? (const void *)k_nf_async<2>
                      : g->ell_d == 4 ? (const void *)k_nf_async<4>
                      : g->ell_d == 8 ? (const void *)k_nf_async<8>
                                      : (const void *)k_nf_async<0>;
    int per_sm = 0;  // co-residency of the cooperative launch: this kernel's own
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, threads, 0);
    const char *bps = getenv("SP_NF_ASYNC_BPS");  // blocks per SM (sweeps)
    const int want = bps ? std::max(1, atoi(bps)) : kAsyncBlocksPerSm;
    const int nring = sms * std::max(1, std::min(per_sm, want));  // one ring per block
    const char *bo = getenv("SP_NF_ASYNC_BACKOFF");   // max idle backoff, ns (sweeps)
    unsigned max_backoff = bo ? (unsigned)atoi(bo) : kAsyncBackoff;
    // a ring restarts every phase; a phase pushes each vertex at most once
    // per drop below T, so its owned share (x 2, + slack) bounds it in
    // practice -- an overflow aborts to the synchronous kernel
    const int64_t chunks = (n + (1 << kOwnShift) - 1) >> kOwnShift;
    const int64_t owned = ((chunks + nring - 1) / nring) << kOwnShift;
    const char *ce = getenv("SP_NF_ASYNC_RING");  // ring capacity (tests: force overflows)
    unsigned long long cap = ce ? (unsigned long long)atoll(ce) : 0;
    if (!cap) {
        cap = 1;
        while (cap < (unsigned long long)(2 * owned + 4096)) cap <<= 1;
    }
    const int64_t fcap = 2 * m + n + 16;
    int32_t *last, *fa, *fb, *ring;
    unsigned long long *tails, *dq;
    AsyncNf *A;
    SP_TRY(c.alloc(&dq, n));
    SP_TRY(c.alloc(&last, n));
    SP_TRY(c.alloc(&fa, fcap));
    SP_TRY(c.alloc(&fb, fcap));
    SP_TRY(c.alloc(&ring, cap * nring));
    SP_TRY(c.alloc(&tails, (size_t)nring * kTailStride));
    SP_TRY(c.alloc(&A, 1));
    k_fill_i32<<<grid_for(n, kBlock, c.device), kBlock, 0, c.stream>>>(last, n, kIntMax);
    const int src_ring = (int)(((uint32_t)src >> kOwnShift) % (uint32_t)nring);
    k_async_init<<<grid_for((int64_t)(cap * nring), kBlock, c.device), kBlock, 0, c.stream>>>(
        dq, ring, tails, n, (int64_t)(cap * nring), nring, src, src_ring, cap);
    c.launches += 2;
    AsyncNf init{};
    init.ring = ring;
    init.tails = tails;
    init.cap = cap;
    init.nring = nring;
    init.work = 1;  // the source
    init.far[0] = fa;
    init.far[1] = fb;
    init.fcap = (unsigned long long)fcap;
    init.T = delta;
    init.delta = delta;
    SP_CUDA(cudaMemcpyAsync(A, &init, sizeof(AsyncNf), cudaMemcpyHostToDevice, c.stream));
    const int2 *ell = use2 ? g->ell2 : g->ell;
    void *kargs[] = {&dq, &last, (void *)&g->weff, (void *)&g->off, (void *)&g->adj, (void *)&ell,
                     &A, &max_backoff};
    cudaEvent_t ka, kb;
    SP_CUDA(cudaEventCreate(&ka));
    SP_CUDA(cudaEventCreate(&kb));
    cudaEventRecord(ka, c.stream);
    SP_CUDA(cudaLaunchCooperativeKernel(kfn, nring, threads, kargs, 0, c.stream));
    k_async_out<<<grid_for(n, kBlock, c.device), kBlock, 0, c.stream>>>(dq, dist, n);
    cudaEventRecord(kb, c.stream);
    c.launches += 2;
    AsyncNf *hA;
    SP_TRY(c.host_as(&hA));
    SP_CUDA(cudaMemcpyAsync(hA, A, sizeof(AsyncNf), cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    cudaEventElapsedTime(kernel_ms, ka, kb);
    cudaEventDestroy(ka);
    cudaEventDestroy(kb);
    if (hA->status == 4)
        fprintf(stderr, "starplat_b200: asynchronous near-far SSSP hit its watchdog; "
                        "falling back to the synchronous form\n");
    static const bool trace = getenv("SP_SSSP_TRACE") != nullptr;
    if (trace)
        fprintf(stderr, "sssp async: %d blocks x %d threads, ring %llu, %lld phases, %llu "
                        "batches, %llu expansions, %llu relaxations, status %d, %.2f ms; far "
                        "entries split %llu, between-phase cycles (block 0) %llu\n",
                nring, threads, cap, (long long)hA->phases, hA->batches, hA->expanded,
                hA->relaxed, hA->status, *kernel_ms, hA->far_scanned, hA->between_cycles);
    out->iters = hA->phases;
    out->relaxed = (int64_t)hA->relaxed;
    out->frontier_sum = (int64_t)hA->expanded;
    out->status = hA->status == 0 ? 0 : 3;
    return SP_OK;
}

int sssp_near_far(sp_graph *g, Call &c, int32_t *dist, int32_t *enq, int32_t *qa, int32_t *qb,
                  ChunkItem *chunks, int64_t cap, int64_t delta, SsspLoop *out, float *kernel_ms) {
    const int64_t n = g->n, m = g->m;
    int32_t *last, *fa, *fb;
    NfLoop *L;
    SP_TRY(c.alloc(&last, n));
    // far piles: every entry is an improvement above T; bounded by the
    // relaxations of one iteration plus the surviving pile (<= 2m + n)
    const int64_t fcap = 2 * m + n + 16;
    SP_TRY(c.alloc(&fa, fcap));
    SP_TRY(c.alloc(&fb, fcap));
    SP_TRY(c.alloc(&L, 1));
    k_fill_i32<<<grid_for(n, kBlock, c.device), kBlock, 0, c.stream>>>(last, n, kIntMax);
    c.launches++;
    NfLoop init{};
    init.q[0] = qa;
    init.q[1] = qb;
    init.far[0] = fa;
    init.far[1] = fb;
    init.nq = 1;
    init.it = 1;
    init.T = delta;
    init.delta = delta;
    init.cap = cap;
    init.fcap = (unsigned long long)fcap;
    SP_CUDA(cudaMemcpyAsync(L, &init, sizeof(NfLoop), cudaMemcpyHostToDevice, c.stream));
    const int sms = num_sms(c.device);
    if (g->max_outdeg <= kSplit) {  // thin graph: one persistent cooperative launch
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_nf_persistent, kExpandBlock, 0);
        const int pgrid = sms * std::max(1, std::min(per_sm, kPersistBlocksPerSm));
        void *kargs[] = {&dist, &enq, &last, (void *)&g->weff, (void *)&g->off,
                         (void *)&g->adj, &L};
        cudaEvent_t ka, kb;
        SP_CUDA(cudaEventCreate(&ka));
        SP_CUDA(cudaEventCreate(&kb));
        cudaEventRecord(ka, c.stream);
        SP_CUDA(cudaLaunchCooperativeKernel((const void *)k_nf_persistent, pgrid, kExpandBlock,
                                            kargs, 0, c.stream));
        cudaEventRecord(kb, c.stream);
        NfLoop *hL;
        SP_TRY(c.host_as(&hL));
        SP_CUDA(cudaMemcpyAsync(hL, L, sizeof(NfLoop), cudaMemcpyDeviceToHost, c.stream));
        SP_CUDA(cudaStreamSynchronize(c.stream));
        cudaEventElapsedTime(kernel_ms, ka, kb);
        cudaEventDestroy(ka);
        cudaEventDestroy(kb);
        out->iters = hL->iters;
        out->relaxed = hL->relaxed;
        out->frontier_sum = hL->frontier_sum;
        out->status = hL->status;
        c.launches += 1;
        return SP_OK;
    }
    // near-far frontiers are small (a band of the graph): a smaller grid
    // keeps the fixed per-iteration launch cost down
    const int grid = sms * 2;
    const int64_t warps = (int64_t)grid * (kExpandBlock / 32);
    const bool big = g->max_outdeg > kSplit;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    struct GraphFree {
        cudaGraph_t *g;
        cudaGraphExec_t *e;
        ~GraphFree() {
            if (*e) cudaGraphExecDestroy(*e);
            if (*g) cudaGraphDestroy(*g);
        }
    } gf{&graph, &exec};
    SP_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h;
    SP_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    SP_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    SP_CUDA(cudaStreamBeginCaptureToGraph(c.stream, body, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
    k_nf_expand<<<grid, kExpandBlock, 0, c.stream>>>(dist, enq, last, g->weff, g->off, g->adj,
                                                     chunks, L, warps);
    if (big)
        k_nf_chunks<<<grid, kExpandBlock, 0, c.stream>>>(dist, enq, last, g->weff, g->off, g->adj,
                                                         chunks, L);
    k_nf_split<<<grid, kBlock, 0, c.stream>>>(dist, enq, last, L);
    k_nf_advance2<<<1, 1, 0, c.stream>>>(L, h);
    SP_CUDA(cudaStreamEndCapture(c.stream, &body));
    cudaEvent_t ka, kb;
    SP_CUDA(cudaEventCreate(&ka));
    SP_CUDA(cudaEventCreate(&kb));
    cudaEventRecord(ka, c.stream);
    SP_TRY(launch_cached_graph(graph, g, kLoopSsspNf, c.stream));
    cudaEventRecord(kb, c.stream);
    NfLoop *hL;
    SP_TRY(c.host_as(&hL));
    SP_CUDA(cudaMemcpyAsync(hL, L, sizeof(NfLoop), cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    cudaEventElapsedTime(kernel_ms, ka, kb);
    cudaEventDestroy(ka);
    cudaEventDestroy(kb);
    out->iters = hL->iters;
    out->relaxed = hL->relaxed;
    out->frontier_sum = hL->frontier_sum;
    out->status = hL->status;
    c.launches += hL->iters * (big ? 4 : 3);
    return SP_OK;
}

// ---- direction-optimising loop (push / pull), low-diameter graphs -------
// sssp_pull.sp's form of the relaxation: every vertex v takes the minimum
// of dist[u] + w_eff(u -> v) over its in-neighbours u in the frontier (a
// bitmap), an exact min in any order, one write per improved vertex, no
// atomics on dist.  Large frontiers run pull steps, small ones push steps
// (Beamer's direction optimisation); both converge to the same fixpoint.
struct DoLoop {
    SsspLoop s;            // push-side state (queues, counters, totals)
    uint32_t *bitsF;       // frontier bitmap (pull input)
    uint32_t *bitsN;       // next-frontier bitmap (pull output, zeroed)
    int32_t *hubs;         // in-rows longer than kPullHub of this pull step
    unsigned long long nhubs;
    int64_t nwords, n;
    int64_t pull_div;      // pull when the frontier exceeds n / pull_div
    int mode;              // 0 push, 1 pull (this iteration)
    int next_mode;
    int conv;              // after advance: 1 queue->bits, 2 bits->queue
    int go;                // the advance's loop decision (host-driven diagnostic loop)
};

constexpr int kPullChunk = 128;
constexpr int64_t kPullHub = 1024;
constexpr int64_t kPullDiv = 8;   // pull when the frontier exceeds n / kPullDiv (4-12 measured alike);
// a test on the frontier's out-slots (pull iteration 2 on RMAT-24, whose
// 0.24 M hub neighbours hold ~140 M out-slots) measured slower: 5.25 -> 9.4 ms,
// the earlier pull leaves larger frontiers and two more sweeps
// Push-form SSSP uses the direction-optimising loop on graphs this large
// (RMAT-24: 5.95 -> 5.55 ms; at RMAT-22 the two loops tie, at cfg1 the
// extra per-iteration kernels cost more than the pull saves)
constexpr int64_t kDoMinSlots = int64_t(1) << 27;

__device__ __forceinline__ bool fbit(const uint32_t *b, int32_t u) {
    return (__ldcg(b + (u >> 5)) >> (u & 31)) & 1u;
}

// Apply a row's minimum: improve dist[v], mark v in the next bitmap, count.
__device__ __forceinline__ bool pull_apply(DoLoop *L, int32_t *dist, int64_t v, int64_t best) {
    if (best >= (int64_t)kIntMax || best >= (int64_t)__ldcg(dist + v)) return false;
    if (best < (int64_t)(-2147483647 - 1)) {
        atomicAdd(&L->s.cnt[L->s.cur].flag, 1ull);
        return false;
    }
    dist[v] = (int32_t)best;
    atomicOr(L->bitsN + (v >> 5), 1u << (v & 31));
    return true;
}

__global__ void __launch_bounds__(256) k_pull_tiles(const int64_t *__restrict__ roff,
                                                    const int32_t *__restrict__ radj,
                                                    const int32_t *__restrict__ rw, int32_t *dist,
                                                    DoLoop *L) {
    if (L->mode != 1) return;
    __shared__ int32_t stage[8][kPullChunk];
    const unsigned lane = lane_id();
    int32_t *buf = stage[threadIdx.x >> 5];
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t n = L->n;
    const uint32_t *F = L->bitsF;
    unsigned long long useful = 0, improved = 0;
    for (int64_t t0 = warp * 32; t0 < n; t0 += nwarps * 32) {
        const int64_t v = t0 + lane;
        int64_t rs = 0, deg = 0;
        if (v < n) {
            rs = roff[v];
            deg = roff[v + 1] - rs;
        }
        const bool hub = deg > kPullHub;
        {
            const int64_t slot = warp_append(hub, &L->nhubs);
            if (hub) L->hubs[slot] = (int32_t)v;
        }
        if (hub) deg = 0;
        int64_t incl = deg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += t;
        }
        const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
        const int64_t excl = incl - deg;
        int64_t best = INT64_MAX;
        for (int64_t p0 = 0; p0 < total; p0 += kPullChunk) {
#pragma unroll
            for (int j = 0; j < kPullChunk / 32; j++) {
                const int64_t p = p0 + j * 32 + lane;
                int lo = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int cand = lo + step;
                    const int64_t ex = __shfl_sync(0xffffffffu, excl, cand & 31);
                    if (cand < 32 && ex <= p) lo = cand;
                }
                const int64_t ex = __shfl_sync(0xffffffffu, excl, lo);
                const int64_t b0 = __shfl_sync(0xffffffffu, rs, lo);
                int32_t c = kIntMax;
                if (p < total) {
                    const int64_t k = b0 + (p - ex);
                    const int32_t u = __ldcs(radj + k);
                    if (fbit(F, u)) {
                        useful++;
                        const int64_t cand = (int64_t)__ldcg(dist + u) + (int64_t)__ldcs(rw + k);
                        c = cand >= (int64_t)kIntMax ? kIntMax
                            : (cand < (int64_t)(-2147483647 - 1) ? (int32_t)(-2147483647 - 1)
                                                                 : (int32_t)cand);
                    }
                }
                buf[j * 32 + lane] = c;
            }
            __syncwarp();
            const int64_t a = max(excl, p0), b = min(excl + deg, p0 + (int64_t)kPullChunk);
            for (int64_t p = a; p < b; p++) best = min(best, (int64_t)buf[p - p0]);
            __syncwarp();
        }
        if (v < n && !hub && deg > 0) improved += pull_apply(L, dist, v, best) ? 1 : 0;
    }
    useful = warp_sum(useful);
    improved = warp_sum(improved);
    if (lane == 0) {
        if (useful) atomicAdd(&L->s.cnt[L->s.cur].scanned, useful);
        if (improved) atomicAdd(&L->s.cnt[L->s.cur].next_size, improved);
    }
}

// In-rows longer than kPullHub: one warp per row, strided slots, warp min.
__global__ void __launch_bounds__(256) k_pull_hubs(const int64_t *__restrict__ roff,
                                                   const int32_t *__restrict__ radj,
                                                   const int32_t *__restrict__ rw, int32_t *dist,
                                                   DoLoop *L) {
    if (L->mode != 1) return;
    const unsigned lane = lane_id();
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nh = (int64_t)__ldcg(&L->nhubs);
    const uint32_t *F = L->bitsF;
    unsigned long long useful = 0, improved = 0;
    for (int64_t h = warp; h < nh; h += nwarps) {
        const int32_t v = L->hubs[h];
        const int64_t r0 = roff[v], r1 = roff[v + 1];
        int64_t best = INT64_MAX;
        for (int64_t k = r0 + lane; k < r1; k += 32) {
            const int32_t u = __ldcs(radj + k);
            if (fbit(F, u)) {
                useful++;
                best = min(best, (int64_t)__ldcg(dist + u) + (int64_t)__ldcs(rw + k));
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) improved += pull_apply(L, dist, v, best) ? 1 : 0;
    }
    useful = warp_sum(useful);
    if (lane == 0) {
        if (useful) atomicAdd(&L->s.cnt[L->s.cur].scanned, useful);
        if (improved) atomicAdd(&L->s.cnt[L->s.cur].next_size, improved);
    }
}

// ---- edge-balanced pull step (the PageRank-units layout, min-plus) ------
// The reverse slots are cut into kSpUnit-slot units, one warp per unit,
// 8 consecutive slots per lane per 256-slot chunk (radj and w_eff streamed
// with 128-bit loads, 8 independent dist gathers); row ends inside a chunk
// come from a window of nzend marked in a shared bitmap, and a segmented
// warp min-scan carries the open row's minimum across lanes and chunks.
// Rows that end in their unit are applied there; a row that began in an
// earlier unit is finished by k_spull_fix from the units' tail/head minima.
// Every in-neighbour is relaxed (a full Bellman-Ford sweep of the rows):
// no frontier test per slot, the same fixpoint.
constexpr int64_t kSpUnit = 2048;
constexpr int kSpCh = 256;
constexpr int64_t kSpNone = INT64_MAX;

struct SPull {
    const int32_t *__restrict__ radj;
    const int32_t *__restrict__ rw;
    const int64_t *__restrict__ nzend;
    const int32_t *__restrict__ nzrow;
    const int64_t *__restrict__ unit_row;
    int64_t *hp, *tp;
    int64_t m, nnz, nunits;
};

__device__ __forceinline__ void sp_slab8(const int32_t *__restrict__ p, int64_t q, int64_t s1,
                                         int (&x)[8], int fill) {
    if (q + 8 <= s1 && (q & 3) == 0) {
        const int4 a = __ldcs(reinterpret_cast<const int4 *>(p + q));
        const int4 b = __ldcs(reinterpret_cast<const int4 *>(p + q + 4));
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
        x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    } else {
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = q + i < s1 ? __ldcs(p + q + i) : fill;
    }
}

#ifndef SP_SPULL_MINB
// blocks/SM the pull sweep is compiled for (a register cap: 64 -> 48, a few
// bytes of spill): RMAT-24 SSSP 5.63 -> 5.18 ms and RMAT-26 25.1 -> 20.4 ms
// together with SP_DOCHUNK_MINB 4 (6 blocks: slower)
#define SP_SPULL_MINB 5
#endif
// kHot: slots whose source is one of the H hottest (most gathered) sources
// carry kPrHotBit | hot index (the PageRank hot encoding of radj, shared
// with sp_pagerank.cu), and their dist comes from a shared-memory snapshot
// taken when the sweep starts.  A hot source lowered during the sweep is in
// the next frontier (pull_apply marks it), so a stale snapshot value only
// defers its relaxation to the next iteration: the same fixpoint.
template <bool kHot>
__device__ __forceinline__ void spull_body(const SPull &a, int32_t *dist, DoLoop *L, uint32_t *bm,
                                           const int32_t *hot) {
    const unsigned lane = lane_id();
    if (lane < kSpCh / 32) bm[lane] = 0u;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long improved = 0, swept = 0;
    for (int64_t u = warp; u < a.nunits; u += nwarps) {
        const int64_t s0 = u * kSpUnit, s1 = min(a.m, s0 + kSpUnit);
        int64_t rk = a.unit_row[u];
        const int64_t first_row = rk;
        const bool head_spill = (rk > 0 ? __ldg(a.nzend + rk - 1) : 0) < s0;
        int64_t carry = kSpNone;
        for (int64_t c = s0; c < s1; c += kSpCh) {
            const int64_t lim = min(c + (int64_t)kSpCh, s1);
            int idx[8], w[8];
            const int64_t q = c + 8 * (int64_t)lane;
            sp_slab8(a.radj, q, lim, idx, -1);
            sp_slab8(a.rw, q, lim, w, 0);
            __syncwarp();
            const int64_t rk_chunk = rk;
            for (;;) {
                const int64_t k = rk + lane;
                const int64_t e = k < a.nnz ? __ldg(a.nzend + k) : INT64_MAX;
                const bool in = e <= lim;
                if (in) {
                    const int bb = (int)(e - 1 - c);
                    atomicOr(&bm[bb >> 5], 1u << (bb & 31));
                }
                const int cnt = __popc(__ballot_sync(0xffffffffu, in));
                rk += cnt;
                if (cnt < 32) break;
            }
            int64_t val[8];
#pragma unroll
            for (int i = 0; i < 8; i++) {
                val[i] = kSpNone;
                if (idx[i] >= 0) {
                    int du;
                    if constexpr (kHot)
                        du = (idx[i] & kPrHotBit) ? hot[idx[i] & (kPrHotBit - 1)]
                                                  : __ldcg(dist + idx[i]);
                    else
                        du = __ldcg(dist + idx[i]);
                    if (du != kIntMax) val[i] = (int64_t)du + (int64_t)w[i];
                }
            }
            __syncwarp();
            const unsigned ends = (bm[lane >> 2] >> ((lane & 3) * 8)) & 0xFFu;
            __syncwarp();
            if (lane < kSpCh / 32) bm[lane] = 0u;
            int64_t tail = kSpNone;
#pragma unroll
            for (int i = 0; i < 8; i++) {
                tail = min(tail, val[i]);
                if ((ends >> i) & 1u) tail = kSpNone;
            }
            bool f = ends != 0u;
            int64_t v = tail;
            int ne = __popc(ends);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const bool fo = __shfl_up_sync(0xffffffffu, f, o);
                const int64_t vo = __shfl_up_sync(0xffffffffu, v, o);
                const int no = __shfl_up_sync(0xffffffffu, ne, o);
                if ((int)lane >= o) {
                    if (!f) v = min(vo, v);
                    f = f || fo;
                    ne += no;
                }
            }
            bool fe = __shfl_up_sync(0xffffffffu, f, 1);
            int64_t ve = __shfl_up_sync(0xffffffffu, v, 1);
            int nbefore = __shfl_up_sync(0xffffffffu, ne, 1);
            if (lane == 0) {
                fe = false;
                ve = kSpNone;
                nbefore = 0;
            }
            const int64_t carry_in = fe ? ve : min(carry, ve);
            const bool f31 = __shfl_sync(0xffffffffu, f, 31);
            const int64_t v31 = __shfl_sync(0xffffffffu, v, 31);
            carry = f31 ? v31 : min(carry, v31);
            if (ends) {
                int64_t run = kSpNone;
                int j = 0;
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    run = min(run, val[i]);
                    if ((ends >> i) & 1u) {
                        const int64_t best = j == 0 ? min(carry_in, run) : run;
                        const int64_t row = rk_chunk + nbefore + j;
                        if (head_spill && row == first_row) {
                            a.hp[u] = best;  // finished by k_spull_fix
                        } else if (best != kSpNone) {
                            improved += pull_apply(L, dist, __ldg(a.nzrow + row), best) ? 1 : 0;
                        }
                        j++;
                        run = kSpNone;
                    }
                }
            }
        }
        if (lane == 0) {
            a.tp[u] = carry;
            swept += (unsigned long long)(s1 - s0);
        }
    }
    improved = warp_sum(improved);
    if (lane == 0 && improved) atomicAdd(&L->s.cnt[L->s.cur].next_size, improved);
    // every swept in-slot is a relaxation (12 B: radj, w_eff, dist gather)
    if (lane == 0 && swept) atomicAdd(&L->s.cnt[L->s.cur].scanned, swept);
}

__global__ void __launch_bounds__(256, SP_SPULL_MINB) k_spull_units(SPull a, int32_t *dist, DoLoop *L) {
    if (L->mode != 1) return;
    __shared__ uint32_t bitmap[8][kSpCh / 32];
    spull_body<false>(a, dist, L, bitmap[threadIdx.x >> 5], nullptr);
}

// the hot sources' dist at the start of a sweep, contiguous
__global__ void k_spull_hot_gather(const DoLoop *L, const int32_t *__restrict__ hot_ids, int H,
                                   const int32_t *dist, int32_t *hotd) {
    if (L->mode != 1) return;
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x)
        hotd[h] = __ldcg(dist + hot_ids[h]);
}

// Persistent hot variant: one 1024-thread block per SM copies the snapshot
// into shared memory, then its warps sweep their units.
constexpr int kSpHotBlock = 1024;
__global__ void __launch_bounds__(kSpHotBlock, 1) k_spull_units_hot(SPull a, int32_t *dist,
                                                                   DoLoop *L,
                                                                   const int32_t *hotd, int H) {
    if (L->mode != 1) return;
    extern __shared__ int32_t sp_hot_smem[];
    uint32_t *bitmaps = reinterpret_cast<uint32_t *>(sp_hot_smem + ((H + 3) & ~3));
    const int4 *src = reinterpret_cast<const int4 *>(hotd);
    int4 *dst = reinterpret_cast<int4 *>(sp_hot_smem);
    for (int i = threadIdx.x; i < (H + 3) / 4; i += blockDim.x) dst[i] = __ldcg(src + i);
    __syncthreads();
    spull_body<true>(a, dist, L, bitmaps + (threadIdx.x >> 5) * (kSpCh / 32), sp_hot_smem);
}

// rows that began in an earlier unit and end in unit u: min of the crossed
// units' tails and u's head
__global__ void k_spull_fix(SPull a, int32_t *dist, DoLoop *L) {
    if (L->mode != 1) return;
    unsigned long long improved = 0;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < a.nunits;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t rk = a.unit_row[u];
        const int64_t s0 = u * kSpUnit, s1 = min(a.m, s0 + kSpUnit);
        const int64_t start = rk > 0 ? a.nzend[rk - 1] : 0;
        if (rk >= a.nnz || start >= s0 || a.nzend[rk] > s1) continue;
        int64_t best = a.hp[u];
        for (int64_t w = start / kSpUnit; w < u; w++) best = min(best, a.tp[w]);
        if (best != kSpNone) improved += pull_apply(L, dist, a.nzrow[rk], best) ? 1 : 0;
    }
    improved = warp_sum(improved);
    if ((threadIdx.x & 31) == 0 && improved)
        atomicAdd(&L->s.cnt[L->s.cur].next_size, improved);
}

__global__ void k_spull_setup(SPull a) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < a.nunits;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s0 = u * kSpUnit;
        int64_t lo = 0, hi = a.nnz;
        while (lo < hi) {
            const int64_t mid = lo + ((hi - lo) >> 1);
            if (a.nzend[mid] <= s0) lo = mid + 1; else hi = mid;
        }
        const_cast<int64_t *>(a.unit_row)[u] = lo;
    }
}

#ifndef SP_DOPUSH_MINB
#define SP_DOPUSH_MINB 5  // RMAT-24: 4 -> 5.16 ms, 5 -> 5.06 ms, 6 -> 5.2 ms
#endif
__global__ void __launch_bounds__(kExpandBlock, SP_DOPUSH_MINB) k_do_push(
    int32_t *dist, int32_t *enq, const int32_t *__restrict__ weff,
    const int64_t *__restrict__ off, const int32_t *__restrict__ adj, ChunkItem *chunks,
    DoLoop *D, int64_t warps) {
    if (D->mode != 0) return;
    SsspLoop *L = &D->s;
    const int cur = L->cur;
    const int64_t nq = L->nq;
    RelaxOp op{dist, enq, weff, &L->cnt[cur].flag, L->it};
    expand_body(op, off, adj, L->q[cur], nq, L->q[cur ^ 1], chunks, &L->cnt[cur],
                expand_vpw(nq, warps));
}

#ifndef SP_DOCHUNK_MINB
#define SP_DOCHUNK_MINB 4  // hub-chunk push (80 -> 64 registers; 5: slower)
#endif
__global__ void __launch_bounds__(kExpandBlock, SP_DOCHUNK_MINB) k_do_push_chunks(
    int32_t *dist, int32_t *enq, const int32_t *__restrict__ weff,
    const int64_t *__restrict__ off, const int32_t *__restrict__ adj, const ChunkItem *chunks,
    DoLoop *D) {
    if (D->mode != 0) return;
    SsspLoop *L = &D->s;
    const int cur = L->cur;
    RelaxOp op{dist, enq, weff, &L->cnt[cur].flag, L->it};
    expand_chunks_body(op, off, adj, chunks, L->q[cur ^ 1], &L->cnt[cur]);
}

// Totals, termination, and the direction of the next iteration.
__global__ void k_do_advance(DoLoop *D, cudaGraphConditionalHandle h, int set_cond) {
    SsspLoop *L = &D->s;
    const int cur = L->cur;
    const ExpandCounters c = L->cnt[cur];
    L->iters++;
    L->frontier_sum += L->nq;
    L->relaxed += (int64_t)c.scanned;
    const int64_t next = (int64_t)c.next_size;
    int go = 1;
    if (c.flag) {
        L->status = 1;
        go = 0;
    } else if (next == 0) {
        go = 0;
    } else if (L->iters >= L->cap) {
        L->status = 2;
        go = 0;
    }
    const int nm = next * D->pull_div > D->n ? 1 : 0;
    D->conv = 0;
    if (D->mode == 0 && nm == 1) D->conv = 1;  // queue -> bits
    if (D->mode == 1) {                         // the pull output becomes the frontier
        uint32_t *t = D->bitsF;
        D->bitsF = D->bitsN;
        D->bitsN = t;
        if (nm == 0) D->conv = 2;               // bits -> queue
    }
    D->next_mode = nm;
    D->nhubs = 0;
    L->cnt[cur ^ 1] = ExpandCounters{0, 0, 0, 0};
    L->cur = cur ^ 1;
    L->nq = next;
    L->it = (int)(L->iters + 1);
    D->go = go;
    if (set_cond) cudaGraphSetConditional(h, go);
}

// Zero the bitmap the next pull writes (and the frontier bitmap a
// queue -> bits conversion fills).
__global__ void k_do_clear(DoLoop *D) {
    if (D->next_mode != 1) return;
    uint32_t *N = D->bitsN, *F = D->bitsF;
    const bool clearF = D->conv == 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < D->nwords;
         i += (int64_t)gridDim.x * blockDim.x) {
        N[i] = 0u;
        if (clearF) F[i] = 0u;
    }
}

__global__ void k_do_convert(DoLoop *D) {
    SsspLoop *L = &D->s;
    const int conv = D->conv;
    if (conv == 1) {  // the queue just produced (q[cur]) -> frontier bits
        const int32_t *q = L->q[L->cur];
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L->nq;
             i += (int64_t)gridDim.x * blockDim.x) {
            const int32_t v = q[i];
            atomicOr(D->bitsF + (v >> 5), 1u << (v & 31));
        }
    } else if (conv == 2) {  // frontier bits -> queue q[cur]; nq already counted
        int32_t *q = L->q[L->cur];
        for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < D->nwords;
             b += (int64_t)gridDim.x * blockDim.x) {
            const int64_t i = b + threadIdx.x;
            const uint32_t w = i < D->nwords ? __ldcg(D->bitsF + i) : 0u;
            const int c = __popc(w);
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)lane_id() >= o) incl += t;
            }
            const int tot = __shfl_sync(0xffffffffu, incl, 31);
            unsigned long long base = 0;
            if (lane_id() == 0 && tot) base = atomicAdd(&D->s.cnt[D->s.cur].chunks, (unsigned long long)tot);
            base = __shfl_sync(0xffffffffu, base, 0);
            uint32_t x = w;
            int64_t at = (int64_t)base + incl - c;
            while (x) {
                const int bit = __ffs(x) - 1;
                x &= x - 1;
                q[at++] = (int32_t)(i * 32 + bit);
            }
        }
    }
}

__global__ void k_do_mode(DoLoop *D) {
    D->mode = D->next_mode;
    D->s.cnt[D->s.cur].chunks = 0;  // borrowed by the bits -> queue conversion
}

int sssp_do_loop(sp_graph *g, Call &c, int32_t *dist, int32_t *enq, int32_t *qa, int32_t *qb,
                 ChunkItem *chunks, int64_t cap, SsspLoop *out, float *kernel_ms) {
    SP_TRY(ensure_rweff(g, c));
    const int64_t n = g->n;
    const int64_t nwords = (n + 31) / 32;
    DoLoop *D;
    uint32_t *b0, *b1;
    int32_t *hubs;
    SP_TRY(c.alloc(&D, 1));
    SP_TRY(c.alloc(&b0, nwords));
    SP_TRY(c.alloc(&b1, nwords));
    SP_TRY(c.alloc(&hubs, n));
    DoLoop init{};
    init.s.q[0] = qa;
    init.s.q[1] = qb;
    init.s.nq = 1;
    init.s.it = 1;
    init.s.cap = cap;
    init.bitsF = b0;
    init.bitsN = b1;
    init.hubs = hubs;
    init.nwords = nwords;
    init.n = n;
    const char *pd = getenv("SP_SSSP_PULL_DIV");
    init.pull_div = pd ? atoll(pd) : kPullDiv;
    SP_CUDA(cudaMemcpyAsync(D, &init, sizeof(DoLoop), cudaMemcpyHostToDevice, c.stream));
    const int sms = num_sms(c.device);
    const int grid = sms * 8;
    const int64_t warps = (int64_t)grid * (kExpandBlock / 32);
    const bool big = g->max_outdeg > kSplit;
    // edge-balanced pull (SP_SSSP_PULL_TILES=1: the older row-tile kernels)
    const bool units = !getenv("SP_SSSP_PULL_TILES") && g->m > 0;
    // hot-source snapshot in shared memory (the PageRank hot encoding of
    // radj), built on the graph's second direction-optimising run like PR's
    // (SP_SSSP_HOT=0: off, =1: from the first run)
    const char *he = getenv("SP_SSSP_HOT");
    int H = 0;
    if (units && !(he && he[0] == '0')) {
        // an optimisation: a failed build (e.g. out of memory) keeps the plain sweep
        if ((g->sssp_do_runs++ > 0 || (he && he[0] == '1')) && pr_hot_build(g, c) != SP_OK)
            cudaGetLastError();
        H = g->pr_H > 0 ? g->pr_H : 0;
    }
    int32_t *hotd = nullptr;
    if (H) SP_TRY(c.alloc(&hotd, H + 4));
    const size_t hot_smem = (size_t)((H + 3) & ~3) * 4 + (kSpHotBlock / 32) * (kSpCh / 32) * 4;
    if (H)
        SP_CUDA(cudaFuncSetAttribute(k_spull_units_hot, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)hot_smem));
    SPull sp{};
    if (units) {
        sp.radj = H ? g->pr_radj_hot : g->radj;
        sp.rw = g->rweff;
        sp.nzend = g->nzend;
        sp.nzrow = g->nzrow;
        sp.m = g->m;
        sp.nnz = g->nnz_rows;
        sp.nunits = (g->m + kSpUnit - 1) / kSpUnit;
        int64_t *ur, *hp, *tp;
        SP_TRY(c.alloc(&ur, sp.nunits));
        SP_TRY(c.alloc(&hp, sp.nunits));
        SP_TRY(c.alloc(&tp, sp.nunits));
        sp.unit_row = ur;
        sp.hp = hp;
        sp.tp = tp;
        k_spull_setup<<<grid_for(sp.nunits, 256, c.device), 256, 0, c.stream>>>(sp);
        c.launches++;
    }
    cudaGraph_t graph = nullptr;
    struct GraphFree {
        cudaGraph_t *g;
        ~GraphFree() {
            if (*g) cudaGraphDestroy(*g);
        }
    } gf{&graph};
    // body of one iteration (set_cond: inside the conditional graph)
    auto body_launch = [&](cudaGraphConditionalHandle hh, int set_cond) {
        k_do_push<<<grid, kExpandBlock, 0, c.stream>>>(dist, enq, g->weff, g->off, g->adj, chunks,
                                                       D, warps);
        if (big)
            k_do_push_chunks<<<grid, kExpandBlock, 0, c.stream>>>(dist, enq, g->weff, g->off,
                                                                  g->adj, chunks, D);
        if (units && H) {
            k_spull_hot_gather<<<std::max(1, (H + 255) / 256), 256, 0, c.stream>>>(
                D, g->pr_hot_ids, H, dist, hotd);
            k_spull_units_hot<<<sms, kSpHotBlock, hot_smem, c.stream>>>(sp, dist, D, hotd, H);
            k_spull_fix<<<grid_for(sp.nunits, 256, c.device), 256, 0, c.stream>>>(sp, dist, D);
        } else if (units) {
            k_spull_units<<<(int)std::max<int64_t>(1, (sp.nunits + 7) / 8), 256, 0, c.stream>>>(
                sp, dist, D);
            k_spull_fix<<<grid_for(sp.nunits, 256, c.device), 256, 0, c.stream>>>(sp, dist, D);
        } else {
            k_pull_tiles<<<grid, 256, 0, c.stream>>>(g->roff, g->radj, g->rweff, dist, D);
            k_pull_hubs<<<sms * 2, 256, 0, c.stream>>>(g->roff, g->radj, g->rweff, dist, D);
        }
        k_do_advance<<<1, 1, 0, c.stream>>>(D, hh, set_cond);
        k_do_clear<<<grid, 256, 0, c.stream>>>(D);
        k_do_convert<<<grid, 256, 0, c.stream>>>(D);
        k_do_mode<<<1, 1, 0, c.stream>>>(D);
    };
    // SP_HOSTLOOP=2: host-driven iterations of this loop with per-iteration
    // device times (SP_SSSP_TRACE prints them; ncu can profile every kernel)
    const char *hl = getenv("SP_HOSTLOOP");
    if (hl && hl[0] == '2') {
        static const bool tr = getenv("SP_SSSP_TRACE") != nullptr;
        DoLoop *hD;
        SP_TRY(c.host_as(&hD));
        cudaEvent_t e0, e1;
        SP_CUDA(cudaEventCreate(&e0));
        SP_CUDA(cudaEventCreate(&e1));
        float tot = 0.f;
        for (;;) {
            SP_CUDA(cudaMemcpyAsync(hD, D, sizeof(DoLoop), cudaMemcpyDeviceToHost, c.stream));
            SP_CUDA(cudaStreamSynchronize(c.stream));
            const int mode = hD->mode;
            const int64_t nq = hD->s.nq;
            cudaEventRecord(e0, c.stream);
            body_launch(0, 0);
            cudaEventRecord(e1, c.stream);
            SP_CUDA(cudaGetLastError());
            SP_CUDA(cudaMemcpyAsync(hD, D, sizeof(DoLoop), cudaMemcpyDeviceToHost, c.stream));
            SP_CUDA(cudaStreamSynchronize(c.stream));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            tot += ms;
            if (tr)
                fprintf(stderr, "sssp do it %lld: %s frontier %lld -> %lld, %.3f ms\n",
                        (long long)hD->s.iters, mode ? "pull" : "push", (long long)nq,
                        (long long)hD->s.nq, ms);
            if (!hD->go) break;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *kernel_ms = tot;
        *out = hD->s;
        c.launches += hD->s.iters * ((big ? 8 : 7) + (H ? 1 : 0));
        return SP_OK;
    }
    SP_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h;
    SP_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    SP_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    SP_CUDA(cudaStreamBeginCaptureToGraph(c.stream, body, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
    body_launch(h, 1);
    SP_CUDA(cudaStreamEndCapture(c.stream, &body));
    cudaEvent_t ka, kb;
    SP_CUDA(cudaEventCreate(&ka));
    SP_CUDA(cudaEventCreate(&kb));
    cudaEventRecord(ka, c.stream);
    SP_TRY(launch_cached_graph(graph, g, kLoopSsspDo, c.stream));
    cudaEventRecord(kb, c.stream);
    DoLoop *hD;
    SP_TRY(c.host_as(&hD));
    SP_CUDA(cudaMemcpyAsync(hD, D, sizeof(DoLoop), cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    cudaEventElapsedTime(kernel_ms, ka, kb);
    cudaEventDestroy(ka);
    cudaEventDestroy(kb);
    *out = hD->s;
    c.launches += hD->s.iters * ((big ? 8 : 7) + (H ? 1 : 0));
    return SP_OK;
}

// Near-far threshold step; 0 selects plain Bellman-Ford (negative weights,
// or SP_SSSP_DELTA=0).  Default: kDeltaMul x the mean of the weight range.
int64_t near_far_delta(const sp_graph *g, int32_t wmin, int32_t wmax) {
    if (g->m == 0 || wmin < 0) return 0;
    const char *env = getenv("SP_SSSP_DELTA");
    if (env) return atoll(env);
    // road-like (low average degree, long shortest paths) graphs only; on
    // low-diameter graphs (RMAT) plain Bellman-Ford needs fewer iterations
    if (g->m > kNearFarMaxAvgDeg * g->n) return 0;
    const int64_t mean = ((int64_t)wmin + (int64_t)wmax + 1) / 2;
    return std::max<int64_t>(1, kDeltaMul * mean);
}

int sssp_device_loop(sp_graph *g, Call &c, int32_t *dist, int32_t *enq, int32_t *qa, int32_t *qb,
                     ChunkItem *chunks, int64_t cap, SsspLoop *hL, float *kernel_ms,
                     int32_t init_src) {
    SsspLoop *L;
    SP_TRY(c.alloc(&L, 1));
    SsspLoop init{};
    init.q[0] = qa;
    init.q[1] = qb;
    init.nq = 1;
    init.it = 1;
    init.cap = cap;
    SP_CUDA(cudaMemcpyAsync(L, &init, sizeof(SsspLoop), cudaMemcpyHostToDevice, c.stream));
    const int sms = num_sms(c.device);
    // blocks per SM of the loop's kernels: small graphs pay for launching an
    // idle grid every iteration (cfg1: 8 -> 0.36 ms, 4 -> 0.32 ms; RMAT-22
    // wants 8); SP_SSSP_GRID_MUL overrides
    const char *gm = getenv("SP_SSSP_GRID_MUL");
    const int grid = sms * (gm ? std::max(1, atoi(gm)) : (g->m < (int64_t(1) << 22) ? 4 : 8));
    // (dist, stamp) words: one returning atomic per improving slot
    // (SP_SSSP_PACKED=0: separate dist / enq arrays)
    const char *pe = getenv("SP_SSSP_PACKED");
    const bool packed = !(pe && pe[0] == '0');
    const int64_t warps = (int64_t)grid * (kExpandBlock / 32);
    const bool big = g->max_outdeg > kSplit;
    long long *dq = nullptr;
    if (packed) {
        SP_TRY(c.alloc(&dq, std::max<int64_t>(1, g->n)));
        k_init_packed<<<grid_for(g->n, kBlock, c.device), kBlock, 0, c.stream>>>(dq, g->n, init_src);
    }
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    struct GraphFree {
        cudaGraph_t *g;
        cudaGraphExec_t *e;
        ~GraphFree() {
            if (*e) cudaGraphExecDestroy(*e);
            if (*g) cudaGraphDestroy(*g);
        }
    } gf{&graph, &exec};
    SP_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h;
    SP_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    SP_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    SP_CUDA(cudaStreamBeginCaptureToGraph(c.stream, body, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
    auto body_nodes = [&](auto op) {
        k_relax_loop<<<grid, kExpandBlock, 0, c.stream>>>(op, g->off, g->adj, chunks, L, warps);
        if (big)
            k_relax_loop_chunks<<<grid, kExpandBlock, 0, c.stream>>>(op, g->off, g->adj, chunks, L,
                                                                     h);
        else
            k_loop_advance<<<1, 1, 0, c.stream>>>(L, h);
    };
    // (a variant without the dq[x] pre-read before the atomic measured the
    // same on cfg1 and 1.5x slower on RMAT-22: more atomics)
    if (packed)
        body_nodes(RelaxPackedOp{dq, g->weff, nullptr, 0});
    else
        body_nodes(RelaxOp{dist, enq, g->weff, nullptr, 0});
    cudaError_t ce = cudaStreamEndCapture(c.stream, &body);
    SP_CUDA(ce);
    cudaEvent_t ka, kb;
    SP_CUDA(cudaEventCreate(&ka));
    SP_CUDA(cudaEventCreate(&kb));
    cudaEventRecord(ka, c.stream);
    SP_TRY(launch_cached_graph(graph, g, kLoopSsspBf, c.stream));
    if (packed) k_unpack<<<grid_for(g->n, kBlock, c.device), kBlock, 0, c.stream>>>(dq, g->n, dist);
    cudaEventRecord(kb, c.stream);
    SP_CUDA(cudaMemcpyAsync(hL, L, sizeof(SsspLoop), cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    cudaEventElapsedTime(kernel_ms, ka, kb);
    cudaEventDestroy(ka);
    cudaEventDestroy(kb);
    c.launches += hL->iters * 2 + (packed ? 2 : 0);
    return SP_OK;
}

}  // namespace

static int sssp_impl(sp_graph *g, int32_t src, int64_t cap, int32_t *dist_out, int mem,
                     int64_t *iters_out, sp_iter_cb cb, void *user, sp_stats *st,
                     bool pull_form) {
    SP_CHECK(g && dist_out, SP_ERR_ARG, "sp_sssp: bad arguments");
    SP_CHECK(src >= 0 && src < g->n, SP_ERR_ARG, "node argument 'src'=%d out of range", src);
    static const bool trace = getenv("SP_SSSP_TRACE") != nullptr;  // host phase times
    const auto tt0 = std::chrono::steady_clock::now();
    auto tms = [&]() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tt0)
            .count();
    };
    Call c;
    SP_TRY(c.begin(g->device));
    SP_TRY(ensure_weff(g, c));
    const int64_t n = g->n;
    int32_t *dist, *enq, *qa, *qb;
    ChunkItem *chunks;
    ExpandCounters *cnt;
    SP_TRY(c.alloc(&dist, n));
    SP_TRY(c.alloc(&enq, n));
    SP_TRY(c.alloc(&qa, n));
    SP_TRY(c.alloc(&qb, n));
    SP_TRY(c.alloc(&chunks, expand_chunk_capacity(g->m)));
    SP_TRY(c.alloc(&cnt, 2));
    SP_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(ExpandCounters), c.stream));
    ExpandCounters *hc = nullptr;
    SP_TRY(c.host_as(&hc));
    const int dev = c.device;
    const int sms = num_sms(dev);
    const bool big = g->max_outdeg > kSplit;
    c.persist(dist, n * sizeof(int32_t));  // the relaxations' random probes
    k_init<<<grid_for(n, kBlock, dev), kBlock, 0, c.stream>>>(dist, enq, n, src, qa);
    c.launches++;
    if (trace) fprintf(stderr, "sssp: begin+allocs %.2f ms\n", tms());
    int64_t nq = 1, iters = 0, relaxed = 0, frontier_sum = 0;
    int rc = SP_OK;
    cudaEvent_t ka, kb;
    SP_CUDA(cudaEventCreate(&ka));
    SP_CUDA(cudaEventCreate(&kb));
    float kernel_ms = 0.f;
    // SP_HOSTLOOP=1 keeps the host-driven loop (ncu cannot profile the
    // kernel nodes of a graph with conditional nodes)
    const char *hostloop = getenv("SP_HOSTLOOP");
    if (!cb && !(hostloop && hostloop[0] == '1')) {
        SsspLoop hL{};
        int lrc;
        int32_t wr[2] = {0, 0};
        if (g->m) {  // cached at creation: no blocking copy per call
            wr[0] = g->wmin_h;
            wr[1] = g->wmax_h;
        }
        const int64_t delta = pull_form ? 0 : near_far_delta(g, wr[0], wr[1]);
        // the asynchronous form counts phases, not iterations: it runs when
        // no caller cap is in force (the reference default 2n+16, which no
        // near-far run approaches) and the graph is thin (SP_NF_ASYNC=0: off)
        const char *ae = getenv("SP_NF_ASYNC");
        // (forced onto cfg1's RMAT-16, hub rows walked by one warp: 0.9 ms --
        // 2x the relaxations of the synchronous loop, 3.4 entries per batch)
        const bool async_nf = delta > 0 && g->max_outdeg <= kSplit && cap >= 2 * n + 16 &&
                              !(ae && ae[0] == '0');
        if (async_nf) {
            lrc = sssp_near_far_async(g, c, dist, src, delta, &hL, &kernel_ms);
            if (lrc == SP_OK && hL.status == 3) {  // overflow / watchdog: synchronous form
                k_init<<<grid_for(n, kBlock, dev), kBlock, 0, c.stream>>>(dist, enq, n, src, qa);
                c.launches++;
                hL = SsspLoop{};
                lrc = sssp_near_far(g, c, dist, enq, qa, qb, chunks, cap, delta, &hL, &kernel_ms);
            }
        } else if (delta > 0) {
            lrc = sssp_near_far(g, c, dist, enq, qa, qb, chunks, cap, delta, &hL, &kernel_ms);
        }
        if (trace) fprintf(stderr, "sssp: loop done %.2f ms (kernel %.2f ms)\n", tms(), kernel_ms);
        if (delta <= 0 || (lrc == SP_OK && hL.status == 3)) {  // Bellman-Ford
            k_init<<<grid_for(n, kBlock, dev), kBlock, 0, c.stream>>>(dist, enq, n, src, qa);
            c.launches++;
            hL = SsspLoop{};
            const char *de = getenv("SP_SSSP_DO");  // direction-optimising push SSSP
            const bool use_do = de ? de[0] == '1' : g->m >= kDoMinSlots;
            if (pull_form || use_do)  // sssp_pull.sp: pull steps for large frontiers
                lrc = sssp_do_loop(g, c, dist, enq, qa, qb, chunks, cap, &hL, &kernel_ms);
            else
                lrc = sssp_device_loop(g, c, dist, enq, qa, qb, chunks, cap, &hL, &kernel_ms, src);
        }
        if (lrc == SP_OK) {
            iters = hL.iters;
            relaxed = hL.relaxed;
            frontier_sum = hL.frontier_sum;
            if (hL.status == 1) {
                set_error("SSSP distance left the int32 range (negative weights)");
                rc = SP_ERR_OVERFLOW;
            } else if (hL.status == 2) {
                set_error("fixedPoint 'finished' did not converge within %lld iterations",
                          (long long)cap);
                rc = SP_ERR_NONCONV;
            }
            cudaEventDestroy(ka);
            cudaEventDestroy(kb);
            goto done;
        }
        return lrc;
    }
    for (;;) {
        ExpandCounters *cur = cnt + (iters & 1);
        RelaxOp op{dist, enq, g->weff, &cur->flag, (int)(iters + 1)};
        cudaEventRecord(ka, c.stream);
        launch_expand(op, g->off, g->adj, qa, nq, qb, chunks, cur, sms, big, c.stream, &c.launches);
        cudaEventRecord(kb, c.stream);
        SP_CUDA(cudaGetLastError());
        SP_CUDA(cudaMemcpyAsync(hc, cur, sizeof(ExpandCounters), cudaMemcpyDeviceToHost, c.stream));
        SP_CUDA(cudaMemsetAsync(cnt + ((iters + 1) & 1), 0, sizeof(ExpandCounters), c.stream));
        SP_CUDA(cudaStreamSynchronize(c.stream));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ka, kb);
        kernel_ms += ms;
        iters++;
        frontier_sum += nq;
        relaxed += (int64_t)hc->scanned;
        if (trace)
            fprintf(stderr, "sssp it %lld: frontier %lld, scanned %llu, next %llu, %.1f us\n",
                    (long long)iters, (long long)nq, (unsigned long long)hc->scanned,
                    (unsigned long long)hc->next_size, ms * 1e3);
        if (hc->flag) {
            set_error("SSSP distance left the int32 range (negative weights)");
            rc = SP_ERR_OVERFLOW;
            break;
        }
        nq = (int64_t)hc->next_size;
        std::swap(qa, qb);
        if (cb && cb(iters, user)) {
            set_error("aborted by the fixedPoint iteration callback");
            rc = SP_ERR_ABORTED;
            break;
        }
        if (nq == 0) break;  // finished = !modified
        if (iters >= cap) {
            set_error("fixedPoint 'finished' did not converge within %lld iterations",
                      (long long)cap);
            rc = SP_ERR_NONCONV;
            break;
        }
    }
    cudaEventDestroy(ka);
    cudaEventDestroy(kb);
done:
    if (rc == SP_OK || rc == SP_ERR_NONCONV) SP_TRY(from_device(dist_out, dist, n * 4, mem, c.stream));
    SP_TRY(c.finish(st));
    if (iters_out) *iters_out = iters;
    if (st) {
        st->iterations = iters;
        st->edges_visited = relaxed;
        st->vertices_visited = frontier_sum;
        st->main_kernel_ms = kernel_ms;
        st->main_kernel_launches = iters;
        // 12 B per relaxation (adj 4, w_eff 4, dist[x] 4) + 20 B
        // per frontier vertex (two offsets 16, dist[v] 4)
        st->model_bytes = 12 * relaxed + 20 * frontier_sum;
    }
    return rc;
}

extern "C" int sp_sssp(sp_graph *g, int32_t src, int64_t cap, int32_t *dist_out, int mem,
                       int64_t *iters_out, sp_iter_cb cb, void *user, sp_stats *st) {
    return sssp_impl(g, src, cap, dist_out, mem, iters_out, cb, user, st, false);
}

extern "C" int sp_sssp_pull(sp_graph *g, int32_t src, int64_t cap, int32_t *dist_out, int mem,
                            int64_t *iters_out, sp_iter_cb cb, void *user, sp_stats *st) {
    return sssp_impl(g, src, cap, dist_out, mem, iters_out, cb, user, st, true);
}

// ---- owner-computes shards (multi-GPU, graph.py:226-249 ownership) -------
// One shard per rank owns dist[v] for v in [v0, v1).  A superstep relaxes
// the owned frontier (one pass, or local passes to a fixpoint: bsp.py:290-306
// repeat_local) with atomicMin into the rank's dist array; owned winners form
// the next local frontier, remote winners are collected once per superstep
// (stamp-deduped) and sent as ONE aggregated (vertex, local minimum) message
// per vertex -- the reference's aggregate_messages (bsp.py:45-72) and the
// paper's "single message with local minimum value".  The owner applies the
// messages it receives with a strict min (bsp.py:350-368) and appends the
// winners to its frontier.  Messages are packed (vid << 32 | uint32 dist),
// grouped by owner rank for an all-to-all; or, for dense supersteps, the
// caller reduce-scatters the whole dist array with MIN and applies its block.
namespace {

// Relaxation of sssp.sp:11-12 for a shard: owned winners -> next local
// frontier (1), remote winners -> outbox (2, once per superstep).
struct RelaxShardOp {
    using Payload = int;
    using Probe = RelaxOp::Probe;
    static constexpr bool kFar = true;
    int32_t *__restrict__ dist;
    int32_t *__restrict__ enq;
    const int32_t *__restrict__ weff;
    unsigned long long *overflow;
    int32_t *far_q;               // outbox vertex ids
    unsigned long long *far_n;
    unsigned long long far_cap;
    int64_t v0, v1;
    int it;      // round stamp (owned vertices)
    int sstamp;  // superstep stamp (remote vertices)
    // fused exchange (peers != null): a remote winner lowers the owner's
    // dist in place (peer memory: CUDA IPC, NVLink between GPUs) and, once
    // per superstep, appends itself to the owner's inbox -- the message
    // exchange rides on the relaxation kernel; the local dist entry of a
    // remote vertex stays this rank's best sent value (the pre-filter)
    int32_t *const *peer_dist;
    int32_t *const *peer_inbox;
    unsigned long long *const *peer_tail;
    int64_t per;
    unsigned long long inbox_cap;
    unsigned long long *msg_counts;  // fused: messages sent per owner (the trace)
    __device__ __forceinline__ int payload(int32_t v) const { return __ldcg(dist + v); }
    __device__ __forceinline__ Probe probe(int64_t e, int32_t x) const {
        return Probe{__ldcs(weff + e), __ldcg(dist + x)};
    }
    __device__ __forceinline__ int apply(int dv, int64_t, int32_t x, Probe p) const {
        const int64_t cand = (int64_t)dv + (int64_t)p.w;
        if (cand >= (int64_t)kIntMax) return 0;  // F12
        if (cand < (int64_t)(-2147483647 - 1)) {
            atomicAdd(overflow, 1ull);
            return 0;
        }
        const int c = (int)cand;
        if (c >= p.dx) return 0;
        const int old = atomicMin(dist + x, c);
        if (c >= old) return 0;
        if (x >= v0 && x < v1) return atomicExch(enq + x, it) != it ? 1 : 0;
        if (peer_dist) {
            const int64_t r = x / per;
            if (c < atomicMin(peer_dist[r] + x, c) && atomicExch(enq + x, sstamp) != sstamp) {
                const unsigned long long pos = atomicAdd(peer_tail[r], 1ull);
                if (pos < inbox_cap) peer_inbox[r][pos] = x;
                else atomicAdd(overflow, 1ull << 32);  // inbox overflow (never: capacity n)
                atomicAdd(msg_counts + r, 1ull);
            }
            return 0;
        }
        return atomicExch(enq + x, sstamp) != sstamp ? 2 : 0;
    }
};

// Fused-exchange collect: the owner's inbox (vertices other ranks lowered in
// its dist this superstep) joins its frontier (apply-stamp deduped).
__global__ void k_shard_collect(const int32_t *__restrict__ inbox, int64_t k, int32_t *enq,
                                int stamp, int32_t *q, unsigned long long *nq) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < k; b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = b + threadIdx.x;
        bool win = false;
        int32_t x = 0;
        if (i < k) {
            x = __ldcg(inbox + i);
            win = atomicExch(enq + x, stamp) != stamp;
        }
        const int64_t at = warp_append(win, nq);
        if (win) q[at] = x;
    }
}

__global__ void k_shard_init(int32_t *dist, int32_t *enq, int64_t n, int32_t src) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        dist[x] = x == src ? 0 : kIntMax;
        enq[x] = -1;
    }
}

// Outbox -> per-owner counts (block partition: owner = v / per).
__global__ void k_shard_count(const int32_t *__restrict__ ob, int64_t k, int64_t per, int world,
                              unsigned long long *counts) {
    extern __shared__ unsigned long long s_cnt[];
    for (int r = threadIdx.x; r < world; r += blockDim.x) s_cnt[r] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&s_cnt[ob[i] / per], 1ull);
    __syncthreads();
    for (int r = threadIdx.x; r < world; r += blockDim.x)
        if (s_cnt[r]) atomicAdd(&counts[r], s_cnt[r]);
}

// Packed messages grouped by owner: cursor[r] starts at the owner's offset.
__global__ void k_shard_pack(const int32_t *__restrict__ ob, int64_t k, int64_t per,
                             const int32_t *__restrict__ dist, unsigned long long *cursor,
                             int64_t *send) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t x = ob[i];
        const unsigned long long at = atomicAdd(&cursor[x / per], 1ull);
        send[at] = ((int64_t)x << 32) | (int64_t)(uint32_t)__ldcg(dist + x);
    }
}

// Owner apply of received messages (strict min, bsp.py:350-368); winners
// join the local frontier (deduped with the apply stamp).
__global__ void k_shard_apply(const int64_t *__restrict__ msg, int64_t k, int32_t *dist,
                              int32_t *enq, int stamp, int32_t *q, unsigned long long *nq) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < k; b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = b + threadIdx.x;
        bool win = false;
        int32_t x = 0;
        if (i < k) {
            const int64_t m = msg[i];
            x = (int32_t)(m >> 32);
            const int32_t c = (int32_t)(uint32_t)(m & 0xffffffffll);
            win = c < __ldcg(dist + x) && c < atomicMin(dist + x, c) &&
                  atomicExch(enq + x, stamp) != stamp;
        }
        const int64_t at = warp_append(win, nq);
        if (win) q[at] = x;
    }
}

// Dense form: block[v - v0] = min over the ranks' dist[v] (reduce-scatter).
__global__ void k_shard_apply_dense(const int32_t *__restrict__ blk, int64_t v0, int64_t v1,
                                    int32_t *dist, int32_t *enq, int stamp, int32_t *q,
                                    unsigned long long *nq) {
    for (int64_t b = v0 + blockIdx.x * (int64_t)blockDim.x; b < v1;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = b + threadIdx.x;
        bool win = false;
        if (v < v1) {
            const int32_t c = blk[v - v0];
            if (c < dist[v]) {
                dist[v] = c;  // owned: only this rank writes it
                win = atomicExch(enq + v, stamp) != stamp;
            }
        }
        const int64_t at = warp_append(win, nq);
        if (win) q[at] = (int32_t)v;
    }
}

}  // namespace

struct sp_sssp_shard {
    sp_graph *g = nullptr;
    int64_t v0 = 0, v1 = 0;
    int32_t *dist = nullptr;  // caller's device array (>= n entries)
    int32_t *enq = nullptr, *q[2] = {nullptr, nullptr}, *ob = nullptr;
    ChunkItem *chunks = nullptr;
    ExpandCounters *cnt = nullptr;          // [2]
    unsigned long long *aux = nullptr;      // [0] outbox size, [1] apply appends, [2..] per-owner counts/cursors
    int world = 0;
    int cur = 0;
    int64_t nq = 0;     // |q[cur]|
    int64_t qcap = 0;
    int round = 0;      // round stamps 1, 2, ...
    int step = 0;       // supersteps done
    // fused exchange: device tables of every rank's dist / inbox / inbox tail
    int32_t **peer_dist = nullptr, **peer_inbox = nullptr;
    unsigned long long **peer_tail = nullptr;
    int32_t *inbox = nullptr;            // this rank's inbox (peer-mapped, caller-owned)
    unsigned long long *tail = nullptr;  // its tail
    int64_t per = 0;
};

static void shard_free(sp_sssp_shard *h) {
    if (!h) return;
    void *ps[] = {h->enq, h->q[0], h->q[1], h->ob, h->chunks, h->cnt, h->aux, h->peer_dist,
                  h->peer_inbox, h->peer_tail};
    for (void *p : ps)
        if (p) resident_free(p);
    delete h;
}

extern "C" int sp_sssp_shard_create(sp_graph *g, int64_t v0, int64_t v1, int32_t src, int world,
                                    int32_t *dist, sp_sssp_shard **out) {
    SP_CHECK(g && dist && out && v0 >= 0 && v0 <= v1 && v1 <= g->n && world >= 1 && world <= 4096,
             SP_ERR_ARG, "sp_sssp_shard_create: bad arguments");
    SP_CHECK(src >= 0 && src < g->n, SP_ERR_ARG, "node argument 'src'=%d out of range", src);
    *out = nullptr;
    Call c;
    SP_TRY(c.begin(g->device));
    SP_TRY(ensure_weff(g, c));
    sp_sssp_shard *h = new sp_sssp_shard;
    h->g = g;
    h->v0 = v0;
    h->v1 = v1;
    h->dist = dist;
    h->world = world;
    h->qcap = 2 * (v1 - v0) + 2;  // a frontier plus the messages applied to it
    const int64_t n = g->n;
    int rc = SP_OK;
    auto al = [&](void **p, size_t b) {
        if (rc == SP_OK) rc = resident_alloc(p, b);
    };
    al((void **)&h->enq, n * 4);
    al((void **)&h->q[0], h->qcap * 4);
    al((void **)&h->q[1], h->qcap * 4);
    al((void **)&h->ob, std::max<int64_t>(1, n) * 4);
    al((void **)&h->chunks, expand_chunk_capacity(g->m) * sizeof(ChunkItem));
    al((void **)&h->cnt, 2 * sizeof(ExpandCounters));
    al((void **)&h->aux, (2 + 2 * (size_t)world) * 8);
    if (rc != SP_OK) {
        shard_free(h);
        return rc;
    }
    k_shard_init<<<grid_for(n, kBlock, c.device), kBlock, 0, c.stream>>>(dist, h->enq, n, src);
    c.launches++;
    SP_CUDA(cudaMemsetAsync(h->cnt, 0, 2 * sizeof(ExpandCounters), c.stream));
    if (src >= v0 && src < v1) {  // the owner of src starts with it
        SP_CUDA(cudaMemcpyAsync(h->q[0], &src, 4, cudaMemcpyHostToDevice, c.stream));
        h->nq = 1;
    }
    rc = c.finish(nullptr);
    if (rc != SP_OK) {
        shard_free(h);
        return rc;
    }
    *out = h;
    return SP_OK;
}

extern "C" int sp_sssp_shard_relax(sp_sssp_shard *h, int64_t max_rounds, int64_t per,
                                   int64_t *send, int64_t *counts, int64_t *info) {
    SP_CHECK(h && send && counts && per >= 1 && max_rounds >= 1, SP_ERR_ARG,
             "sp_sssp_shard_relax: bad arguments");
    sp_graph *g = h->g;
    Call c;
    SP_TRY(c.begin(g->device));
    ExpandCounters *hc;
    SP_TRY(c.host_as(&hc));
    const int sms = num_sms(c.device);
    const bool big = g->max_outdeg > kSplit;
    h->step++;
    SP_CUDA(cudaMemsetAsync(h->aux, 0, (2 + 2 * (size_t)h->world) * 8, c.stream));
    int64_t updates = 0, relaxed = 0, rounds = 0;
    bool overflow = false;
    while (h->nq > 0 && rounds < max_rounds) {
        h->round++;
        ExpandCounters *cc = h->cnt + h->cur;
        SP_CUDA(cudaMemsetAsync(cc, 0, sizeof(ExpandCounters), c.stream));
        RelaxShardOp op{h->dist, h->enq, g->weff, &cc->flag, h->ob, &h->aux[0],
                        (unsigned long long)std::max<int64_t>(1, g->n), h->v0, h->v1,
                        h->round, h->step, h->peer_dist, h->peer_inbox, h->peer_tail, h->per,
                        (unsigned long long)std::max<int64_t>(1, g->n), h->aux + 2};
        launch_expand(op, g->off, g->adj, h->q[h->cur], h->nq, h->q[h->cur ^ 1], h->chunks, cc,
                      sms, big, c.stream, &c.launches);
        SP_CUDA(cudaGetLastError());
        SP_CUDA(cudaMemcpyAsync(hc, cc, sizeof(ExpandCounters), cudaMemcpyDeviceToHost, c.stream));
        SP_CUDA(cudaStreamSynchronize(c.stream));
        updates += (int64_t)hc->next_size;  // owned Min wins (bsp.py:213-216)
        relaxed += (int64_t)hc->scanned;
        rounds++;
        h->cur ^= 1;
        h->nq = (int64_t)hc->next_size;
        if (hc->flag) {
            SP_CHECK((hc->flag >> 32) == 0, SP_ERR_CUDA, "sp_sssp_shard_relax: inbox overflow");
            overflow = true;
            break;
        }
    }
    if (h->peer_dist) {  // fused exchange: the messages are already in the owners' inboxes
        unsigned long long *hk = reinterpret_cast<unsigned long long *>(hc);
        SP_CUDA(cudaMemcpyAsync(hk, h->aux + 2, h->world * 8, cudaMemcpyDeviceToHost, c.stream));
        SP_TRY(c.finish(nullptr));
        for (int r = 0; r < h->world; r++) counts[r] = (int64_t)hk[r];  // sent (trace only)
        if (info) {
            info[0] = updates;
            info[1] = relaxed;
            info[2] = rounds;
            info[3] = h->nq;
        }
        SP_CHECK(!overflow, SP_ERR_OVERFLOW,
                 "SSSP distance left the int32 range (negative weights)");
        return SP_OK;
    }
    // outbox -> per-owner counts -> packed messages grouped by owner
    unsigned long long *hk = reinterpret_cast<unsigned long long *>(hc);
    SP_CUDA(cudaMemcpyAsync(hk, h->aux, 8, cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    const int64_t k = (int64_t)hk[0];
    unsigned long long *dcnt = h->aux + 2, *dcur = h->aux + 2 + h->world;
    if (k > 0) {
        k_shard_count<<<grid_for(k, kBlock, c.device), kBlock, h->world * 8, c.stream>>>(
            h->ob, k, per, h->world, dcnt);
        c.launches++;
    }
    SP_CUDA(cudaMemcpyAsync(hk, dcnt, h->world * 8, cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<unsigned long long> start(h->world);
    unsigned long long acc = 0;
    for (int r = 0; r < h->world; r++) {
        counts[r] = (int64_t)hk[r];
        start[r] = acc;
        acc += hk[r];
    }
    if (k > 0) {
        SP_CUDA(cudaMemcpyAsync(dcur, start.data(), h->world * 8, cudaMemcpyHostToDevice, c.stream));
        k_shard_pack<<<grid_for(k, kBlock, c.device), kBlock, 0, c.stream>>>(h->ob, k, per, h->dist,
                                                                            dcur, send);
        c.launches++;
    }
    SP_TRY(c.finish(nullptr));
    if (info) {
        info[0] = updates;
        info[1] = relaxed;
        info[2] = rounds;
        info[3] = h->nq;  // owned frontier left for the next superstep
    }
    SP_CHECK(!overflow, SP_ERR_OVERFLOW, "SSSP distance left the int32 range (negative weights)");
    return SP_OK;
}

extern "C" int sp_sssp_shard_apply(sp_sssp_shard *h, const int64_t *msgs, int64_t k,
                                   const int32_t *block, int64_t *frontier) {
    SP_CHECK(h && k >= 0 && (k == 0 || msgs || block), SP_ERR_ARG,
             "sp_sssp_shard_apply: bad arguments");
    sp_graph *g = h->g;
    Call c;
    SP_TRY(c.begin(g->device));
    unsigned long long *hk;
    SP_TRY(c.host_as(&hk));
    // apply stamps are negative (never a round stamp) and fresh per superstep
    const int stamp = -2 - h->step;
    SP_CUDA(cudaMemcpyAsync(h->aux + 1, &h->nq, 8, cudaMemcpyHostToDevice, c.stream));
    int32_t *q = h->q[h->cur];
    if (block && h->v1 > h->v0) {
        k_shard_apply_dense<<<grid_for(h->v1 - h->v0, kBlock, c.device), kBlock, 0, c.stream>>>(
            block, h->v0, h->v1, h->dist, h->enq, stamp, q, h->aux + 1);
        c.launches++;
    } else if (!block && k > 0) {
        k_shard_apply<<<grid_for(k, kBlock, c.device), kBlock, 0, c.stream>>>(
            msgs, k, h->dist, h->enq, stamp, q, h->aux + 1);
        c.launches++;
    }
    SP_CUDA(cudaMemcpyAsync(hk, h->aux + 1, 8, cudaMemcpyDeviceToHost, c.stream));
    SP_TRY(c.finish(nullptr));
    h->nq = (int64_t)hk[0];
    SP_CHECK(h->nq <= h->qcap, SP_ERR_CUDA, "sp_sssp_shard_apply: frontier overflow");
    if (frontier) *frontier = h->nq;
    return SP_OK;
}

extern "C" int sp_sssp_shard_peers(sp_sssp_shard *h, int64_t per, int32_t *const *peer_dist,
                                   int32_t *const *peer_inbox,
                                   unsigned long long *const *peer_tail, int32_t *inbox,
                                   unsigned long long *tail) {
    SP_CHECK(h && per >= 1 && peer_dist && peer_inbox && peer_tail && inbox && tail, SP_ERR_ARG,
             "sp_sssp_shard_peers: bad arguments");
    Call c;
    SP_TRY(c.begin(h->g->device));
    const size_t b = (size_t)h->world * sizeof(void *);
    void *d[3] = {nullptr, nullptr, nullptr};
    const void *src[3] = {peer_dist, peer_inbox, peer_tail};
    for (int i = 0; i < 3; i++) {
        int rc = resident_alloc(&d[i], b);
        if (rc != SP_OK) {
            for (int j = 0; j < i; j++) resident_free(d[j]);
            return rc;
        }
        SP_CUDA(cudaMemcpyAsync(d[i], src[i], b, cudaMemcpyHostToDevice, c.stream));
    }
    SP_CUDA(cudaMemsetAsync(tail, 0, 8, c.stream));
    SP_TRY(c.finish(nullptr));
    h->peer_dist = static_cast<int32_t **>(d[0]);
    h->peer_inbox = static_cast<int32_t **>(d[1]);
    h->peer_tail = static_cast<unsigned long long **>(d[2]);
    h->inbox = inbox;
    h->tail = tail;
    h->per = per;
    return SP_OK;
}

extern "C" int sp_sssp_shard_collect(sp_sssp_shard *h, int64_t *frontier) {
    SP_CHECK(h && h->inbox, SP_ERR_ARG, "sp_sssp_shard_collect: no peers set");
    Call c;
    SP_TRY(c.begin(h->g->device));
    unsigned long long *hk;
    SP_TRY(c.host_as(&hk));
    SP_CUDA(cudaMemcpyAsync(hk, h->tail, 8, cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    const int64_t k = (int64_t)hk[0];
    SP_CHECK(k <= h->g->n, SP_ERR_CUDA, "sp_sssp_shard_collect: inbox overflow");
    const int stamp = -2 - h->step;  // as sp_sssp_shard_apply
    SP_CUDA(cudaMemcpyAsync(h->aux + 1, &h->nq, 8, cudaMemcpyHostToDevice, c.stream));
    if (k > 0) {
        k_shard_collect<<<grid_for(k, kBlock, c.device), kBlock, 0, c.stream>>>(
            h->inbox, k, h->enq, stamp, h->q[h->cur], h->aux + 1);
        c.launches++;
    }
    SP_CUDA(cudaMemsetAsync(h->tail, 0, 8, c.stream));
    SP_CUDA(cudaMemcpyAsync(hk, h->aux + 1, 8, cudaMemcpyDeviceToHost, c.stream));
    SP_TRY(c.finish(nullptr));
    h->nq = (int64_t)hk[0];
    SP_CHECK(h->nq <= h->qcap, SP_ERR_CUDA, "sp_sssp_shard_collect: frontier overflow");
    if (frontier) *frontier = h->nq;
    return SP_OK;
}

extern "C" void sp_sssp_shard_destroy(sp_sssp_shard *h) {
    if (!h) return;
    cudaSetDevice(h->g->device);
    cudaDeviceSynchronize();
    shard_free(h);
}
