// sp_bc.cu -- corpus/programs/bc.sp on sm_100a (Brandes, level-synchronous).
//
// Reference semantics (bc.sp:4-20 under trident/interp.py):
//   for src in sourceSet (list order, duplicates re-run, interp.py:384-385):
//     sigma = delta = 0; sigma[src] = 1
//     iterateInBFS from src over forward adjacency (interp.py:445-461):
//       ascending levels: sigma_v += sigma_w for in-neighbours w at level-1
//     iterateInReverse (descending levels):
//       delta_v += sigma_v / sigma_w * (1 + delta_w) over out-neighbours w at
//       level+1, then bc_v += delta_v / 2 if v != src.
//
// Fast mode (default) runs the sources in batches of kLanes = 8 with
// lane-major vertex state and direction-optimising discovery -- see
// "Batched sources" below (bc_run_batches).  Deterministic mode and
// SP_BC_BATCH=0 use the per-source plan:
// Device plan per source (graph resident; level int32[n], sigma/delta f64[n],
// one queue int32[n] holding all BFS levels back to back):
//   level L -> L+1 : load-balanced top-down expansion (sp_expand.cuh) with a
//                    CAS on level[x] (-1 -> L+1) appending the next level;
//                    one frontier-size read per level.  Fast mode pushes
//                    sigma in the same pass (DiscoverSigmaOp, exact);
//   sigma(L+1)     : deterministic mode: ordered pull fold over reverse-CSR
//                    rows of the new level (sp_fold.cuh), term = sigma[u] if
//                    level[u] == L;
//   reverse sweep  : ordered fold over CSR rows of each level, deepest first,
//                    term = sigma_v / sigma_w * (1 + delta_w) if level[w] ==
//                    L+1, then bc += delta / 2 in the same kernel.
// The root's own sigma pull only adds +0.0 terms (its "parents" are the
// unreached level -1 vertices) and the deepest level has no children, so
// both are skipped without changing a bit.  Sigma values are path counts:
// integer-valued doubles, exact in any summation order below 2^53.
#include <algorithm>
#include <chrono>
#include <thread>
#include <vector>

#include "sp_expand.cuh"
#include "sp_fold.cuh"

using namespace sp;

namespace {

constexpr int64_t kBcHub = 8192;  // rows longer than this take the CTA fold
constexpr int kBcWorkers = 4;     // concurrent sources (host threads/streams), per-source fast path
constexpr int kBbWorkers = 4;     // concurrent source batches, batched fast path (3: 60.8 ms, 4: 59.6 ms at cfg4)

// Per-vertex record, 16 bytes: level (int32) and, in fast mode, the child
// coefficient coef[w] = (1 + delta[w]) / sigma[w] (written when delta[w] is
// final).  A delta-fold term then needs ONE random 16-byte read (level and
// coef share a sector) instead of level, sigma[w] and delta[w].  `level`
// below points at the record array viewed as int32, stride kVs.
constexpr int64_t kVs = 4;
__device__ __forceinline__ int32_t *lvl(int32_t *vs, int32_t x) { return vs + kVs * (int64_t)x; }
__device__ __forceinline__ const int32_t *lvl(const int32_t *vs, int32_t x) {
    return vs + kVs * (int64_t)x;
}

struct DiscoverOp {
    using Payload = int;
    using Probe = int;  // level[x]
    int32_t *__restrict__ level;
    int next;
    __device__ __forceinline__ int payload(int32_t) const { return 0; }
    __device__ __forceinline__ int probe(int64_t, int32_t x) const { return __ldcg(lvl(level, x)); }
    __device__ __forceinline__ bool apply(int, int64_t, int32_t x, int lx) const {
        if (lx != -1) return false;
        return atomicCAS(lvl(level, x), -1, next) == -1;
    }
};

// Fast mode: discovery and the sigma accumulation of bc.sp:10-12 in one
// push over the level-L out-edges.  Every edge v -> x with level[x] == L+1
// (won or lost CAS alike) adds sigma[v]; sigma values are path counts, i.e.
// integer-valued doubles, so the atomic adds are exact in any order (below
// 2^53) and the result equals the reference's ordered fold bit for bit.
struct DiscoverSigmaOp {
    using Payload = double;
    using Probe = int;  // level[x]
    int32_t *__restrict__ level;
    double *__restrict__ sigma;
    int next;
    __device__ __forceinline__ double payload(int32_t v) const { return __ldcg(sigma + v); }
    __device__ __forceinline__ int probe(int64_t, int32_t x) const { return __ldcg(lvl(level, x)); }
    __device__ __forceinline__ bool apply(double sv, int64_t, int32_t x, int lx) const {
        if (lx != -1 && lx != next) return false;
        bool won = false;
        if (lx == -1) {
            const int old = atomicCAS(lvl(level, x), -1, next);
            won = old == -1;
            if (!won && old != next) return false;
        }
        atomicAdd(sigma + x, sv);
        return won;
    }
};

struct SigmaFold {  // bc.sp:10-12 over reverse-CSR slots (deterministic mode)
    const int32_t *__restrict__ radj;
    const int32_t *__restrict__ level;
    double *__restrict__ sigma;
    int parent_level;
    __device__ __forceinline__ double payload(int32_t) const { return 0.0; }
    __device__ __forceinline__ int32_t key(int64_t k) const { return radj[k]; }
    __device__ __forceinline__ double term(double, int32_t u) const {
        return __ldg(lvl(level, u)) == parent_level ? sigma[u] : 0.0;
    }
    __device__ __forceinline__ void finish(int32_t v, double s) const { sigma[v] = s; }
};

struct DeltaFold {  // bc.sp:14-19 over CSR slots (deterministic mode: exact formula)
    const int32_t *__restrict__ adj;
    const int32_t *__restrict__ level;
    const double *__restrict__ sigma;
    double *__restrict__ delta;
    double *__restrict__ bc;
    int child_level;
    int32_t src;
    __device__ __forceinline__ double payload(int32_t v) const { return sigma[v]; }
    __device__ __forceinline__ int32_t key(int64_t e) const { return adj[e]; }
    __device__ __forceinline__ double term(double sv, int32_t w) const {
        if (__ldg(lvl(level, w)) != child_level) return 0.0;
        return __dmul_rn(__ddiv_rn(sv, sigma[w]), __dadd_rn(1.0, delta[w]));
    }
    __device__ __forceinline__ void finish(int32_t v, double s) const {
        delta[v] = s;
        if (v != src) bc[v] = __dadd_rn(bc[v], __ddiv_rn(s, 2.0));
    }
};

// Fast mode: term = sigma_v * coef_w from one 16-byte record read
// (sigma_v / sigma_w * (1 + delta_w) regrouped: a few ulps apart).
struct DeltaFoldFast {
    const int32_t *__restrict__ adj;
    int32_t *__restrict__ vs;  // records (level, coef)
    const double *__restrict__ sigma;
    double *__restrict__ delta;
    double *__restrict__ bc;
    int child_level;
    int32_t src;
    __device__ __forceinline__ double payload(int32_t v) const { return sigma[v]; }
    __device__ __forceinline__ int32_t key(int64_t e) const { return __ldcs(adj + e); }
    __device__ __forceinline__ double term(double sv, int32_t w) const {
        const int4 r = __ldg(reinterpret_cast<const int4 *>(vs) + w);
        if (r.x != child_level) return 0.0;
        return __dmul_rn(sv, __hiloint2double(r.w, r.z));
    }
    __device__ __forceinline__ void finish(int32_t v, double s) const {
        delta[v] = s;
        reinterpret_cast<double *>(vs)[2 * (int64_t)v + 1] =
            __ddiv_rn(__dadd_rn(1.0, s), sigma[v]);
        if (v != src) bc[v] = __dadd_rn(bc[v], __ddiv_rn(s, 2.0));
    }
};

// coef of the deepest level's vertices (no children: delta = 0)
__global__ void k_leaf_coef(const int32_t *__restrict__ q, int64_t nq, int32_t *vs,
                            const double *__restrict__ sigma) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = q[i];
        reinterpret_cast<double *>(vs)[2 * (int64_t)v + 1] = __ddiv_rn(1.0, sigma[v]);
    }
}

__global__ void k_root(int32_t *level, double *sigma, int32_t *queue, int32_t s) {
    level[kVs * (int64_t)s] = 0;
    sigma[s] = 1.0;
    queue[0] = s;
}


// One worker: a stream (its thread's), its own scratch and bc partial, and
// the sources srcs[first], srcs[first + stride], ... in list order.
struct BcWorker {
    int64_t levels = 0, scanned = 0, reached = 0, launches = 0, pull_steps = 0;
    int rc = SP_OK;
    char err[512] = "";
};

int bc_run_sources(sp_graph *g, const std::vector<int32_t> &srcs, int64_t first, int64_t stride,
                   bool det, double *bc_dst, int bc_mem, bool bc_accumulate_only,
                   double *sigma_out, double *delta_out, int mem, BcWorker &wk) {
    Call c;
    // worker k of a multi-worker call runs on the device's persistent slot-k stream
    SP_TRY(stride > 1 ? c.begin_worker(g->device, (int)first) : c.begin(g->device));
    const int64_t n = g->n;
    const int64_t nsrc = (int64_t)srcs.size();
    const int sms = num_sms(c.device);
    int32_t *level, *queue, *hubs, *reg_v, *reg_nch;
    uint4 *items;
    int64_t *reg_base;
    double *csum;
    double *sigma, *delta, *bc;
    ChunkItem *chunks;
    ExpandCounters *cnt;
    unsigned long long *nhubs;
    SP_TRY(c.alloc(&level, kVs * n));  // 16-byte (level, coef) records
    SP_TRY(c.alloc(&queue, n));
    SP_TRY(c.alloc(&hubs, n));
    const int64_t ccap = fold_chunk_capacity(g->m);
    SP_TRY(c.alloc(&reg_v, n));
    SP_TRY(c.alloc(&reg_nch, n));
    SP_TRY(c.alloc(&reg_base, n));
    SP_TRY(c.alloc(&items, ccap));
    SP_TRY(c.alloc(&csum, ccap));
    SP_TRY(c.alloc(&sigma, n));
    SP_TRY(c.alloc(&delta, n));
    SP_TRY(c.alloc(&bc, n));
    SP_TRY(c.alloc(&chunks, expand_chunk_capacity(g->m)));
    SP_TRY(c.alloc(&cnt, 1));
    SP_TRY(c.alloc(&nhubs, 3));
    const FoldLists fl{hubs, nhubs, FoldChunks{reg_v, reg_base, reg_nch, items, csum, nullptr}};
    c.persist(level, kVs * n * sizeof(int32_t));  // BFS/fold probes hit the records at random
    SP_CUDA(cudaMemsetAsync(bc, 0, n * sizeof(double), c.stream));
    SP_CUDA(cudaMemsetAsync(sigma, 0, n * sizeof(double), c.stream));
    SP_CUDA(cudaMemsetAsync(delta, 0, n * sizeof(double), c.stream));
    ExpandCounters *hc = nullptr;
    SP_TRY(c.host_as(&hc));
    const bool big_out = g->max_outdeg > kSplit;
    std::vector<int64_t> ls;
    int64_t last_done = -1;
    for (int64_t si = first; si < nsrc; si += stride) {
        const int32_t s = srcs[si];
        SP_CUDA(cudaMemsetAsync(level, 0xFF, kVs * n * sizeof(int32_t), c.stream));
        if (last_done >= 0) {
            SP_CUDA(cudaMemsetAsync(sigma, 0, n * sizeof(double), c.stream));
            SP_CUDA(cudaMemsetAsync(delta, 0, n * sizeof(double), c.stream));
        }
        k_root<<<1, 1, 0, c.stream>>>(level, sigma, queue, s);
        c.launches++;
        ls.assign({0, 1});
        for (int L = 0;; L++) {
            const int64_t q0 = ls[L], q1 = ls[L + 1];
            SP_CUDA(cudaMemsetAsync(cnt, 0, sizeof(ExpandCounters), c.stream));
            if (det) {
                DiscoverOp op{level, L + 1};
                launch_expand(op, g->off, g->adj, queue + q0, q1 - q0, queue + q1, chunks, cnt,
                              sms, big_out, c.stream, &c.launches);
            } else {
                DiscoverSigmaOp op{level, sigma, L + 1};
                launch_expand(op, g->off, g->adj, queue + q0, q1 - q0, queue + q1, chunks, cnt,
                              sms, big_out, c.stream, &c.launches);
            }
            SP_CUDA(cudaGetLastError());
            SP_CUDA(cudaMemcpyAsync(hc, cnt, sizeof(ExpandCounters), cudaMemcpyDeviceToHost,
                                    c.stream));
            SP_CUDA(cudaStreamSynchronize(c.stream));
            wk.scanned += (int64_t)hc->scanned;
            const int64_t nnew = (int64_t)hc->next_size;
            if (nnew == 0) break;
            ls.push_back(q1 + nnew);
            if (det) {
                SigmaFold sf{g->radj, level, sigma, L};
                launch_fold(sf, g->roff, queue + q1, nnew, kBcHub, fl, true, g->max_indeg, sms,
                            c.stream, &c.launches);
            }
        }
        const int nlev = (int)ls.size() - 1;
        wk.levels += nlev;
        wk.reached += ls.back();
        if (!det && nlev >= 2) {
            const int64_t d0 = ls[nlev - 1], d1 = ls[nlev];
            k_leaf_coef<<<grid_for(d1 - d0, 256, c.device), 256, 0, c.stream>>>(queue + d0,
                                                                               d1 - d0, level,
                                                                               sigma);
            c.launches++;
        }
        for (int L = nlev - 2; L >= 0; L--) {
            if (det) {
                DeltaFold df{g->adj, level, sigma, delta, bc, L + 1, s};
                launch_fold(df, g->off, queue + ls[L], ls[L + 1] - ls[L], kBcHub, fl, det,
                            g->max_outdeg, sms, c.stream, &c.launches);
            } else {
                DeltaFoldFast df{g->adj, level, sigma, delta, bc, L + 1, s};
                launch_fold(df, g->off, queue + ls[L], ls[L + 1] - ls[L], kBcHub, fl, det,
                            g->max_outdeg, sms, c.stream, &c.launches);
            }
        }
        SP_CUDA(cudaGetLastError());
        last_done = si;
    }
    // bc partial out (a device buffer of the caller, or the final output)
    if (bc_accumulate_only) {
        SP_CUDA(cudaMemcpyAsync(bc_dst, bc, n * 8, cudaMemcpyDeviceToDevice, c.stream));
    } else {
        SP_TRY(from_device(bc_dst, bc, n * 8, bc_mem, c.stream));
    }
    if (last_done == nsrc - 1) {  // this worker ran the list's last source
        if (sigma_out) SP_TRY(from_device(sigma_out, sigma, n * 8, mem, c.stream));
        if (delta_out) SP_TRY(from_device(delta_out, delta, n * 8, mem, c.stream));
    }
    SP_TRY(c.finish(nullptr));
    wk.launches = c.launches;
    return SP_OK;
}

// ---------------------------------------------------------------------------
// Batched sources (fast mode).  kLanes sources run one BFS together: vertex
// state is lane-major per vertex -- level int32[kLanes] (one 32-byte sector),
// sigma and coef f64[kLanes] -- so one random level read answers "which
// sources see this neighbour at the next level" for all of them, and the
// delta fold reads a neighbour's coef only for the lanes that match.  The
// per-source arithmetic is unchanged: sigma by exact integer atomics during
// discovery, delta_v = sigma_v * sum(coef_w) over children, coef_v =
// (1 + delta_v) / sigma_v, bc_v += delta_v / 2 for v != src.  A vertex is
// queued once per distinct depth it has across the lanes (stamp[v] = last
// depth queued), so level d's queue holds every vertex with some lane at d.
constexpr int kLanes = 8;
constexpr int kBbShort = 64;     // rows up to this length: one thread, sequential (32: 69.6 ms, 64: 61 ms, 128: 67 ms at cfg4)
constexpr int kBbSplit = 256;    // longer rows: 256-slot chunks, one warp each
constexpr double kBbPullRatio = 4.0;  // direction choice, see bc_run_batches

struct BatchSrc {
    int32_t s[kLanes];  // -1: unused lane
};

// A vertex's kLanes levels (one 32-byte sector) / 4 of its f64 lanes, each
// read with ONE 256-bit load (LDG.256): a random 32-byte read costs one L1
// wavefront instead of two (int4 x 2) or eight (scalar lanes).
struct Lev8 {
    int x[kLanes];
};
__device__ __forceinline__ Lev8 load_lev(const int32_t *lev, int32_t v) {  // L2 (.cg)
    Lev8 l;
    asm volatile("ld.global.cg.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(l.x[0]), "=r"(l.x[1]), "=r"(l.x[2]), "=r"(l.x[3]), "=r"(l.x[4]),
                   "=r"(l.x[5]), "=r"(l.x[6]), "=r"(l.x[7])
                 : "l"(lev + kLanes * (int64_t)v));
    return l;
}
__device__ __forceinline__ Lev8 load_lev_ro(const int32_t *lev, int32_t v) {  // read-only path
    Lev8 l;
    asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(l.x[0]), "=r"(l.x[1]), "=r"(l.x[2]), "=r"(l.x[3]), "=r"(l.x[4]), "=r"(l.x[5]),
          "=r"(l.x[6]), "=r"(l.x[7])
        : "l"(lev + kLanes * (int64_t)v));
    return l;
}
__device__ __forceinline__ void load_f64x4_ro(const double *p, double (&o)[4]) {
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
        : "l"(p));
}
__device__ __forceinline__ unsigned lanes_eq(const Lev8 &l, int d) {
    unsigned m = 0;
#pragma unroll
    for (int s = 0; s < kLanes; s++) m |= (unsigned)(l.x[s] == d) << s;
    return m;
}
// acc[s] += coef_w[s] for the lanes in m (m != 0): two 256-bit loads
__device__ __forceinline__ void add_lanes(const double *cw, unsigned m, double (&acc)[kLanes]) {
    double c[kLanes];
    if (m & 0x0Fu) load_f64x4_ro(cw, *reinterpret_cast<double(*)[4]>(c));
    if (m & 0xF0u) load_f64x4_ro(cw + 4, *reinterpret_cast<double(*)[4]>(c + 4));
#pragma unroll
    for (int s = 0; s < kLanes; s++)
        if (m >> s & 1u) acc[s] = __dadd_rn(acc[s], c[s]);
}

// Discovery + sigma push for all lanes of level `cur` in one pass.
struct BatchDiscoverOp {
    using Payload = unsigned long long;  // v | lanes at `cur` << 32
    using Probe = unsigned;              // lanes unvisited | lanes at `next` << 8
    int32_t *__restrict__ lev;
    double *__restrict__ sig;
    int32_t *__restrict__ stamp;
    int cur, next;
    __device__ __forceinline__ Payload payload(int32_t v) const {
        return (unsigned)v | (Payload)lanes_eq(load_lev_ro(lev, v), cur) << 32;
    }
    __device__ __forceinline__ unsigned probe(int64_t, int32_t x) const {
        const Lev8 l = load_lev(lev, x);
        return lanes_eq(l, -1) | lanes_eq(l, next) << 8;
    }
    __device__ __forceinline__ bool apply(Payload pay, int64_t, int32_t x, unsigned pr) const {
        unsigned act = (unsigned)(pay >> 32) & (pr | pr >> 8) & 0xFFu;
        if (!act) return false;
        const int64_t v8 = kLanes * (int64_t)(unsigned)pay, x8 = kLanes * (int64_t)x;
        bool won = false;
        do {
            const int s = __ffs(act) - 1;
            act &= act - 1;
            if (pr >> s & 1u) {
                const int old = atomicCAS(lev + x8 + s, -1, next);
                if (old == -1) won = true;
                else if (old != next) continue;
            }
            atomicAdd(sig + x8 + s, __ldg(sig + v8 + s));
        } while (act);
        return won && atomicMax(stamp + x, next) < next;
    }
};

__global__ void k_bb_root(int32_t *lev, double *sig, int32_t *stamp, int32_t *queue, BatchSrc b) {
    int k = 0;
    for (int s = 0; s < kLanes; s++) {
        const int32_t v = b.s[s];
        if (v < 0) continue;
        lev[kLanes * (int64_t)v + s] = 0;
        sig[kLanes * (int64_t)v + s] = 1.0;
        if (stamp[v] != 0) {
            stamp[v] = 0;
            queue[k++] = v;
        }
    }
}

struct BatchFold {
    const int64_t *__restrict__ off;
    const int32_t *__restrict__ adj;
    const int32_t *__restrict__ lev;
    const double *__restrict__ sig;
    double *__restrict__ coef;
    double *__restrict__ bc;
    double *__restrict__ dlast;  // delta of lane `last` (or null)
    int last;
    BatchSrc src;
    int d;
    // delta/coef/bc of v's lanes `act` (at depth d) from their child sums
    __device__ __forceinline__ void finish(int32_t v, unsigned act, const double (&acc)[kLanes]) const {
        const int64_t v8 = kLanes * (int64_t)v;
        double add = 0.0;
        bool any = false;
#pragma unroll
        for (int s = 0; s < kLanes; s++) {
            if (!(act >> s & 1u)) continue;
            const double sv = sig[v8 + s];
            const double dv = __dmul_rn(sv, acc[s]);
            coef[v8 + s] = __ddiv_rn(__dadd_rn(1.0, dv), sv);
            if (s == last && dlast) dlast[v] = dv;
            if (v != src.s[s]) {
                add = __dadd_rn(add, __ddiv_rn(dv, 2.0));
                any = true;
            }
        }
        if (any) bc[v] = __dadd_rn(bc[v], add);
    }
    // add the coef of w's lanes at d+1 among `act` to acc
    __device__ __forceinline__ void term(int32_t w, unsigned act, double (&acc)[kLanes]) const {
        const unsigned m = lanes_eq(load_lev_ro(lev, w), d + 1) & act;
        if (m) add_lanes(coef + kLanes * (int64_t)w, m, acc);
    }
};

// Long rows: registered (vertex, first chunk, chunk count), one work item
// per 256-slot chunk; a chunk's per-lane sums go to csum[item] and the
// row's finish adds them in chunk order (fixed shape: the batched path is
// deterministic run to run, like the per-source one).
struct BbChunks {
    int32_t *reg_v;              // long rows of this level
    int64_t *reg_base;           // first chunk item
    int32_t *reg_nch;            // chunk count
    uint4 *items;                // {reg index, first slot lo, hi, count}
    double *csum;                // [item][kLanes] chunk sums
    unsigned long long *counts;  // [0] long rows, [1] chunks
};

__device__ __forceinline__ void bb_register(const BbChunks &ck, int64_t r, int32_t v, int64_t r0,
                                            int64_t deg) {
    ck.reg_v[r] = v;
    const int nch = (int)((deg + kBbSplit - 1) / kBbSplit);
    const int64_t b0 = (int64_t)atomicAdd(&ck.counts[1], (unsigned long long)nch);
    ck.reg_base[r] = b0;
    ck.reg_nch[r] = nch;
    for (int c = 0; c < nch; c++) {
        const int64_t s0 = r0 + (int64_t)c * kBbSplit;
        const int64_t len = min((int64_t)kBbSplit, r0 + deg - s0);
        ck.items[b0 + c] = make_uint4((unsigned)r, (unsigned)(uint64_t)s0,
                                      (unsigned)((uint64_t)s0 >> 32), (unsigned)len);
    }
}

// warp sums of acc per lane in `act`, stored as the chunk's partials
__device__ __forceinline__ void bb_store_chunk(const BbChunks &ck, int64_t k, unsigned act,
                                               const double (&acc)[kLanes]) {
    double mine = 0.0;
#pragma unroll
    for (int s = 0; s < kLanes; s++) {
        double x = 0.0;
        if (act >> s & 1u) {  // warp-uniform
            x = acc[s];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
        }
        if ((int)lane_id() == s) mine = x;
    }
    if (lane_id() < kLanes) ck.csum[kLanes * k + lane_id()] = mine;
}

// Row r's lane sums from its chunks' partials, by one warp: lane j adds
// chunks j, j+32, ... in order, then a fixed xor tree -- the same shape
// every run (deterministic), and a hub row's hundreds of chunks are not
// summed by a single thread.  Every lane returns the sums.
__device__ __forceinline__ void bb_row_sums(const BbChunks &ck, int64_t r, double (&acc)[kLanes]) {
    const int64_t b0 = ck.reg_base[r];
    const int nch = ck.reg_nch[r];
#pragma unroll
    for (int s = 0; s < kLanes; s++) acc[s] = 0.0;
    for (int c = lane_id(); c < nch; c += 32) {
        double p[kLanes];
        load_f64x4_ro(ck.csum + kLanes * (b0 + c), *reinterpret_cast<double(*)[4]>(p));
        load_f64x4_ro(ck.csum + kLanes * (b0 + c) + 4, *reinterpret_cast<double(*)[4]>(p + 4));
#pragma unroll
        for (int s = 0; s < kLanes; s++) acc[s] = __dadd_rn(acc[s], p[s]);
    }
#pragma unroll
    for (int s = 0; s < kLanes; s++)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            acc[s] = __dadd_rn(acc[s], __shfl_xor_sync(0xffffffffu, acc[s], o));
}

// Level d's rows: short rows folded by one thread; long rows registered and
// cut into chunks.  Deepest level (leaf = true): no children, coef = 1/sigma.
#ifndef SP_BBROWS_MINB
#define SP_BBROWS_MINB 5
#endif
__global__ void __launch_bounds__(256, SP_BBROWS_MINB) k_bb_rows(BatchFold f, const int32_t *__restrict__ q,
                                                 int64_t nq, bool leaf, BbChunks ck) {
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < nq;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        int32_t v = -1;
        unsigned act = 0;
        int64_t r0 = 0, deg = 0;
        if (i < nq) {
            v = q[i];
            act = lanes_eq(load_lev_ro(f.lev, v), f.d);
            r0 = f.off[v];
            deg = leaf ? 0 : f.off[v + 1] - r0;
        }
        const bool longrow = deg > kBbShort;
        const int64_t r = warp_append(longrow, &ck.counts[0]);
        if (longrow) {
            bb_register(ck, r, v, r0, deg);
        } else if (v >= 0) {
            double acc[kLanes];
#pragma unroll
            for (int s = 0; s < kLanes; s++) acc[s] = 0.0;
            for (int64_t e = r0; e < r0 + deg; e += 4) {
                int32_t w[4];
#pragma unroll
                for (int u = 0; u < 4; u++) w[u] = e + u < r0 + deg ? __ldg(f.adj + e + u) : -1;
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (w[u] >= 0) f.term(w[u], act, acc);
            }
            f.finish(v, act, acc);
        }
    }
}

// One warp per chunk: lanes take slots j*32 + lane, then a fixed-shape warp
// reduction per source lane into the chunk's partials.
#ifndef SP_BB_MINB
// blocks/SM the batched chunk kernels are compiled for (76 -> 64 registers)
// -- with SP_BBROWS_MINB 5, BC cfg4 65 -> 55 ms in one measurement pair
#define SP_BB_MINB 4
#endif
__global__ void __launch_bounds__(256, SP_BB_MINB) k_bb_chunks(BatchFold f, BbChunks ck) {
    constexpr int kPer = kBbSplit / 32;
    const unsigned lane = lane_id();
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nitems = (int64_t)__ldcg(&ck.counts[1]);
    const uint4 none = make_uint4(0, 0, 0, 0);
    // software pipeline over the warp's chunks: the descriptor two ahead and
    // the slots + row lanes of the next chunk load while this chunk's level
    // and coef reads are in flight
    auto load = [&](const uint4 it, int32_t (&w)[kPer], unsigned &act) {
        const int64_t s0 = (int64_t)(((uint64_t)it.z << 32) | it.y);
#pragma unroll
        for (int j = 0; j < kPer; j++) {
            const unsigned p = j * 32 + lane;
            w[j] = p < it.w ? __ldcs(f.adj + s0 + p) : -1;
        }
        act = it.w ? lanes_eq(load_lev_ro(f.lev, ck.reg_v[it.x]), f.d) : 0u;
    };
    int32_t w[kPer];
    unsigned act;
    load(warp < nitems ? ck.items[warp] : none, w, act);
    uint4 d1 = warp + nwarps < nitems ? ck.items[warp + nwarps] : none;
    for (int64_t k = warp; k < nitems; k += nwarps) {
        const uint4 d2 = k + 2 * nwarps < nitems ? ck.items[k + 2 * nwarps] : none;
        int32_t wn[kPer];
        unsigned actn;
        load(d1, wn, actn);
        unsigned m[kPer];
#pragma unroll
        for (int j = 0; j < kPer; j++)
            m[j] = w[j] >= 0 ? lanes_eq(load_lev_ro(f.lev, w[j]), f.d + 1) & act : 0u;
        double acc[kLanes];
#pragma unroll
        for (int s = 0; s < kLanes; s++) acc[s] = 0.0;
#pragma unroll
        for (int j = 0; j < kPer; j++)
            if (m[j]) add_lanes(f.coef + kLanes * (int64_t)w[j], m[j], acc);
        bb_store_chunk(ck, k, act, acc);
#pragma unroll
        for (int j = 0; j < kPer; j++) w[j] = wn[j];
        act = actn;
        d1 = d2;
    }
}

// one warp per long row
#ifndef SP_BBFIN_MINB
#define SP_BBFIN_MINB 5  // BC cfg4: 59.7 -> 56.8 ms
#endif
__global__ void __launch_bounds__(256, SP_BBFIN_MINB) k_bb_finish(BatchFold f, BbChunks ck) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nreg = (int64_t)__ldcg(&ck.counts[0]);
    for (int64_t r = warp; r < nreg; r += nwarps) {
        double acc[kLanes];
        bb_row_sums(ck, r, acc);
        if (lane_id() == 0) {
            const int32_t v = ck.reg_v[r];
            f.finish(v, lanes_eq(load_lev_ro(f.lev, v), f.d), acc);
        }
    }
}

// Bottom-up (pull) form of one discovery step, for the large middle levels
// (direction optimisation): every vertex w with a lane still unvisited sums
// sigma over its in-neighbours at level d for those lanes, and the lanes
// with a non-zero sum join level d+1 -- written by w's owner alone, so no
// CAS and no sigma atomics.  Sums of path counts are exact in any order, so
// sigma is identical to the push form's.  Concurrent readers of lev[w] see
// -1 or d+1, never d, so the in-place update is race-free.
struct BatchPull {
    const int64_t *__restrict__ roff;
    const int32_t *__restrict__ radj;
    int32_t *__restrict__ lev;
    double *__restrict__ sig;
    int32_t *__restrict__ stamp;
    int32_t *__restrict__ qn;   // next level's queue
    ExpandCounters *cnt;        // next_size
    int d;
    __device__ __forceinline__ void term(int32_t v, unsigned pm, double (&acc)[kLanes]) const {
        const unsigned m = lanes_eq(load_lev_ro(lev, v), d) & pm;
        if (m) add_lanes(sig + kLanes * (int64_t)v, m, acc);
    }
    // lanes of w with a parent join level d+1; true => w is queued
    __device__ __forceinline__ bool finish(int32_t w, unsigned pm,
                                           const double (&acc)[kLanes]) const {
        const int64_t w8 = kLanes * (int64_t)w;
        bool any = false;
#pragma unroll
        for (int s = 0; s < kLanes; s++)
            if ((pm >> s & 1u) && acc[s] != 0.0) {
                lev[w8 + s] = d + 1;
                sig[w8 + s] = acc[s];
                any = true;
            }
        if (any) stamp[w] = d + 1;
        return any;
    }
};

#ifndef SP_BBPULL_MINB
#define SP_BBPULL_MINB 5  // BC cfg4: 59.7 -> 57.5 ms (6: 65 ms)
#endif
__global__ void __launch_bounds__(256, SP_BBPULL_MINB) k_bb_pull_rows(BatchPull f, int64_t n, BbChunks ck) {
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        unsigned pm = 0;
        int64_t r0 = 0, deg = 0;
        if (i < n) {
            pm = lanes_eq(load_lev_ro(f.lev, (int32_t)i), -1);
            if (pm) {
                r0 = f.roff[i];
                deg = f.roff[i + 1] - r0;
            }
        }
        const bool longrow = deg > kBbShort;
        const int64_t r = warp_append(longrow, &ck.counts[0]);
        bool push = false;
        if (longrow) {
            bb_register(ck, r, (int32_t)i, r0, deg);
        } else if (deg > 0) {
            double acc[kLanes];
#pragma unroll
            for (int s = 0; s < kLanes; s++) acc[s] = 0.0;
            for (int64_t e = r0; e < r0 + deg; e += 4) {
                int32_t v[4];
#pragma unroll
                for (int u = 0; u < 4; u++) v[u] = e + u < r0 + deg ? __ldg(f.radj + e + u) : -1;
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (v[u] >= 0) f.term(v[u], pm, acc);
            }
            push = f.finish((int32_t)i, pm, acc);
        }
        const int64_t slot = warp_append(push, &f.cnt->next_size);
        if (push) f.qn[slot] = (int32_t)i;
    }
}

__global__ void __launch_bounds__(256, SP_BB_MINB) k_bb_pull_chunks(BatchPull f, BbChunks ck) {
    constexpr int kPer = kBbSplit / 32;
    const unsigned lane = lane_id();
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nitems = (int64_t)__ldcg(&ck.counts[1]);
    const uint4 none = make_uint4(0, 0, 0, 0);
    // pipelined like k_bb_chunks
    auto load = [&](const uint4 it, int32_t (&v)[kPer], unsigned &pm) {
        const int64_t s0 = (int64_t)(((uint64_t)it.z << 32) | it.y);
#pragma unroll
        for (int j = 0; j < kPer; j++) {
            const unsigned p = j * 32 + lane;
            v[j] = p < it.w ? __ldcs(f.radj + s0 + p) : -1;
        }
        pm = it.w ? lanes_eq(load_lev_ro(f.lev, ck.reg_v[it.x]), -1) : 0u;
    };
    int32_t v[kPer];
    unsigned pm;
    load(warp < nitems ? ck.items[warp] : none, v, pm);
    uint4 d1 = warp + nwarps < nitems ? ck.items[warp + nwarps] : none;
    for (int64_t k = warp; k < nitems; k += nwarps) {
        const uint4 d2 = k + 2 * nwarps < nitems ? ck.items[k + 2 * nwarps] : none;
        int32_t vn[kPer];
        unsigned pmn;
        load(d1, vn, pmn);
        unsigned m[kPer];
#pragma unroll
        for (int j = 0; j < kPer; j++)
            m[j] = v[j] >= 0 ? lanes_eq(load_lev_ro(f.lev, v[j]), f.d) & pm : 0u;
        double acc[kLanes];
#pragma unroll
        for (int s = 0; s < kLanes; s++) acc[s] = 0.0;
#pragma unroll
        for (int j = 0; j < kPer; j++)
            if (m[j]) add_lanes(f.sig + kLanes * (int64_t)v[j], m[j], acc);
        bb_store_chunk(ck, k, pm, acc);
#pragma unroll
        for (int j = 0; j < kPer; j++) v[j] = vn[j];
        pm = pmn;
        d1 = d2;
    }
}

// one warp per long row
__global__ void __launch_bounds__(256) k_bb_pull_finish(BatchPull f, BbChunks ck) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nreg = (int64_t)__ldcg(&ck.counts[0]);
    for (int64_t r = warp; r < nreg; r += nwarps) {
        double acc[kLanes];
        bb_row_sums(ck, r, acc);
        if (lane_id() == 0) {
            const int32_t w = ck.reg_v[r];
            if (f.finish(w, lanes_eq(load_lev(f.lev, w), -1), acc))
                f.qn[atomicAdd(&f.cnt->next_size, 1ull)] = w;
        }
    }
}

// Over a level's queue right after it is complete: the next step's push
// cost (out-slots of the queue), the in-slots of vertices that just lost
// their last unvisited lane (the pull cost drops by these), and the batch
// statistics (lanes reached at this depth, their out-slots, lane mask).
// out: [0] push cost, [1] pull-cost decrement, [2] reached, [3] slots,
// [4] lane mask.
__global__ void k_bb_frontier(const int32_t *__restrict__ lev, const int64_t *__restrict__ off,
                              const int64_t *__restrict__ roff, const int32_t *__restrict__ q,
                              const unsigned long long *nq_dev, int64_t nq_host, int depth,
                              unsigned long long *out) {
    const int64_t nq = nq_dev ? (int64_t)*nq_dev : nq_host;
    unsigned long long fe = 0, dec = 0, reached = 0, slots = 0;
    unsigned lanes = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = q[i];
        const Lev8 l = load_lev(lev, v);
        const unsigned nm = lanes_eq(l, depth);
        const int64_t od = off[v + 1] - off[v];
        fe += od;
        if (!lanes_eq(l, -1)) dec += roff[v + 1] - roff[v];
        reached += __popc(nm);
        slots += (unsigned long long)__popc(nm) * od;
        lanes |= nm;
    }
    fe = warp_sum(fe);
    dec = warp_sum(dec);
    reached = warp_sum(reached);
    slots = warp_sum(slots);
    lanes = __reduce_or_sync(0xffffffffu, lanes);
    if (lane_id() == 0) {
        if (fe) atomicAdd(out, fe);
        if (dec) atomicAdd(out + 1, dec);
        if (reached) atomicAdd(out + 2, reached);
        if (slots) atomicAdd(out + 3, slots);
        if (lanes) atomicOr(out + 4, (unsigned long long)lanes);
    }
}

__global__ void k_bb_lane_out(const double *__restrict__ sig, int lane, int64_t n, double *out) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        out[v] = sig[kLanes * v + lane];
}

// One worker over batches first, first + stride, ... of kLanes sources each
// (sources in list order).  Same contract as bc_run_sources (fast mode).
int bc_run_batches(sp_graph *g, const std::vector<int32_t> &srcs, int64_t first, int64_t stride,
                   double *bc_dst, int bc_mem, bool bc_accumulate_only, double *sigma_out,
                   double *delta_out, int mem, BcWorker &wk) {
    Call c;
    // worker k of a multi-worker call runs on the device's persistent slot-k stream
    const auto wt0 = std::chrono::steady_clock::now();
    static const bool wtrace = getenv("SP_BC_TRACE") != nullptr;
    SP_TRY(stride > 1 ? c.begin_worker(g->device, (int)first) : c.begin(g->device));
    const int64_t n = g->n;
    const int64_t nsrc = (int64_t)srcs.size();
    const int64_t nb = (nsrc + kLanes - 1) / kLanes;
    const int sms = num_sms(c.device);
    int32_t *lev, *stamp, *queue, *reg_v, *reg_nch;
    int64_t *reg_base;
    double *sig, *coef, *bc, *csum, *dlast = nullptr;
    uint4 *items;
    ChunkItem *chunks;
    ExpandCounters *cnt;
    unsigned long long *counts;
    const int64_t qcap = kLanes * n;
    SP_TRY(c.alloc(&lev, kLanes * n));
    SP_TRY(c.alloc(&sig, kLanes * n));
    SP_TRY(c.alloc(&coef, kLanes * n));
    const int64_t icap = g->m / kBbSplit + n + 1;  // chunk items per level
    SP_TRY(c.alloc(&stamp, n));
    SP_TRY(c.alloc(&queue, qcap));
    SP_TRY(c.alloc(&reg_v, n));
    SP_TRY(c.alloc(&reg_nch, n));
    SP_TRY(c.alloc(&reg_base, n));
    SP_TRY(c.alloc(&items, icap));
    SP_TRY(c.alloc(&csum, kLanes * icap));
    SP_TRY(c.alloc(&bc, n));
    SP_TRY(c.alloc(&chunks, expand_chunk_capacity(g->m)));
    SP_TRY(c.alloc(&cnt, 1));
    SP_TRY(c.alloc(&counts, 2 + 5));
    const int fgrid = sms * 2;  // frontier passes: small grids, grid-stride
    if (delta_out) SP_TRY(c.alloc(&dlast, n));
    if (wtrace) {
        cudaStreamSynchronize(c.stream);
        fprintf(stderr, "  worker %lld: setup+allocs %.2f ms\n", (long long)first,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wt0)
                    .count());
    }
    const BbChunks ck{reg_v, reg_base, reg_nch, items, csum, counts};
    c.persist(lev, kLanes * n * sizeof(int32_t));  // the per-slot probe target
    SP_CUDA(cudaMemsetAsync(bc, 0, n * sizeof(double), c.stream));
    ExpandCounters *hc = nullptr;
    SP_TRY(c.host_as(&hc));
    // the call's pinned block: counters at 0, batch stats at 64
    unsigned long long *hs = reinterpret_cast<unsigned long long *>(hc) + 8;
    const bool big_out = g->max_outdeg > kSplit;
    // pull when (push cost) * ratio > (pull cost); SP_BC_PULL overrides, 0 = push only
    const char *pe = getenv("SP_BC_PULL");
    const double pull_ratio = pe ? atof(pe) : kBbPullRatio;
    std::vector<int64_t> ls;
    for (int64_t b = first; b < nb; b += stride) {
        BatchSrc bs;
        int used = 0;
        for (int s = 0; s < kLanes; s++) {
            const int64_t i = b * kLanes + s;
            bs.s[s] = i < nsrc ? srcs[i] : -1;
        }
        int nq0 = 0;  // distinct sources = queue length of depth 0
        for (int s = 0; s < kLanes; s++) {
            if (bs.s[s] < 0) continue;
            used++;
            bool dup = false;
            for (int t = 0; t < s; t++) dup |= bs.s[t] == bs.s[s];
            nq0 += !dup;
        }
        SP_CUDA(cudaMemsetAsync(lev, 0xFF, kLanes * n * sizeof(int32_t), c.stream));
        SP_CUDA(cudaMemsetAsync(stamp, 0xFF, n * sizeof(int32_t), c.stream));
        SP_CUDA(cudaMemsetAsync(sig, 0, kLanes * n * sizeof(double), c.stream));
        k_bb_root<<<1, 1, 0, c.stream>>>(lev, sig, stamp, queue, bs);
        c.launches++;
        ls.assign({0, (int64_t)nq0});
        // per-depth frontier pass: out[5 * d .. 5 * d + 4] (see k_bb_frontier)
        unsigned long long *fo = counts + 2;
        SP_CUDA(cudaMemsetAsync(fo, 0, 5 * sizeof(unsigned long long), c.stream));
        k_bb_frontier<<<fgrid, 256, 0, c.stream>>>(lev, g->off, g->roff, queue, nullptr, nq0, 0,
                                                   fo);
        c.launches++;
        int64_t mu = g->m;  // pull cost: in-slots of vertices with an unvisited lane
        int lane_last[kLanes] = {0};
        for (int d = 0;; d++) {
            const int64_t q0 = ls[d], q1 = ls[d + 1];
            // the previous frontier pass (depth d) is in fo: read it with this step's counters
            SP_CUDA(cudaMemsetAsync(cnt, 0, sizeof(ExpandCounters), c.stream));
            if (d == 0) {
                SP_CUDA(cudaMemcpyAsync(hs, fo, 5 * 8, cudaMemcpyDeviceToHost, c.stream));
                SP_CUDA(cudaStreamSynchronize(c.stream));
            }
            const int64_t mf = (int64_t)hs[0];
            mu -= (int64_t)hs[1];
            wk.reached += (int64_t)hs[2];
            wk.scanned += (int64_t)hs[3];
            for (int s = 0; s < kLanes; s++)
                if (hs[4] >> s & 1u) lane_last[s] = d;
            // pull when its cost (pending in-slots + a sequential pass over
            // the level array) is below ratio x the push cost
            const bool pull = d > 0 && pull_ratio > 0 &&
                              (double)mf * pull_ratio > (double)mu + 0.25 * (double)n;
            if (pull) {
                wk.pull_steps++;
                BatchPull f{g->roff, g->radj, lev, sig, stamp, queue + q1, cnt, d};
                SP_CUDA(cudaMemsetAsync(counts, 0, 2 * sizeof(unsigned long long), c.stream));
                k_bb_pull_rows<<<grid_for(n, 256, c.device), 256, 0, c.stream>>>(f, n, ck);
                c.launches++;
                if (g->max_indeg > kBbShort) {
                    k_bb_pull_chunks<<<sms * 8, 256, 0, c.stream>>>(f, ck);
                    k_bb_pull_finish<<<sms * 8, 256, 0, c.stream>>>(f, ck);
                    c.launches += 2;
                }
            } else {
                BatchDiscoverOp op{lev, sig, stamp, d, d + 1};
                launch_expand(op, g->off, g->adj, queue + q0, q1 - q0, queue + q1, chunks, cnt,
                              sms, big_out, c.stream, &c.launches);
            }
            SP_CUDA(cudaGetLastError());
            SP_CUDA(cudaMemsetAsync(fo, 0, 5 * sizeof(unsigned long long), c.stream));
            k_bb_frontier<<<fgrid, 256, 0, c.stream>>>(lev, g->off, g->roff, queue + q1,
                                                       &cnt->next_size, 0, d + 1, fo);
            c.launches++;
            SP_CUDA(cudaMemcpyAsync(hs, fo, 5 * 8, cudaMemcpyDeviceToHost, c.stream));
            SP_CUDA(cudaMemcpyAsync(hc, cnt, sizeof(ExpandCounters), cudaMemcpyDeviceToHost,
                                    c.stream));
            SP_CUDA(cudaStreamSynchronize(c.stream));
            const int64_t nnew = (int64_t)hc->next_size;
            if (nnew == 0) break;
            ls.push_back(q1 + nnew);
        }
        for (int s = 0; s < used; s++) wk.levels += lane_last[s] + 1;
        const int D = (int)ls.size() - 2;  // deepest depth
        const bool is_last = b == nb - 1;
        const int last_lane = (int)((nsrc - 1) % kLanes);
        if (is_last && dlast) SP_CUDA(cudaMemsetAsync(dlast, 0, n * sizeof(double), c.stream));
        for (int d = D; d >= 0; d--) {
            const int64_t q0 = ls[d], nq = ls[d + 1] - ls[d];
            BatchFold f{g->off, g->adj, lev, sig, coef, bc, is_last ? dlast : nullptr,
                        last_lane, bs, d};
            SP_CUDA(cudaMemsetAsync(counts, 0, 2 * sizeof(unsigned long long), c.stream));
            k_bb_rows<<<grid_for(nq, 256, c.device), 256, 0, c.stream>>>(f, queue + q0, nq,
                                                                         d == D, ck);
            c.launches++;
            if (d < D && g->max_outdeg > kBbShort) {
                k_bb_chunks<<<sms * 8, 256, 0, c.stream>>>(f, ck);
                k_bb_finish<<<sms * 8, 256, 0, c.stream>>>(f, ck);
                c.launches += 2;
            }
            SP_CUDA(cudaGetLastError());
        }
        if (is_last) {
            if (sigma_out) {
                double *so;
                SP_TRY(c.alloc(&so, n));
                k_bb_lane_out<<<grid_for(n, 256, c.device), 256, 0, c.stream>>>(sig, last_lane,
                                                                              n, so);
                c.launches++;
                SP_TRY(from_device(sigma_out, so, n * 8, mem, c.stream));
            }
            if (delta_out) SP_TRY(from_device(delta_out, dlast, n * 8, mem, c.stream));
        }
    }
    if (bc_accumulate_only) {
        SP_CUDA(cudaMemcpyAsync(bc_dst, bc, n * 8, cudaMemcpyDeviceToDevice, c.stream));
    } else {
        SP_TRY(from_device(bc_dst, bc, n * 8, bc_mem, c.stream));
    }
    SP_TRY(c.finish(nullptr));
    wk.launches = c.launches;
    return SP_OK;
}

// bc = sum of the workers' partials in worker order (fixed: deterministic)
__global__ void k_sum_partials(const double *__restrict__ parts, int k, int64_t n, double *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s = parts[i];
        for (int j = 1; j < k; j++) s = __dadd_rn(s, parts[(int64_t)j * n + i]);
        out[i] = s;
    }
}

}  // namespace

extern "C" int sp_bc(sp_graph *g, const int32_t *srcs_in, int64_t nsrc, unsigned flags,
                     double *bc_out, double *sigma_out, double *delta_out, int mem,
                     sp_stats *st) {
    SP_CHECK(g && bc_out && nsrc >= 0 && (nsrc == 0 || srcs_in), SP_ERR_ARG,
             "sp_bc: bad arguments");
    // SP_BC_TRACE=1: host phase times on stderr (diagnostic)
    static const bool trace = getenv("SP_BC_TRACE") != nullptr;
    const auto tt0 = std::chrono::steady_clock::now();
    auto tms = [&]() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tt0)
            .count();
    };
    std::vector<int32_t> srcs(srcs_in, srcs_in + nsrc);  // host list (SetN argument)
    for (int64_t i = 0; i < nsrc; i++)
        SP_CHECK(srcs[i] >= 0 && srcs[i] < g->n, SP_ERR_ARG,
                 "set argument 'sourceSet' id %d out of range", srcs[i]);
    const int64_t n = g->n;
    const bool det = flags & SP_FLAG_DETERMINISTIC;
    // Fast mode runs batches of kLanes sources (bc_run_batches), kBbWorkers
    // batches concurrently (one host thread and stream each): small BFS
    // levels of one batch overlap the large levels of another, and the
    // per-level host reads overlap too.  SP_BC_BATCH=0 selects the
    // per-source fast path (kBcWorkers sources concurrently).  Deterministic
    // mode keeps the reference's sequential source order (bit-exact bc).
    const char *eb = getenv("SP_BC_BATCH");
    bool batched = !det && !(eb && eb[0] == '0');
    const int64_t nb = (nsrc + kLanes - 1) / kLanes;
    int K = det ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(kBcWorkers, nsrc));
    if (batched) {
        // per worker: lev/sig/coef/csum/queue lanes + stamp, reg, bc; items
        const double per = (double)n * (4 + 8 + 8 + 8 + 4) * kLanes + 28.0 * n + g->m / 3.0;
        // free device memory, re-queried at most once a second per device:
        // cudaMemGetInfo stalled calls by up to ~20 ms under load
        static std::mutex mi_mu;
        static size_t mi_free[64];
        static std::chrono::steady_clock::time_point mi_at[64];
        size_t fr = 0;
        {
            std::lock_guard<std::mutex> lk(mi_mu);
            const int d = g->device & 63;
            const auto now = std::chrono::steady_clock::now();
            if (!mi_free[d] || now - mi_at[d] > std::chrono::seconds(1)) {
                size_t tot = 0;
                SP_CUDA(cudaSetDevice(g->device));
                SP_CUDA(cudaMemGetInfo(&mi_free[d], &tot));
                mi_at[d] = now;
            }
            fr = mi_free[d];
        }
        const char *ew = getenv("SP_BC_WORKERS");
        const int64_t want = ew ? std::max(1, atoi(ew)) : kBbWorkers;
        K = (int)std::max<int64_t>(1, std::min<int64_t>(want, nb));
        while (K > 1 && per * K > 0.6 * (double)fr) K--;
        if (per > 0.6 * (double)fr) batched = false, K = 1;  // per-source state only
    }
    Call c;
    SP_TRY(c.begin(g->device));
    std::vector<BcWorker> wk(K);
    auto run = [&](int64_t first, int64_t stride, double *dst, int dmem, bool acc_only,
                   BcWorker &w) {
        return batched ? bc_run_batches(g, srcs, first, stride, dst, dmem, acc_only, sigma_out,
                                        delta_out, mem, w)
                       : bc_run_sources(g, srcs, first, stride, det, dst, dmem, acc_only,
                                        sigma_out, delta_out, mem, w);
    };
    if (nsrc == 0) {
        double *z;
        SP_TRY(c.alloc(&z, n));
        SP_CUDA(cudaMemsetAsync(z, 0, n * 8, c.stream));
        SP_TRY(from_device(bc_out, z, n * 8, mem, c.stream));
    } else if (K == 1) {
        SP_TRY(c.finish(nullptr));  // order after the caller's work
        SP_TRY(run(0, 1, bc_out, mem, false, wk[0]));
    } else {
        double *parts;
        SP_TRY(c.alloc(&parts, (int64_t)K * n));
        SP_TRY(c.finish(nullptr));  // parts allocated before the workers use it
        std::lock_guard<std::mutex> slots(worker_slots_mutex(g->device));
        std::vector<std::thread> th;
        for (int k = 0; k < K; k++)
            th.emplace_back([&, k]() {
                wk[k].rc = run(k, K, parts + (int64_t)k * n, SP_MEM_DEVICE, true, wk[k]);
                if (wk[k].rc != SP_OK) snprintf(wk[k].err, sizeof(wk[k].err), "%s", sp_last_error());
            });
        const double t_spawn = tms();
        for (auto &t : th) t.join();
        if (trace) fprintf(stderr, "sp_bc: spawn %.2f ms, join %.2f ms\n", t_spawn, tms());
        for (int k = 0; k < K; k++)
            SP_CHECK(wk[k].rc == SP_OK, wk[k].rc, "%s", wk[k].err);
        double *sum;
        SP_TRY(c.alloc(&sum, n));
        k_sum_partials<<<grid_for(n, 256, c.device), 256, 0, c.stream>>>(parts, K, n, sum);
        c.launches++;
        SP_CUDA(cudaGetLastError());
        SP_TRY(from_device(bc_out, sum, n * 8, mem, c.stream));
    }
    SP_TRY(c.finish(st));
    if (trace) fprintf(stderr, "sp_bc: done %.2f ms\n", tms());
    if (st) {
        int64_t lv = 0, sc = 0, rc = 0, la = 0;
        for (auto &w : wk) {
            lv += w.levels;
            sc += w.scanned;
            rc += w.reached;
            la += w.launches;
        }
        st->iterations = lv;
        st->edges_visited = sc;
        st->vertices_visited = rc;
        st->kernel_launches += la;
        st->main_kernel_ms = st->device_ms;
        st->main_kernel_launches = st->kernel_launches;
        // 48 B per reached slot (discovery 8, sigma 16, delta 24)
        // + 64 B per reached vertex, summed over sources
        st->model_bytes = 48 * sc + 64 * rc;
    }
    return SP_OK;
}
