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
#include <thread>
#include <vector>

#include "sp_expand.cuh"
#include "sp_fold.cuh"

using namespace sp;

namespace {

constexpr int64_t kBcHub = 8192;  // rows longer than this take the CTA fold
constexpr int kBcWorkers = 4;     // concurrent sources (host threads/streams), fast mode

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
    __device__ __forceinline__ double term(double, int64_t k) const {
        const int32_t u = radj[k];
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
    __device__ __forceinline__ double term(double sv, int64_t e) const {
        const int32_t w = adj[e];
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
    __device__ __forceinline__ double term(double sv, int64_t e) const {
        const int32_t w = __ldcs(adj + e);
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
    int64_t levels = 0, scanned = 0, reached = 0, launches = 0;
    int rc = SP_OK;
    char err[512] = "";
};

int bc_run_sources(sp_graph *g, const std::vector<int32_t> &srcs, int64_t first, int64_t stride,
                   bool det, double *bc_dst, int bc_mem, bool bc_accumulate_only,
                   double *sigma_out, double *delta_out, int mem, BcWorker &wk) {
    Call c;
    SP_TRY(c.begin(g->device));
    const int64_t n = g->n;
    const int64_t nsrc = (int64_t)srcs.size();
    const int sms = num_sms(c.device);
    int32_t *level, *queue, *hubs, *reg_v, *reg_nch, *item_reg;
    int64_t *reg_base;
    double *csum;
    double *sigma, *delta, *bc;
    uint2 *chunks;
    ExpandCounters *cnt;
    unsigned long long *nhubs;
    SP_TRY(c.alloc(&level, kVs * n));  // 16-byte (level, coef) records
    SP_TRY(c.alloc(&queue, n));
    SP_TRY(c.alloc(&hubs, n));
    const int64_t ccap = fold_chunk_capacity(g->m);
    SP_TRY(c.alloc(&reg_v, n));
    SP_TRY(c.alloc(&reg_nch, n));
    SP_TRY(c.alloc(&reg_base, n));
    SP_TRY(c.alloc(&item_reg, ccap));
    SP_TRY(c.alloc(&csum, ccap));
    SP_TRY(c.alloc(&sigma, n));
    SP_TRY(c.alloc(&delta, n));
    SP_TRY(c.alloc(&bc, n));
    SP_TRY(c.alloc(&chunks, expand_chunk_capacity(g->m)));
    SP_TRY(c.alloc(&cnt, 1));
    SP_TRY(c.alloc(&nhubs, 3));
    const FoldLists fl{hubs, nhubs, FoldChunks{reg_v, reg_base, reg_nch, item_reg, csum, nullptr}};
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
    std::vector<int32_t> srcs(srcs_in, srcs_in + nsrc);  // host list (SetN argument)
    for (int64_t i = 0; i < nsrc; i++)
        SP_CHECK(srcs[i] >= 0 && srcs[i] < g->n, SP_ERR_ARG,
                 "set argument 'sourceSet' id %d out of range", srcs[i]);
    const int64_t n = g->n;
    const bool det = flags & SP_FLAG_DETERMINISTIC;
    // Fast mode runs kBcWorkers sources concurrently (one host thread and
    // stream each): small BFS levels of one source overlap the large levels
    // of another, and the per-level host reads overlap too.  Deterministic
    // mode keeps the reference's sequential source order (bit-exact bc).
    const int K = det ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(kBcWorkers, nsrc));
    Call c;
    SP_TRY(c.begin(g->device));
    std::vector<BcWorker> wk(K);
    if (nsrc == 0) {
        double *z;
        SP_TRY(c.alloc(&z, n));
        SP_CUDA(cudaMemsetAsync(z, 0, n * 8, c.stream));
        SP_TRY(from_device(bc_out, z, n * 8, mem, c.stream));
    } else if (K == 1) {
        SP_TRY(c.finish(nullptr));  // order after the caller's work
        SP_TRY(bc_run_sources(g, srcs, 0, 1, det, bc_out, mem, false, sigma_out, delta_out, mem,
                              wk[0]));
    } else {
        double *parts;
        SP_TRY(c.alloc(&parts, (int64_t)K * n));
        SP_TRY(c.finish(nullptr));  // parts allocated before the workers use it
        std::vector<std::thread> th;
        for (int k = 0; k < K; k++)
            th.emplace_back([&, k]() {
                wk[k].rc = bc_run_sources(g, srcs, k, K, det, parts + (int64_t)k * n,
                                          SP_MEM_DEVICE, true, sigma_out, delta_out, mem, wk[k]);
                if (wk[k].rc != SP_OK) snprintf(wk[k].err, sizeof(wk[k].err), "%s", sp_last_error());
            });
        for (auto &t : th) t.join();
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
