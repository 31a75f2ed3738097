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
#include <vector>

#include "sp_expand.cuh"
#include "sp_fold.cuh"

using namespace sp;

namespace {

constexpr int64_t kBcHub = 8192;  // rows longer than this take the CTA fold

struct DiscoverOp {
    using Payload = int;
    using Probe = int;  // level[x]
    int32_t *__restrict__ level;
    int next;
    __device__ __forceinline__ int payload(int32_t) const { return 0; }
    __device__ __forceinline__ int probe(int64_t, int32_t x) const { return __ldcg(level + x); }
    __device__ __forceinline__ bool apply(int, int64_t, int32_t x, int lx) const {
        if (lx != -1) return false;
        return atomicCAS(level + x, -1, next) == -1;
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
    __device__ __forceinline__ int probe(int64_t, int32_t x) const { return __ldcg(level + x); }
    __device__ __forceinline__ bool apply(double sv, int64_t, int32_t x, int lx) const {
        if (lx != -1 && lx != next) return false;
        bool won = false;
        if (lx == -1) {
            const int old = atomicCAS(level + x, -1, next);
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
        return __ldg(level + u) == parent_level ? sigma[u] : 0.0;
    }
    __device__ __forceinline__ void finish(int32_t v, double s) const { sigma[v] = s; }
};

struct DeltaFold {  // bc.sp:14-19 over CSR slots
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
        if (__ldg(level + w) != child_level) return 0.0;
        return __dmul_rn(__ddiv_rn(sv, sigma[w]), __dadd_rn(1.0, delta[w]));
    }
    __device__ __forceinline__ void finish(int32_t v, double s) const {
        delta[v] = s;
        if (v != src) bc[v] = __dadd_rn(bc[v], __ddiv_rn(s, 2.0));
    }
};

__global__ void k_root(int32_t *level, double *sigma, int32_t *queue, int32_t s) {
    level[s] = 0;
    sigma[s] = 1.0;
    queue[0] = s;
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
    Call c;
    SP_TRY(c.begin(g->device));
    const int64_t n = g->n;
    const int sms = num_sms(c.device);
    const bool det = flags & SP_FLAG_DETERMINISTIC;
    int32_t *level, *queue, *hubs, *reg_v, *reg_nch, *item_reg;
    int64_t *reg_base;
    double *csum;
    double *sigma, *delta, *bc;
    uint2 *chunks;
    ExpandCounters *cnt;
    unsigned long long *nhubs;
    SP_TRY(c.alloc(&level, n));
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
    SP_CUDA(cudaMemsetAsync(bc, 0, n * sizeof(double), c.stream));
    SP_CUDA(cudaMemsetAsync(sigma, 0, n * sizeof(double), c.stream));
    SP_CUDA(cudaMemsetAsync(delta, 0, n * sizeof(double), c.stream));
    ExpandCounters *hc = nullptr;
    SP_TRY(c.host_as(&hc));
    const bool big_out = g->max_outdeg > kSplit;
    int64_t levels_total = 0, scanned_total = 0, reached_total = 0;
    std::vector<int64_t> ls;
    for (int64_t si = 0; si < nsrc; si++) {
        const int32_t s = srcs[si];
        SP_CUDA(cudaMemsetAsync(level, 0xFF, n * sizeof(int32_t), c.stream));
        if (si > 0) {
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
            scanned_total += (int64_t)hc->scanned;
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
        levels_total += nlev;
        reached_total += ls.back();
        for (int L = nlev - 2; L >= 0; L--) {
            DeltaFold df{g->adj, level, sigma, delta, bc, L + 1, s};
            launch_fold(df, g->off, queue + ls[L], ls[L + 1] - ls[L], kBcHub, fl, det,
                        g->max_outdeg, sms, c.stream, &c.launches);
        }
        SP_CUDA(cudaGetLastError());
    }
    SP_TRY(from_device(bc_out, bc, n * 8, mem, c.stream));
    if (sigma_out) SP_TRY(from_device(sigma_out, sigma, n * 8, mem, c.stream));
    if (delta_out) SP_TRY(from_device(delta_out, delta, n * 8, mem, c.stream));
    SP_TRY(c.finish(st));
    if (st) {
        st->iterations = levels_total;
        st->edges_visited = scanned_total;
        st->vertices_visited = reached_total;
        st->main_kernel_ms = st->device_ms;
        st->main_kernel_launches = st->kernel_launches;
        // 48 B per reached slot (discovery 8, sigma 16, delta 24)
        // + 64 B per reached vertex, summed over sources
        st->model_bytes = 48 * scanned_total + 64 * reached_total;
    }
    return SP_OK;
}
