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
// Candidates >= INT_MAX never win (interp.py:11-14).
#include <algorithm>

#include "sp_expand.cuh"

using namespace sp;

namespace {

constexpr int kBlock = 256;

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
        return Probe{__ldg(weff + e), __ldcg(dist + x)};
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
        const int old = atomicMin(dist + x, c);
        return c < old && atomicExch(enq + x, it) != it;
    }
};

__global__ void k_init(int32_t *dist, int32_t *enq, int64_t n, int32_t src, int32_t *q) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        dist[x] = x == src ? 0 : kIntMax;
        enq[x] = x == src ? 0 : -1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) q[0] = src;
}

}  // namespace

extern "C" int sp_sssp(sp_graph *g, int32_t src, int64_t cap, int32_t *dist_out, int mem,
                       int64_t *iters_out, sp_iter_cb cb, void *user, sp_stats *st) {
    SP_CHECK(g && dist_out, SP_ERR_ARG, "sp_sssp: bad arguments");
    SP_CHECK(src >= 0 && src < g->n, SP_ERR_ARG, "node argument 'src'=%d out of range", src);
    Call c;
    SP_TRY(c.begin(g->device));
    SP_TRY(ensure_weff(g, c));
    const int64_t n = g->n;
    int32_t *dist, *enq, *qa, *qb;
    uint2 *chunks;
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
    k_init<<<grid_for(n, kBlock, dev), kBlock, 0, c.stream>>>(dist, enq, n, src, qa);
    c.launches++;
    int64_t nq = 1, iters = 0, relaxed = 0, frontier_sum = 0;
    int rc = SP_OK;
    cudaEvent_t ka, kb;
    SP_CUDA(cudaEventCreate(&ka));
    SP_CUDA(cudaEventCreate(&kb));
    float kernel_ms = 0.f;
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
    if (rc == SP_OK || rc == SP_ERR_NONCONV) SP_TRY(from_device(dist_out, dist, n * 4, mem, c.stream));
    SP_TRY(c.finish(st));
    if (iters_out) *iters_out = iters;
    if (st) {
        st->iterations = iters;
        st->edges_visited = relaxed;
        st->vertices_visited = frontier_sum;
        st->main_kernel_ms = kernel_ms;
        st->main_kernel_launches = iters;
    }
    return rc;
}

// ---- block-partitioned supersteps (multi-GPU, graph.py:226-249 ownership)
namespace {

// Relaxation without a next-frontier queue: ownership decides the frontier
// after the exchange (k_block_frontier), not the relaxing rank.
struct RelaxNoPushOp {
    using Payload = int;
    using Probe = RelaxOp::Probe;
    int32_t *__restrict__ dist;
    const int32_t *__restrict__ weff;
    unsigned long long *overflow;
    __device__ __forceinline__ int payload(int32_t v) const { return __ldcg(dist + v); }
    __device__ __forceinline__ Probe probe(int64_t e, int32_t x) const {
        return Probe{__ldg(weff + e), __ldcg(dist + x)};
    }
    __device__ __forceinline__ bool apply(int dv, int64_t, int32_t x, Probe p) const {
        const int64_t cand = (int64_t)dv + (int64_t)p.w;
        if (cand >= (int64_t)kIntMax) return false;
        if (cand < (int64_t)(-2147483647 - 1)) {
            atomicAdd(overflow, 1ull);
            return false;
        }
        if ((int)cand < p.dx) atomicMin(dist + x, (int)cand);
        return false;
    }
};

// F = {v in [v0, v1): dist[v] < last[v]}; last[v] = dist[v] for v in F.
__global__ void k_block_frontier(const int32_t *__restrict__ dist, int32_t *__restrict__ last,
                                 int64_t v0, int64_t v1, int32_t *q, unsigned long long *cnt) {
    for (int64_t b = v0 + blockIdx.x * (int64_t)blockDim.x; b < v1;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = b + threadIdx.x;
        int32_t d = 0;
        bool in = false;
        if (v < v1) {
            d = dist[v];
            in = d < last[v];
        }
        const int64_t slot = warp_append(in, cnt);
        if (in) {
            q[slot] = (int32_t)v;
            last[v] = d;
        }
    }
}

__global__ void k_block_init(int32_t *dist, int32_t *last, int64_t n, int32_t src) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        dist[x] = x == src ? 0 : kIntMax;
        last[x] = kIntMax;
    }
}

}  // namespace

extern "C" int sp_sssp_block_init(sp_graph *g, int32_t src, int32_t *dist, int32_t *last) {
    SP_CHECK(g && dist && last, SP_ERR_ARG, "sp_sssp_block_init: bad arguments");
    SP_CHECK(src >= 0 && src < g->n, SP_ERR_ARG, "node argument 'src'=%d out of range", src);
    Call c;
    SP_TRY(c.begin(g->device));
    SP_TRY(ensure_weff(g, c));
    k_block_init<<<grid_for(g->n, kBlock, c.device), kBlock, 0, c.stream>>>(dist, last, g->n, src);
    c.launches++;
    SP_CUDA(cudaGetLastError());
    return c.finish(nullptr);
}

extern "C" int sp_sssp_block_step(sp_graph *g, int64_t v0, int64_t v1, int32_t *dist,
                                  int32_t *last, int64_t *frontier, int64_t *relaxed) {
    SP_CHECK(g && dist && last && v0 >= 0 && v0 <= v1 && v1 <= g->n, SP_ERR_ARG,
             "sp_sssp_block_step: bad arguments");
    Call c;
    SP_TRY(c.begin(g->device));
    SP_TRY(ensure_weff(g, c));
    const int64_t nb = std::max<int64_t>(1, v1 - v0);
    int32_t *q, *qn;
    uint2 *chunks;
    ExpandCounters *cnt;
    SP_TRY(c.alloc(&q, nb));
    SP_TRY(c.alloc(&qn, 1));
    SP_TRY(c.alloc(&chunks, expand_chunk_capacity(g->m)));
    SP_TRY(c.alloc(&cnt, 2));
    SP_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(ExpandCounters), c.stream));
    ExpandCounters *h;
    SP_TRY(c.host_as(&h));
    if (v1 > v0) {
        k_block_frontier<<<grid_for(v1 - v0, kBlock, c.device), kBlock, 0, c.stream>>>(
            dist, last, v0, v1, q, &cnt[1].next_size);
        c.launches++;
    }
    SP_CUDA(cudaMemcpyAsync(h, &cnt[1], sizeof(ExpandCounters), cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    const int64_t nq = (int64_t)h->next_size;
    if (nq) {
        RelaxNoPushOp op{dist, g->weff, &cnt->flag};
        launch_expand(op, g->off, g->adj, q, nq, qn, chunks, cnt, num_sms(c.device),
                      g->max_outdeg > kSplit, c.stream, &c.launches);
        SP_CUDA(cudaGetLastError());
        SP_CUDA(cudaMemcpyAsync(h, cnt, sizeof(ExpandCounters), cudaMemcpyDeviceToHost, c.stream));
    } else {
        h->scanned = 0;
        h->flag = 0;
    }
    SP_TRY(c.finish(nullptr));
    SP_CHECK(!h->flag, SP_ERR_OVERFLOW, "SSSP distance left the int32 range (negative weights)");
    if (frontier) *frontier = nq;
    if (relaxed) *relaxed = (int64_t)h->scanned;
    return SP_OK;
}
