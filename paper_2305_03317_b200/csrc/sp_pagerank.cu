// sp_pagerank.cu -- corpus/programs/pr.sp on sm_100a.
//
// Reference semantics (pr.sp:10-29 under trident/interp.py):
//   per iteration, for every v: sum = left fold over the reverse-CSR row of v
//   (ascending source id, then eid; graph.py:92) of u.rank / outdeg(u);
//   newRank = (1-d)/n + d*sum; diff = max |newRank - rank|; rank_nxt = newRank;
//   then rank = rank_nxt; iter++; stop when diff < eps || iter >= maxIter.
//
// Device layout: contrib[2][n] f64 (contrib[u] = rank[u]/outdeg(u), written
// by the previous iteration -- the same IEEE division the interpreter does
// per slot), rank[n] f64 updated in place (each vertex reads only its own
// rank), outdeg int32[n], reverse CSR (roff int64, radj int32), and one
// f64 diff slot per iteration (max via atomicMax on the bit pattern of a
// non-negative double: exact and order-independent).
//
// Kernel k_pull (one launch per iteration): a warp owns a tile of 32
// consecutive vertices, whose rows form ONE contiguous slab of radj.  The
// warp streams that slab in 128-slot chunks: coalesced radj loads, 4
// independent contrib gathers per lane in flight, values staged in shared
// memory; then every lane folds the part of ITS row inside the chunk,
// sequentially, in CSR order -> bit-identical to the interpreter's left fold.
// Rows with in-degree > kHub (fast mode only) are excluded from the slab and
// summed by k_hub (one CTA per hub, fixed-shape tree: deterministic run to
// run, within ~1e-16 relative of the left fold).  SP_FLAG_DETERMINISTIC
// disables the hub path, making every vertex bit-exact.
// No FMA contraction anywhere: __dadd_rn/__dmul_rn are used explicitly.
#include <algorithm>

#include "sp_common.cuh"

using namespace sp;

namespace {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kChunk = 128;  // slab slots staged per warp per step
constexpr int kHub = 4096;   // must match sp_graph.cu kHubIn
constexpr int kHubBlock = 512;

__global__ void k_init(double *rank, double *contrib, const int32_t *__restrict__ outdeg,
                       int64_t v0, int64_t v1, double r0) {
    for (int64_t x = v0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < v1;
         x += (int64_t)gridDim.x * blockDim.x) {
        rank[x - v0] = r0;
        int d = outdeg[x];
        contrib[x - v0] = d > 0 ? __ddiv_rn(r0, (double)d) : 0.0;
    }
}

// Fixed-shape CTA reduction of one hub row.
__global__ void __launch_bounds__(kHubBlock) k_hub(const int64_t *__restrict__ roff,
                                                   const int32_t *__restrict__ radj,
                                                   const double *__restrict__ contrib,
                                                   const int32_t *__restrict__ hubs, int64_t nhubs,
                                                   int64_t v0, int64_t v1,
                                                   double *__restrict__ hubsum) {
    __shared__ double red[kHubBlock / 32];
    for (int64_t h = blockIdx.x; h < nhubs; h += gridDim.x) {
        int32_t v = hubs[h];
        if (v < v0 || v >= v1) continue;
        int64_t b = roff[v], e = roff[v + 1];
        double s = 0.0;
        for (int64_t k = b + threadIdx.x; k < e; k += kHubBlock) s = __dadd_rn(s, contrib[radj[k]]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x < 32) {
            double t = threadIdx.x < kHubBlock / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, o));
            if (threadIdx.x == 0) hubsum[v] = t;
        }
        __syncthreads();
    }
}

// One PageRank iteration for vertices [v0, v1).
//   contrib_in: full n-array (global ids); rank/contrib_out: local, index v-v0.
template <bool kUseHubs>
__global__ void __launch_bounds__(kBlock) k_pull(
    const int64_t *__restrict__ roff, const int32_t *__restrict__ radj,
    const int32_t *__restrict__ outdeg, const double *__restrict__ contrib_in,
    const double *__restrict__ hubsum, double *__restrict__ rank,
    double *__restrict__ contrib_out, int64_t v0, int64_t v1, double base, double damping,
    double *diff_slot) {
    __shared__ double stage[kWarps][kChunk];
    __shared__ double red[kWarps];
    const unsigned lane = lane_id();
    const int wib = threadIdx.x >> 5;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double dmax = 0.0;
    double *buf = stage[wib];
    for (int64_t t0 = v0 + warp * 32; t0 < v1; t0 += nwarps * 32) {
        const int64_t v = t0 + lane;
        const bool live = v < v1;
        int64_t rs = 0, re = 0;
        if (live) {
            rs = roff[v];
            re = roff[v + 1];
        }
        bool hub = kUseHubs && live && (re - rs) > kHub;
        int64_t deg = hub ? 0 : re - rs;
        // positions of this lane's row inside the warp's flattened slab
        int64_t incl = deg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t tt = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += tt;
        }
        const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
        const int64_t excl = incl - deg;
        // Without hub rows the tile's slab is radj[roff[t0] .. roff[t0+32]):
        // slot p is simply radj[sb + p].  Tiles holding a hub row (fast mode,
        // rare) map slots to rows by a binary search over the lane prefix.
        const unsigned hubmask = __ballot_sync(0xffffffffu, hub);
        const int64_t sb = __shfl_sync(0xffffffffu, rs, 0);
        double sum = 0.0;
        for (int64_t p0 = 0; p0 < total; p0 += kChunk) {
#pragma unroll
            for (int j = 0; j < kChunk / 32; j++) {
                const int64_t p = p0 + j * 32 + lane;
                int64_t idx = sb + p;
                if (kUseHubs && hubmask) {
                    int lo = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        int cand = lo + step;
                        int64_t ex = __shfl_sync(0xffffffffu, excl, cand & 31);
                        if (cand < 32 && ex <= p) lo = cand;
                    }
                    int64_t ex = __shfl_sync(0xffffffffu, excl, lo);
                    int64_t b0 = __shfl_sync(0xffffffffu, rs, lo);
                    idx = b0 + (p - ex);
                }
                double val = 0.0;
                if (p < total) val = contrib_in[radj[idx]];
                buf[j * 32 + lane] = val;
            }
            __syncwarp();
            // sequential left fold of this lane's slice of the chunk
            int64_t a = max(excl, p0), b = min(excl + deg, p0 + (int64_t)kChunk);
            for (int64_t p = a; p < b; p++) sum = __dadd_rn(sum, buf[p - p0]);
            __syncwarp();
        }
        if (live) {
            if (hub) sum = hubsum[v];
            double nr = __dadd_rn(base, __dmul_rn(damping, sum));
            double r = rank[v - v0];
            double d = __dsub_rn(nr, r);
            if (d < 0.0) d = __dsub_rn(0.0, d);
            dmax = fmax(dmax, d);
            rank[v - v0] = nr;
            int od = outdeg[v];
            contrib_out[v - v0] = od > 0 ? __ddiv_rn(nr, (double)od) : 0.0;
        }
    }
    dmax = warp_max(dmax);
    if (lane == 0) red[wib] = dmax;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = threadIdx.x < kWarps ? red[threadIdx.x] : 0.0;
        t = warp_max(t);
        if (threadIdx.x == 0) atomic_max_nonneg(diff_slot, t);
    }
}

int launch_iteration(sp_graph *g, Call &c, bool use_hubs, int64_t v0, int64_t v1, double damping,
                     const double *cin, double *rank, double *cout, double *hubsum,
                     double *diff_slot, cudaEvent_t ka, cudaEvent_t kb) {
    const int dev = c.device;
    const double base = (1.0 - damping) / (double)g->n;  // pr.sp:17, no FMA on host either
    if (use_hubs) {
        int gh = (int)std::min<int64_t>(g->nhubs_in, (int64_t)num_sms(dev) * 4);
        k_hub<<<gh, kHubBlock, 0, c.stream>>>(g->roff, g->radj, cin, g->hubs_in, g->nhubs_in, v0,
                                              v1, hubsum);
        c.launches++;
    }
    int64_t tiles = (v1 - v0 + 31) / 32;
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>((tiles + kWarps - 1) / kWarps,
                                                           (int64_t)num_sms(dev) * 8));
    if (ka) cudaEventRecord(ka, c.stream);
    if (use_hubs)
        k_pull<true><<<grid, kBlock, 0, c.stream>>>(g->roff, g->radj, g->outdeg, cin, hubsum, rank,
                                                    cout, v0, v1, base, damping, diff_slot);
    else
        k_pull<false><<<grid, kBlock, 0, c.stream>>>(g->roff, g->radj, g->outdeg, cin, hubsum, rank,
                                                     cout, v0, v1, base, damping, diff_slot);
    if (kb) cudaEventRecord(kb, c.stream);
    c.launches++;
    SP_CUDA(cudaGetLastError());
    return SP_OK;
}

}  // namespace

extern "C" int sp_pagerank(sp_graph *g, double damping, double epsilon, int64_t max_iter,
                           int64_t cap, unsigned flags, double *rank_out, int mem,
                           int64_t *iter_out, double *diff_out, int64_t *iters_out,
                           sp_iter_cb cb, void *user, sp_stats *st) {
    SP_CHECK(g && (rank_out || g->n == 0), SP_ERR_ARG, "sp_pagerank: bad arguments");
    Call c;
    SP_TRY(c.begin(g->device));
    const int64_t n = g->n;
    const bool use_hubs = !(flags & SP_FLAG_DETERMINISTIC) && g->nhubs_in > 0;
    double *rank, *ca, *cb2, *hubsum = nullptr, *diffs;
    SP_TRY(c.alloc(&rank, n));
    SP_TRY(c.alloc(&ca, n));
    SP_TRY(c.alloc(&cb2, n));
    if (use_hubs) SP_TRY(c.alloc(&hubsum, n));
    const int64_t kSlots = 1024;  // diff slots, recycled in a ring
    SP_TRY(c.alloc(&diffs, kSlots));
    SP_CUDA(cudaMemsetAsync(diffs, 0, kSlots * sizeof(double), c.stream));
    double *hdiff = nullptr;
    SP_CUDA(cudaMallocHost(&hdiff, sizeof(double)));
    struct HostFree { double *p; ~HostFree() { if (p) cudaFreeHost(p); } } hf{hdiff};
    const double r0 = n ? 1.0 / (double)n : 0.0;  // pr.sp:6
    if (n) {
        k_init<<<grid_for(n, 256, c.device), 256, 0, c.stream>>>(rank, ca, g->outdeg, 0, n, r0);
        c.launches++;
    }
    cudaEvent_t ka, kb;
    SP_CUDA(cudaEventCreate(&ka));
    SP_CUDA(cudaEventCreate(&kb));
    float kernel_ms = 0.f;
    int64_t iter = 0, iters = 0;
    double diff = 0.0;
    int rc = SP_OK;
    for (;;) {
        double *slot = diffs + (iters % kSlots);
        if (n) {
            rc = launch_iteration(g, c, use_hubs, 0, n, damping, ca, rank, cb2, hubsum, slot, ka, kb);
            if (rc) break;
            SP_CUDA(cudaMemcpyAsync(hdiff, slot, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
            SP_CUDA(cudaMemsetAsync(diffs + ((iters + 1) % kSlots), 0, sizeof(double), c.stream));
            SP_CUDA(cudaStreamSynchronize(c.stream));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ka, kb);
            kernel_ms += ms;
            diff = *hdiff;
            std::swap(ca, cb2);
        } else {
            diff = 0.0;
        }
        iter = iter + 1;
        iters++;
        if (cb && cb(iters, user)) {
            set_error("aborted by the fixedPoint iteration callback");
            rc = SP_ERR_ABORTED;
            break;
        }
        if (diff < epsilon || iter >= max_iter) break;  // pr.sp:10
        if (iters >= cap) {
            set_error("fixedPoint 'converged' did not converge within %lld iterations",
                      (long long)cap);
            rc = SP_ERR_NONCONV;
            break;
        }
    }
    cudaEventDestroy(ka);
    cudaEventDestroy(kb);
    if (rc == SP_OK && n) SP_TRY(from_device(rank_out, rank, n * 8, mem, c.stream));
    SP_TRY(c.finish(st));
    if (iter_out) *iter_out = iter;
    if (diff_out) *diff_out = diff;
    if (iters_out) *iters_out = iters;
    if (st) {
        st->iterations = iters;
        st->edges_visited = iters * g->m;
        st->vertices_visited = iters * n;
        st->main_kernel_ms = kernel_ms;
        st->main_kernel_launches = iters;
    }
    return rc;
}

extern "C" int sp_pagerank_block_init(sp_graph *g, int64_t v0, int64_t v1, double *rank_local,
                                      double *contrib_out) {
    SP_CHECK(g && v0 >= 0 && v0 <= v1 && v1 <= g->n, SP_ERR_ARG, "bad vertex block");
    SP_CUDA(cudaSetDevice(g->device));
    if (v1 > v0) {
        k_init<<<grid_for(v1 - v0, 256, g->device), 256>>>(rank_local, contrib_out, g->outdeg, v0,
                                                           v1, 1.0 / (double)g->n);
        SP_CUDA(cudaGetLastError());
    }
    SP_CUDA(cudaDeviceSynchronize());
    return SP_OK;
}

extern "C" int sp_pagerank_block_step(sp_graph *g, int64_t v0, int64_t v1, double damping,
                                      const double *contrib_in, double *rank_local,
                                      double *contrib_out, double *diff, unsigned flags,
                                      sp_stats *st) {
    SP_CHECK(g && v0 >= 0 && v0 <= v1 && v1 <= g->n && diff, SP_ERR_ARG, "bad vertex block");
    Call c;
    SP_TRY(c.begin(g->device));
    const bool use_hubs = !(flags & SP_FLAG_DETERMINISTIC) && g->nhubs_in > 0;
    double *hubsum = nullptr, *slot;
    if (use_hubs) SP_TRY(c.alloc(&hubsum, g->n));
    SP_TRY(c.alloc(&slot, 1));
    SP_CUDA(cudaMemsetAsync(slot, 0, sizeof(double), c.stream));
    if (v1 > v0)
        SP_TRY(launch_iteration(g, c, use_hubs, v0, v1, damping, contrib_in, rank_local,
                                contrib_out, hubsum, slot, nullptr, nullptr));
    SP_CUDA(cudaMemcpyAsync(diff, slot, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    SP_TRY(c.finish(st));
    return SP_OK;
}
