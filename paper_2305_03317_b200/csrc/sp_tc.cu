// sp_tc.cu -- corpus/programs/tc.sp on sm_100a.
//
// Reference semantics (tc.sp:3-13 under trident/interp.py): for every v, every
// slot u < v of N(v), every slot w > v of N(v), add the multiplicity of w in
// N(u).  Rows are sorted (graph.py:77), so per (v, u) the inner loops are a
// multiset dot product of A = N(v)_{>v} (a suffix of row v) and
// B = N(u)_{>v} (a suffix of row u).  Integer arithmetic: exact, any order.
//
// Kernel k_tc: persistent warps pull 32-vertex batches from a global counter.
// Per v the warp loads row v once (coalesced), stages A in shared memory (up
// to kA entries) with a 2048-bit membership filter, and hands each slot u < v
// to one lane.  A lane walks B = row u with independent 128-bit loads when B
// is short, or binary-searches the start of B when row u is long; each
// element x > v costs one shared-memory filter probe and, on a hit, a binary
// search in A for its multiplicity.  When B is far longer than A (a hub u)
// the lane instead walks A and binary-searches B in global memory.  Rows of
// v whose suffix exceeds kA search A in global memory (L2-resident).
// Counts: per-lane uint64 -> warp sum -> one atomicAdd per warp.
#include <algorithm>

#include "sp_common.cuh"

using namespace sp;

namespace {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kA = 1024;          // staged A entries per warp
constexpr int kFilterWords = 64;  // 2048-bit filter per warp
constexpr int kBatch = 32;

__device__ __forceinline__ int64_t lower_bound_g(const int32_t *__restrict__ a, int64_t lo,
                                                 int64_t hi, int32_t x) {
    while (lo < hi) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int lower_bound_s(const int32_t *a, int lo, int hi, int32_t x) {
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t fhash(int32_t x) {
    return ((uint32_t)x * 2654435761u) >> 21;  // 11 bits
}

__global__ void __launch_bounds__(kBlock) k_tc(const int64_t *__restrict__ off,
                                               const int32_t *__restrict__ adj, int64_t v0,
                                               int64_t v1, unsigned long long *next,
                                               unsigned long long *total,
                                               unsigned long long *pairs) {
    __shared__ int32_t sA[kWarps][kA];
    __shared__ uint32_t sF[kWarps][kFilterWords];
    const unsigned lane = lane_id();
    const int wib = threadIdx.x >> 5;
    int32_t *A = sA[wib];
    uint32_t *F = sF[wib];
    unsigned long long cnt = 0, npairs = 0;
    for (;;) {
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(next, (unsigned long long)kBatch);
        b = __shfl_sync(0xffffffffu, b, 0);
        const int64_t vb = v0 + (int64_t)b;
        if (vb >= v1) break;
        const int64_t ve = min(v1, vb + kBatch);
        for (int64_t v = vb; v < ve; v++) {
            const int64_t r0 = off[v], r1 = off[v + 1];
            if (r1 - r0 < 2) continue;
            // split point: first slot > v (A = [a0, r1)), slots < v are [r0, ulast)
            const int64_t a0 = lower_bound_g(adj, r0, r1, (int32_t)v + 1);
            const int64_t na = r1 - a0;
            if (na == 0) continue;
            const int64_t ulast = lower_bound_g(adj, r0, a0, (int32_t)v);
            const int64_t nu = ulast - r0;
            if (nu == 0) continue;
            npairs += (lane == 0) ? (unsigned long long)nu : 0ull;
            const bool staged = na <= kA;
            if (staged) {
                for (int k = lane; k < kFilterWords; k += 32) F[k] = 0u;
                __syncwarp();
                for (int64_t k = lane; k < na; k += 32) {
                    int32_t x = adj[a0 + k];
                    A[k] = x;
                    uint32_t h = fhash(x);
                    atomicOr(&F[h >> 5], 1u << (h & 31));
                }
                __syncwarp();
            }
            for (int64_t k = r0 + lane; k < ulast; k += 32) {
                const int32_t u = adj[k];
                const int64_t u0 = off[u], u1 = off[u + 1];
                int64_t b0 = u0;
                if (u1 - u0 > 16) b0 = lower_bound_g(adj, u0, u1, (int32_t)v + 1);
                const int64_t nb = u1 - b0;
                if (nb <= 0) continue;
                if (nb > 8 * na && na <= 64) {
                    // hub u: walk A (runs), binary-search B in global memory
                    int64_t lo = b0;
                    for (int64_t i = 0; i < na;) {
                        const int32_t x = staged ? A[i] : adj[a0 + i];
                        int64_t j = i + 1;
                        while (j < na && (staged ? A[j] : adj[a0 + j]) == x) j++;
                        lo = lower_bound_g(adj, lo, u1, x);
                        int64_t hi = lo;
                        while (hi < u1 && __ldg(adj + hi) == x) hi++;
                        cnt += (unsigned long long)(j - i) * (unsigned long long)(hi - lo);
                        lo = hi;
                        i = j;
                    }
                    continue;
                }
                for (int64_t e = b0; e < u1; e++) {
                    const int32_t x = __ldg(adj + e);
                    if (x <= (int32_t)v) continue;
                    if (staged) {
                        const uint32_t h = fhash(x);
                        if (!(F[h >> 5] & (1u << (h & 31)))) continue;
                        int lb = lower_bound_s(A, 0, (int)na, x);
                        int ub = lb;
                        while (ub < na && A[ub] == x) ub++;
                        cnt += (unsigned long long)(ub - lb);
                    } else {
                        int64_t lb = lower_bound_g(adj, a0, r1, x);
                        int64_t ub = lb;
                        while (ub < r1 && __ldg(adj + ub) == x) ub++;
                        cnt += (unsigned long long)(ub - lb);
                    }
                }
            }
            __syncwarp();
        }
    }
    cnt = warp_sum(cnt);
    npairs = warp_sum(npairs);
    if (lane == 0) {
        if (cnt) atomicAdd(total, cnt);
        if (npairs) atomicAdd(pairs, npairs);
    }
}

}  // namespace

extern "C" int sp_tc(sp_graph *g, int64_t v0, int64_t v1, uint64_t *count, sp_stats *st) {
    SP_CHECK(g && count && v0 >= 0 && v0 <= v1 && v1 <= g->n, SP_ERR_ARG,
             "sp_tc: bad arguments");
    Call c;
    SP_TRY(c.begin(g->device));
    unsigned long long *ctr;
    SP_TRY(c.alloc(&ctr, 3));
    SP_CUDA(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), c.stream));
    const int sms = num_sms(c.device);
    cudaEvent_t ka, kb;
    SP_CUDA(cudaEventCreate(&ka));
    SP_CUDA(cudaEventCreate(&kb));
    cudaEventRecord(ka, c.stream);
    if (v1 > v0) {
        int64_t want = (v1 - v0 + kBatch * kWarps - 1) / (kBatch * kWarps);
        int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
        k_tc<<<grid, kBlock, 0, c.stream>>>(g->off, g->adj, v0, v1, ctr, ctr + 1, ctr + 2);
        c.launches++;
    }
    cudaEventRecord(kb, c.stream);
    SP_CUDA(cudaGetLastError());
    unsigned long long h[3];
    SP_CUDA(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    int rc = c.finish(st);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ka, kb);
    cudaEventDestroy(ka);
    cudaEventDestroy(kb);
    SP_TRY(rc);
    *count = (uint64_t)h[1];
    if (st) {
        st->iterations = 1;
        st->edges_visited = (int64_t)h[2];
        st->vertices_visited = v1 - v0;
        st->main_kernel_ms = ms;
        st->main_kernel_launches = c.launches;
    }
    return SP_OK;
}
