// sp_tc.cu -- corpus/programs/tc.sp on sm_100a.
//
// Reference semantics (tc.sp:3-13 under trident/interp.py): for every v, every
// slot u < v of N(v), every slot w > v of N(v), add the multiplicity of w in
// N(u).  Integer arithmetic: exact in any order.  For a triangle a < b < c
// with slot multiplicities m_ab, m_bc, m_ac the program adds m_ab*m_bc*m_ac
// exactly once (v = b, u = a, w = c); self-loops never take part (u < v < w).
//
// Undirected graphs (mirror slots: mult(b in N(a)) == mult(a in N(b))): that
// product is symmetric in the three vertices, so any total order of the
// vertices counts the same triangles with the same weights.  The backend
// orients every edge from the lower to the higher rank, rank(v) = (degree v,
// v), which bounds every out-row by sqrt(2m) whatever the skew:
//   upper CSR  (ustart8, ulen, uadj): row a = the neighbours x of a with
//              rank(x) > rank(a), ascending id, duplicates kept, each row
//              padded to whole 32-byte sectors; uinfo[e] = (row start, row
//              length) of the vertex slot e points to, so a row is found
//              without a dependent random offset load; built once per graph
//              on the device (count -> scan -> fill -> info) and cached;
//   count    = sum over slots b of N+(a), over slots x of N+(b), of
//              mult(x in N+(a))  (= m_ab * m_bc * m_ac summed per triangle).
// Rows and elements are degree RANKS, not vertex ids (the count is
// label-invariant): row r belongs to vertex uorder[r], rows ascend by rank,
// each row's elements are ascending ranks -- so for a row of the top ranks
// ("hub" rows, r >= n - H) every element of N+(a) and of every N+(b) lies
// in [n - H, n), and k_tc_big counts them in a direct-indexed 16-bit array
// instead of hash probes.  The build ranks the vertices by (degree, id)
// (one radix sort), emits (row rank, element rank) keys for every upper
// slot and sorts them (one 64-bit radix sort), then places the rows.
// Kernel k_tc_fwd: persistent warps pull 32-vertex batches from a global
// counter.  Per vertex a the warp stages A = N+(a), the row starts of its
// b's (from uinfo) and a prefix of their element-holding 16-byte half-sector
// counts (all-padding halves are skipped) in shared
// memory with a 4096-bit membership filter, then walks all rows N+(b) as one
// flattened space of 16-byte half-sectors: each lane loads one int4 per step
// and keeps kUnroll independent loads in flight (the walk is DRAM-latency
// bound otherwise); the rows of a block of 32U half-sectors come from a
// bitmap of the row starts inside it (walk_owners: U shared loads, U+1
// warp OR/add reductions and a popcount per lane).  Every element costs one
// shared-memory filter probe and, on a hit, a binary search in A for its
// multiplicity.  Counts: per-lane uint64 -> warp sum -> one atomicAdd per
// warp.
//
// Vertices whose upper row is longer than kA are counted by k_tc_big, one
// CTA per vertex with A staged in dynamic shared memory.
//
// Directed graphs (no mirror, the program's orientation matters): k_tc_mid
// follows tc.sp literally -- per middle vertex v, A = N(v)_{>v} staged with
// the same filter, each slot u < v of N(v) scans N(u)_{>v}.
#include <cub/cub.cuh>
#include <stdlib.h>

#include <algorithm>
#include <chrono>
#include <mutex>

#include "sp_common.cuh"

using namespace sp;

namespace {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kA = 256;            // warp path: upper rows up to kA (longer: k_tc_big)
constexpr int kT = 512;            // warp path: hash table entries (>= 2 kA)
// per-warp shared words: keys[kT], 16-bit multiplicities packed two per
// word (a count is at most kA), row starts, prefix, filter -- 5.6 KB, so
// 5 blocks of 8 warps fit an SM (6.7 KB with 32-bit counts: 4 blocks)
constexpr int kFwdWarpWords = kT + kT / 2 + 2 * kA + 1 + 128;
constexpr int kFilterWords = 128;  // 4096-bit filter per warp
constexpr int kFilterShift = 20;   // 32 - log2(4096)
constexpr int kBatch = 32;
#ifndef SP_TC_PLAIN_UNROLL
#define SP_TC_PLAIN_UNROLL 2
#endif
constexpr int kUnroll = SP_TC_PLAIN_UNROLL;  // 16-byte loads in flight per lane in k_tc_fwd_plain (cfg3: 1 / 2 / 3 / 4 -> 9.00 / 8.56 / 9.35 / 9.69 ms)
constexpr int kUnrollHash = 4;     // ... in k_tc_fwd_hash (skewed graphs; 2 is faster on cfg3)
#ifndef SP_TC_PAD
#define SP_TC_PAD 8
#endif
#ifndef SP_TC_HUB_SMEM
#define SP_TC_HUB_SMEM (32 * 1024)  // bits, RMAT-24: 16 KB 308 ms, 32 KB 280, 48 KB 304 (16-bit: 32 KB 382, 64 KB 488)
#endif
constexpr int kHubSmem = SP_TC_HUB_SMEM;  // bytes of hub bits / 16-bit counts (256 K / 16 K ranks)
#ifndef SP_TC_HUB_MIN
#define SP_TC_HUB_MIN 128  // RMAT-22: 256 -> 63.9 ms, 128 -> 46.7; RMAT-24: 279.6 -> 282.5 (32, 64: no better)
#endif
constexpr int kHubMinRow = SP_TC_HUB_MIN;  // hub rows longer than this go to k_tc_big
constexpr int kPad = SP_TC_PAD;     // upper rows padded/aligned to 32-byte sectors
constexpr int kQ = kPad / 4;       // 16-byte quarters per padded block

std::mutex g_up_mu;  // guards the lazy upper-CSR build

__device__ __forceinline__ int64_t lower_bound_g(const int32_t *__restrict__ a, int64_t lo,
                                                 int64_t hi, int32_t x) {
    while (lo < hi) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t fhash(int32_t x) {
    return ((uint32_t)x * 2654435761u) >> kFilterShift;  // 12 bits
}

// multiplicity of x in sorted A (shared memory, na entries)
__device__ __forceinline__ int mult_s(const int32_t *A, int na, int32_t x) {
    int lo = 0, hi = na;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (A[mid] < x) lo = mid + 1; else hi = mid;
    }
    int c = 0;
    while (lo < na && A[lo] == x) { c++; lo++; }
    return c;
}

// multiplicity of x in sorted adj[lo, hi) (global memory)
__device__ __forceinline__ int64_t mult_g(const int32_t *__restrict__ adj, int64_t lo, int64_t hi,
                                          int32_t x) {
    int64_t p = lower_bound_g(adj, lo, hi, x), c = 0;
    while (p < hi && __ldg(adj + p) == x) { c++; p++; }
    return c;
}

// Stage sorted A = adj[a0, a0+na) into shared memory and set its filter bits.
__device__ __forceinline__ void stage_a(const int32_t *__restrict__ adj, int64_t a0, int64_t na,
                                        int32_t *A, uint32_t *F, unsigned lane) {
    for (int k = lane; k < kFilterWords; k += 32) F[k] = 0u;
    __syncwarp();
    for (int64_t k = lane; k < na; k += 32) {
        const int32_t x = adj[a0 + k];
        A[k] = x;
        const uint32_t h = fhash(x);
        atomicOr(&F[h >> 5], 1u << (h & 31));
    }
    __syncwarp();
}

// Append the non-empty rows of one 32-row staging chunk (lane: sector start
// s8, `secs` element-holding half-sectors) to B/S at nr; returns the new
// running half-sector total (nr and the total are warp-uniform).
__device__ __forceinline__ int stage_rows(uint32_t *B, int32_t *S, int &nr, int carry,
                                          uint32_t s8, int secs, unsigned lane) {
    int incl = secs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl += t;
    }
    const unsigned keep = __ballot_sync(0xffffffffu, secs > 0);
    if (secs > 0) {
        const int at = nr + __popc(keep & ((1u << lane) - 1u));
        B[at] = s8;
        S[at] = carry + incl - secs;
    }
    nr += __popc(keep);
    return carry + __shfl_sync(0xffffffffu, incl, 31);
}

// Rows owning the half-sectors h0 + 32u + lane (u < U) of a flattened walk
// over rows whose first half-sectors S[0..nr) strictly increase (S[0] = 0,
// S[nr] = the total; empty rows are not listed).  r = the row holding h0
// (warp-uniform), advanced to the row holding h0 + 32U.  The at most 32U
// rows starting inside the block are read with U independent conflict-free
// shared loads per lane and OR-reduced into a 32U-bit start bitmap; a
// lane's owner is then a popcount -- instead of U independent log2(nr)-step
// binary searches (~30% of the skewed-graph walk's instructions).
template <int U>
__device__ __forceinline__ void walk_owners(const int32_t *S, int nr, int h0, int &r,
                                            unsigned lane, int (&own)[U]) {
    unsigned words[U];
#pragma unroll
    for (int u = 0; u < U; u++) words[u] = 0u;
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < U; j++) {
        const int c = r + 1 + j * 32 + (int)lane;
        const int off = (c <= nr ? S[c] : 0x7fffffff) - h0;  // >= 1
        cnt += off <= 32 * U ? 1 : 0;
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int b = off - 32 * u;
            words[u] |= (b >= 0 && b < 32) ? (1u << b) : 0u;
        }
    }
    const unsigned le = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
    int base = r;
#pragma unroll
    for (int u = 0; u < U; u++) {
        const unsigned w = __reduce_or_sync(0xffffffffu, words[u]);
        own[u] = base + __popc(w & le);
        base += __popc(w);
    }
    r += (int)__reduce_add_sync(0xffffffffu, (unsigned)cnt);
}

// ---- upper CSR build (undirected) -------------------------------------

// rank = position in ascending (degree, id) order: keys for the sort
__global__ void k_rank_keys(const int32_t *__restrict__ deg, int64_t n, uint64_t *key,
                            int32_t *id) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        key[v] = ((uint64_t)(uint32_t)deg[v] << 32) | (uint32_t)v;
        id[v] = (int32_t)v;
    }
}

__global__ void k_rank_scatter(const int32_t *__restrict__ order, int64_t n, int32_t *rank) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        rank[order[r]] = (int32_t)r;
}

constexpr int kUpU = 4;  // upper-CSR build: 32-element groups in flight per warp step

// Row rank[v] of the upper CSR = the ranks of v's neighbours ranked above v.
__global__ void k_up_count(const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
                           const int32_t *__restrict__ rank, int64_t n, int32_t *ulen,
                           int64_t *len64, int64_t *pad8) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    for (int64_t v = warp; v < n; v += nw) {
        const int64_t r0 = off[v], r1 = off[v + 1];
        const int32_t rv = rank[v];
        int64_t c = 0;
        // kUpU x 32 elements per step, loads first: a hub row of 10^6
        // elements is otherwise a long chain of adj -> rank round trips
        for (int64_t e0 = r0 + lane; e0 < r1; e0 += 32 * kUpU) {
            int32_t x[kUpU];
#pragma unroll
            for (int j = 0; j < kUpU; j++) x[j] = e0 + 32 * j < r1 ? __ldg(adj + e0 + 32 * j) : -1;
#pragma unroll
            for (int j = 0; j < kUpU; j++) c += x[j] >= 0 && __ldg(rank + x[j]) > rv ? 1 : 0;
        }
        c = warp_sum(c);
        if (lane == 0) {
            ulen[rv] = (int32_t)c;
            len64[rv] = c;
            pad8[rv] = (c + kPad - 1) / kPad;  // 32-byte sectors of the padded row
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        pad8[n] = 0;
        len64[n] = 0;
    }
}

// (row rank, element rank) keys of every upper slot, row-grouped by S.
__global__ void k_up_emit(const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
                          const int32_t *__restrict__ rank, const int64_t *__restrict__ S,
                          int64_t n, uint64_t *keys) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    for (int64_t v = warp; v < n; v += nw) {
        const int64_t r0 = off[v], r1 = off[v + 1];
        const int32_t rv = rank[v];
        int64_t pos = S[rv];
        for (int64_t e0 = r0; e0 < r1; e0 += 32 * kUpU) {
            int32_t x[kUpU], rx[kUpU];
#pragma unroll
            for (int j = 0; j < kUpU; j++) {
                const int64_t e = e0 + 32 * j + lane;
                x[j] = e < r1 ? __ldg(adj + e) : -1;
            }
#pragma unroll
            for (int j = 0; j < kUpU; j++) rx[j] = x[j] >= 0 ? __ldg(rank + x[j]) : -1;
#pragma unroll
            for (int j = 0; j < kUpU; j++) {
                const bool keep = x[j] >= 0 && rx[j] > rv;
                const unsigned m = __ballot_sync(0xffffffffu, keep);
                if (keep)
                    keys[pos + __popc(m & ((1u << lane) - 1u))] =
                        ((uint64_t)(uint32_t)rv << 32) | (uint32_t)rx[j];
                pos += __popc(m);
            }
        }
    }
}

// Sorted keys -> padded rows: uadj (ascending element ranks) and uinfo
// (start and length of the row each element points to).
__global__ void k_up_place(const uint64_t *__restrict__ keys, int64_t mu,
                           const int64_t *__restrict__ S, const int64_t *__restrict__ start8,
                           const int32_t *__restrict__ ulen, int32_t *uadj, uint2 *uinfo) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < mu;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        const int64_t r = (int64_t)(k >> 32);
        const int32_t y = (int32_t)(uint32_t)k;
        const int64_t at = kPad * start8[r] + (i - S[r]);
        uadj[at] = y;
        uinfo[at] = make_uint2((uint32_t)start8[y], (uint32_t)ulen[y]);
    }
}

__global__ void k_up_dups(const uint64_t *__restrict__ keys, int64_t mu, unsigned long long *dup) {
    for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < mu;
         i += (int64_t)gridDim.x * blockDim.x)
        if (keys[i] == keys[i - 1]) {
            *dup = 1ull;
            return;
        }
}

__global__ void k_up_start(const int64_t *__restrict__ start8, int64_t n, uint32_t *ustart8) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n;
         v += (int64_t)gridDim.x * blockDim.x)
        ustart8[v] = (uint32_t)start8[v];
}

__global__ void k_big_list(const int32_t *__restrict__ ulen, int64_t n, int thr, int64_t hub_base,
                           int hub_min, int32_t *list, unsigned long long *cnt) {
    unsigned long long mx = 0;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = b + threadIdx.x;
        const int32_t l = v < n ? ulen[v] : 0;
        mx = max(mx, (unsigned long long)l);
        const bool big = l > thr || (v >= hub_base && l > hub_min);
        const int64_t slot = warp_append(big, &cnt[0]);
        if (big) list[slot] = (int32_t)v;
    }
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&cnt[1], mx);
}

__global__ void k_big_keys(const int32_t *__restrict__ big, const int32_t *__restrict__ ulen,
                           int64_t nbig, uint32_t *key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nbig;
         i += (int64_t)gridDim.x * blockDim.x)
        key[i] = (uint32_t)ulen[big[i]];
}

template <class F>
static int cub_call(Call &c, F f) {  // two-phase CUB call with stream-ordered scratch
    size_t tmp = 0;
    SP_CUDA(f(nullptr, tmp));
    void *dt = nullptr;
    SP_TRY(scratch_alloc(&dt, tmp, c.stream));
    cudaError_t e = f(dt, tmp);
    scratch_free(dt, c.stream);
    SP_CUDA(e);
    return SP_OK;
}

int ensure_upper(sp_graph *g, Call &c) {
    std::lock_guard<std::mutex> lk(g_up_mu);
    if (g->m_up >= 0) return SP_OK;
    prep_mark(g, kPrepTcUpper, 0, c.stream);
    const int64_t n = g->n;
    // SP_TC_TRACE: host time of each build phase (synchronising; diagnostics)
    static const bool trace = getenv("SP_TC_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char *what) {
        if (!trace) return;
        cudaStreamSynchronize(c.stream);
        cudaMemPool_t pool;
        uint64_t used = 0, resv = 0;
        if (cudaDeviceGetDefaultMemPool(&pool, c.device) == cudaSuccess) {
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &resv);
        }
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        fprintf(stderr, "tc upper build: %-12s %8.2f ms (pool used %.1f / reserved %.1f GiB, free %.1f GiB)\n",
                what,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                    .count(),
                used / 1073741824.0, resv / 1073741824.0, fr / 1073741824.0);
    };
    // ---- degree ranks (ascending (degree, id)); rows and elements are ranks
    uint64_t *rkey, *rkey_s;
    int32_t *rid, *rank;
    int32_t *order = nullptr, *ulen = nullptr;
    SP_TRY(c.alloc(&rkey, n));
    SP_TRY(c.alloc(&rkey_s, n));
    SP_TRY(c.alloc(&rid, n));
    SP_TRY(c.alloc(&rank, n));
    SP_TRY(resident_alloc((void **)&order, std::max<int64_t>(1, n) * sizeof(int32_t)));
    SP_TRY(resident_alloc((void **)&ulen, std::max<int64_t>(1, n) * sizeof(int32_t)));
    struct Guard {
        void *p[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
        bool keep = false;
        ~Guard() { if (!keep) for (void *q : p) resident_free(q); }
    } gd;
    gd.p[0] = ulen;
    gd.p[4] = order;
    mark("alloc ranks");
    const int gridn = grid_for(n, 256, c.device, 16);
    k_rank_keys<<<gridn, 256, 0, c.stream>>>(g->outdeg, n, rkey, rid);
    int nbits = 1;
    while (nbits < 31 && ((int64_t)1 << nbits) < n) nbits++;
    int dbits = 1;
    while (dbits < 31 && ((int64_t)1 << dbits) <= g->max_outdeg) dbits++;
    SP_TRY(cub_call(c, [&](void *t, size_t &s) {
        return cub::DeviceRadixSort::SortPairs(t, s, rkey, rkey_s, rid, order, n, 0, 32 + dbits,
                                               c.stream);
    }));
    k_rank_scatter<<<gridn, 256, 0, c.stream>>>(order, n, rank);
    mark("ranks");
    // ---- row lengths, unpadded (S) and padded (start8) row starts
    int64_t *len64, *pad8, *S, *start8;
    SP_TRY(c.alloc(&len64, n + 1));
    SP_TRY(c.alloc(&pad8, n + 1));
    SP_TRY(c.alloc(&S, n + 1));
    SP_TRY(c.alloc(&start8, n + 1));
    const int grid = grid_for(n * 32, 256, c.device, 16);
    k_up_count<<<grid, 256, 0, c.stream>>>(g->off, g->adj, rank, n, ulen, len64, pad8);
    mark("count");
    SP_TRY(cub_call(c, [&](void *t, size_t &s) {
        return cub::DeviceScan::ExclusiveSum(t, s, pad8, start8, n + 1, c.stream);
    }));
    SP_TRY(cub_call(c, [&](void *t, size_t &s) {
        return cub::DeviceScan::ExclusiveSum(t, s, len64, S, n + 1, c.stream);
    }));
    int64_t *h;
    SP_TRY(c.host_as(&h));
    SP_CUDA(cudaMemcpyAsync(h, start8 + n, 8, cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaMemcpyAsync(h + 3, S + n, 8, cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    const int64_t mpad = kPad * h[0], mu = h[3];
    SP_CHECK(h[0] < (int64_t)0xFFFFFFFFll, SP_ERR_UNSUPPORTED,
             "triangle counting: upper CSR of %lld slots exceeds the 2^35 limit",
             (long long)mpad);
    int32_t *uadj = nullptr;
    uint2 *uinfo = nullptr;
    uint32_t *ustart8 = nullptr;
    SP_TRY(resident_alloc((void **)&uadj, std::max<int64_t>(8, mpad) * sizeof(int32_t)));
    gd.p[1] = uadj;
    SP_TRY(resident_alloc((void **)&uinfo, std::max<int64_t>(8, mpad) * sizeof(uint2)));
    gd.p[2] = uinfo;
    SP_TRY(resident_alloc((void **)&ustart8, (n + 1) * sizeof(uint32_t)));
    gd.p[3] = ustart8;
    SP_CUDA(cudaMemsetAsync(uadj, 0xFF, std::max<int64_t>(8, mpad) * sizeof(int32_t), c.stream));
    SP_CUDA(cudaMemsetAsync(uinfo, 0, std::max<int64_t>(8, mpad) * sizeof(uint2), c.stream));
    mark("alloc rows");
    // ---- (row, element) keys, sorted: every row ascending
    if (mu > 0) {
        uint64_t *keys, *keys_s;
        SP_TRY(c.alloc(&keys, mu));
        SP_TRY(c.alloc(&keys_s, mu));
        mark("alloc keys");
        k_up_emit<<<grid, 256, 0, c.stream>>>(g->off, g->adj, rank, S, n, keys);
        mark("emit");
        SP_TRY(cub_call(c, [&](void *t, size_t &s) {
            return cub::DeviceRadixSort::SortKeys(t, s, keys, keys_s, mu, 0, 32 + nbits,
                                                  c.stream);
        }));
        mark("sort");
        k_up_place<<<grid_for(mu, 256, c.device, 16), 256, 0, c.stream>>>(keys_s, mu, S, start8,
                                                                        ulen, uadj, uinfo);
        // a repeated (row, element) key = a multi-edge: multiplicities > 1
        unsigned long long *dup;
        SP_TRY(c.alloc(&dup, 1));
        SP_CUDA(cudaMemsetAsync(dup, 0, 8, c.stream));
        k_up_dups<<<grid_for(mu, 256, c.device, 16), 256, 0, c.stream>>>(keys_s, mu, dup);
        SP_CUDA(cudaMemcpyAsync(h + 4, dup, 8, cudaMemcpyDeviceToHost, c.stream));
        SP_CUDA(cudaStreamSynchronize(c.stream));
    } else {
        h[4] = 0;
    }
    mark("place+dups");
    const bool simple = h[4] == 0;
    k_up_start<<<grid_for(n + 1, 256, c.device, 16), 256, 0, c.stream>>>(start8, n, ustart8);
    c.launches += 9;
    SP_CUDA(cudaGetLastError());
    int32_t *big = nullptr;
    SP_TRY(resident_alloc((void **)&big, std::max<int64_t>(1, n) * sizeof(int32_t)));
    unsigned long long *bc;
    SP_TRY(c.alloc(&bc, 2));
    SP_CUDA(cudaMemsetAsync(bc, 0, 2 * sizeof(unsigned long long), c.stream));
    // SP_TC_WARP_MAX (tests): route shorter rows to k_tc_big too (<= kA)
    const char *wm = getenv("SP_TC_WARP_MAX");
    const int warp_max = wm ? std::max(1, std::min(kA, atoi(wm))) : kA;
    // hub rows (the top ranks, a bitmap / count array in k_tc_big): on
    // simple graphs one bit per rank; rows of those ranks longer than
    // hub_min also go to k_tc_big (SP_TC_HUB_MIN)
    const char *hmn = getenv("SP_TC_HUB_MIN");
    const int hub_min = hmn ? std::max(0, atoi(hmn)) : kHubMinRow;
    const bool hub_bits = simple;
    const int64_t hub_n = std::min<int64_t>(n, (int64_t)kHubSmem * (hub_bits ? 8 : 1) /
                                                   (hub_bits ? 1 : 2));
    const int64_t hub_base = n - hub_n;
    k_big_list<<<grid_for(n, 256, c.device, 16), 256, 0, c.stream>>>(ulen, n, warp_max, hub_base,
                                                                    hub_min, big, bc);
    c.launches += 4;
    SP_CUDA(cudaGetLastError());
    SP_CUDA(cudaMemcpyAsync(h + 1, bc, 16, cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    const int64_t nbig = (int64_t)h[1];
    if (nbig > 1) {  // longest rows first (k_tc_big's dynamic schedule)
        uint32_t *key, *key_s;
        int32_t *big_s;
        SP_TRY(c.alloc(&key, nbig));
        SP_TRY(c.alloc(&key_s, nbig));
        SP_TRY(c.alloc(&big_s, nbig));
        k_big_keys<<<grid_for(nbig, 256, c.device), 256, 0, c.stream>>>(big, ulen, nbig, key);
        size_t stmp = 0;
        SP_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, stmp, key, key_s, big, big_s,
                                                          nbig, 0, 32, c.stream));
        void *st = nullptr;
        SP_TRY(scratch_alloc(&st, stmp, c.stream));
        cudaError_t se = cub::DeviceRadixSort::SortPairsDescending(st, stmp, key, key_s, big,
                                                                   big_s, nbig, 0, 32, c.stream);
        scratch_free(st, c.stream);
        SP_CUDA(se);
        SP_CUDA(cudaMemcpyAsync(big, big_s, nbig * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                c.stream));
        c.launches += 2;
        SP_CUDA(cudaStreamSynchronize(c.stream));
    }
    mark("big list");
    prep_mark(g, kPrepTcUpper, 1, c.stream);
    gd.keep = true;
    g->uorder = order;
    g->tc_simple = simple;
    g->tc_hub_base = hub_base;
    g->tc_hub_min = hub_min;
    g->tc_warp_max = warp_max;
    g->ubig = big;
    g->nbig = (int64_t)h[1];
    g->max_ulen = (int64_t)h[2];
    g->ulen = ulen;
    g->uadj = uadj;
    g->uinfo = uinfo;
    g->ustart8 = ustart8;
    g->m_up_pad = mpad;
    g->m_up = (g->m - 0) / 2;  // informational; exact count not needed
    return SP_OK;
}

// ---- forward intersection (undirected) ---------------------------------

struct TcCounters {
    unsigned long long next;    // vertex batch cursor
    unsigned long long big_next;  // k_tc_big vertex cursor
    unsigned long long total;   // weighted triangle count
    unsigned long long pairs;   // oriented edges (a, b) processed
    unsigned long long elems;   // N+(b) elements probed
    unsigned long long abytes;  // sum over pairs of |N+(a)| (model bytes / 4)
};

// Warp path, plain form: A sorted in shared memory, filter probe, binary
// search on a filter hit (cheapest when hits are rare, e.g. uniform graphs).
#ifndef SP_TCP_MINB
#define SP_TCP_MINB 1
#endif
#ifndef SP_TCH_MINB
#define SP_TCH_MINB 5  // 56 -> 51 registers: 5 blocks/SM (the shared-memory limit); RMAT-24 411 -> 395 ms
#endif
__global__ void __launch_bounds__(kBlock, SP_TCP_MINB) k_tc_fwd_plain(const uint32_t *__restrict__ ustart8,
                                                   const int32_t *__restrict__ ulen,
                                                   const int32_t *__restrict__ uadj,
                                                   const uint2 *__restrict__ uinfo, int64_t v0,
                                                   int64_t v1, int amax, TcCounters *ctr,
                                                   const int32_t *__restrict__ order,
                                                   int64_t id0, int64_t id1, int64_t hub_base, int hub_min) {
    __shared__ int32_t sA[kWarps][kA];
    __shared__ uint32_t sB[kWarps][kA];       // sector start of row b_j
    __shared__ int32_t sS[kWarps][kA + 1];    // half-sector prefix over the rows b_j (element-holding halves only)
    __shared__ uint32_t sF[kWarps][kFilterWords];
    const unsigned lane = lane_id();
    const int wib = threadIdx.x >> 5;
    int32_t *A = sA[wib];
    uint32_t *B = sB[wib];
    int32_t *S = sS[wib];
    uint32_t *F = sF[wib];
    unsigned long long cnt = 0, elems = 0, pairs = 0, abytes = 0;
    for (;;) {
        unsigned long long bt = 0;
        if (lane == 0) bt = atomicAdd(&ctr->next, (unsigned long long)kBatch);
        bt = __shfl_sync(0xffffffffu, bt, 0);
        const int64_t vb = v0 + (int64_t)bt;
        if (vb >= v1) break;
        const int64_t ve = min(v1, vb + kBatch);
        // the batch's row descriptors, one coalesced load
        const int64_t my = vb + lane;
        const uint32_t my_s8 = my < ve ? ustart8[my] : 0u;
        const int32_t my_len = my < ve ? ulen[my] : 0;
        for (int64_t a = vb; a < ve; a++) {
            // rows are degree ranks; a sharded call keeps the rows of its
            // vertex range (warp-uniform)
            if (order) {
                const int32_t id = __ldg(order + a);
                if (id < id0 || id >= id1) continue;
            }
            const int src = (int)(a - vb);
            const int na = __shfl_sync(0xffffffffu, my_len, src);
            if (na < 2) continue;  // a triangle needs b and x in N+(a)
            const int64_t r0 = kPad * (int64_t)__shfl_sync(0xffffffffu, my_s8, src);
            if (na > amax || (a >= hub_base && na > hub_min))
                continue;  // k_tc_big (one CTA per vertex) counts it
            if (lane == 0) {
                pairs += (unsigned long long)na;
                abytes += (unsigned long long)na * (unsigned long long)na;
            }
            // ---- stage A, row starts, half-sector prefix and filter
            for (int k = lane; k < kFilterWords; k += 32) F[k] = 0u;
            __syncwarp();
            int carry = 0, nr = 0;
            for (int k0 = 0; k0 < na; k0 += 32) {
                const int k = k0 + lane;
                int secs = 0;
                uint32_t s8 = 0;
                if (k < na) {
                    const int32_t x = uadj[r0 + k];
                    const uint2 inf = uinfo[r0 + k];
                    A[k] = x;
                    s8 = inf.x;
                    secs = (int)((inf.y + 3u) / 4u);  // half-sectors holding elements
                    elems += inf.y;
                    const uint32_t hh = fhash(x);
                    atomicOr(&F[hh >> 5], 1u << (hh & 31));
                }
                carry = stage_rows(B, S, nr, carry, s8, secs, lane);
            }
            if (lane == 0) S[nr] = carry;
            __syncwarp();
            // ---- flattened walk of all rows b_j in 16-byte half-sectors:
            // one int4 per lane (rows are 32-byte aligned and padded with -1),
            // kUnroll loads in flight per lane, one row search per 4 slots
            const int nhalf = carry;
            for (int h0 = 0; h0 < nhalf; h0 += 32 * kUnroll) {
                int4 xs[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; u++) {
                    const int h = h0 + u * 32 + (int)lane;
                    xs[u] = make_int4(-1, -1, -1, -1);
                    if (h < nhalf) {
                        // short rows (uniform graphs): a few-step binary search
                        // beats walk_owners here (cfg3: 8.53 vs 8.75 ms)
                        int lo = 0, hi = nr;  // last j with S[j] <= h
                        while (hi - lo > 1) {
                            const int mid = (lo + hi) >> 1;
                            if (S[mid] <= h) lo = mid; else hi = mid;
                        }
                        xs[u] = __ldg(reinterpret_cast<const int4 *>(uadj) +
                                      kQ * (int64_t)B[lo] + (h - S[lo]));
                    }
                }
#pragma unroll
                for (int u = 0; u < kUnroll; u++) {
                    const int32_t xv[4] = {xs[u].x, xs[u].y, xs[u].z, xs[u].w};
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const int32_t x = xv[i];
                        if (x < 0) continue;  // padding or past the end
                        const uint32_t hh = fhash(x);
                        if (F[hh >> 5] & (1u << (hh & 31))) cnt += mult_s(A, na, x);
                    }
                }
            }
            __syncwarp();  // A/B/S/F are restaged for the next vertex
        }
    }
    cnt = warp_sum(cnt);
    elems = warp_sum(elems);
    if (lane == 0) {
        if (cnt) atomicAdd(&ctr->total, cnt);
        if (pairs) atomicAdd(&ctr->pairs, pairs);
        if (elems) atomicAdd(&ctr->elems, elems);
        if (abytes) atomicAdd(&ctr->abytes, abytes);
    }
}

// Warp path, hashed form: on a filter hit the multiplicity comes from a
// per-warp hash table of A (skewed graphs, where most probes are hits).
__global__ void __launch_bounds__(kBlock, SP_TCH_MINB) k_tc_fwd_hash(const uint32_t *__restrict__ ustart8,
                                                   const int32_t *__restrict__ ulen,
                                                   const int32_t *__restrict__ uadj,
                                                   const uint2 *__restrict__ uinfo, int64_t v0,
                                                   int64_t v1, int amax, TcCounters *ctr,
                                                   const int32_t *__restrict__ order,
                                                   int64_t id0, int64_t id1, int64_t hub_base, int hub_min) {
    // per warp, dynamic shared memory: hash keys[kT] + counts[kT] of A,
    // sector starts B[kA], half-sector prefix S[kA+1], filter F[kFilterWords]
    extern __shared__ uint32_t fwd_smem[];
    const unsigned lane = lane_id();
    const int wib = threadIdx.x >> 5;
    uint32_t *base = fwd_smem + (size_t)wib * kFwdWarpWords;
    int32_t *HK = reinterpret_cast<int32_t *>(base);
    uint32_t *HC = base + kT;  // two 16-bit counts per word
    uint32_t *B = base + kT + kT / 2;
    int32_t *S = reinterpret_cast<int32_t *>(base + kT + kT / 2 + kA);
    uint32_t *F = base + kT + kT / 2 + 2 * kA + 1;
    unsigned long long cnt = 0, elems = 0, pairs = 0, abytes = 0;
    for (;;) {
        unsigned long long bt = 0;
        if (lane == 0) bt = atomicAdd(&ctr->next, (unsigned long long)kBatch);
        bt = __shfl_sync(0xffffffffu, bt, 0);
        const int64_t vb = v0 + (int64_t)bt;
        if (vb >= v1) break;
        const int64_t ve = min(v1, vb + kBatch);
        // the batch's row descriptors, one coalesced load
        const int64_t my = vb + lane;
        const uint32_t my_s8 = my < ve ? ustart8[my] : 0u;
        const int32_t my_len = my < ve ? ulen[my] : 0;
        for (int64_t a = vb; a < ve; a++) {
            // rows are degree ranks; a sharded call keeps the rows of its
            // vertex range (warp-uniform)
            if (order) {
                const int32_t id = __ldg(order + a);
                if (id < id0 || id >= id1) continue;
            }
            const int src = (int)(a - vb);
            const int na = __shfl_sync(0xffffffffu, my_len, src);
            if (na < 2) continue;  // a triangle needs b and x in N+(a)
            const int64_t r0 = kPad * (int64_t)__shfl_sync(0xffffffffu, my_s8, src);
            if (na > amax || (a >= hub_base && na > hub_min))
                continue;  // k_tc_big (one CTA per vertex) counts it
            if (lane == 0) {
                pairs += (unsigned long long)na;
                abytes += (unsigned long long)na * (unsigned long long)na;
            }
            // ---- hash table of A (with multiplicities), row starts, sector
            // prefix and filter
            int tbits = 5;
            while ((1 << tbits) < 2 * na) tbits++;
            const int T = 1 << tbits;
            for (int k = lane; k < kFilterWords; k += 32) F[k] = 0u;
            for (int k = lane; k < T; k += 32) HK[k] = -1;
            for (int k = lane; k < T / 2; k += 32) HC[k] = 0u;
            __syncwarp();
            int carry = 0, nr = 0;
            for (int k0 = 0; k0 < na; k0 += 32) {
                const int k = k0 + lane;
                int secs = 0;
                uint32_t s8 = 0;
                if (k < na) {
                    const int32_t x = uadj[r0 + k];
                    const uint2 inf = uinfo[r0 + k];
                    uint32_t h = ((uint32_t)x * 2654435761u) >> (32 - tbits);
                    for (;;) {
                        const int32_t old = atomicCAS(&HK[h], -1, x);
                        if (old == -1 || old == x) {
                            atomicAdd(&HC[h >> 1], 1u << ((h & 1u) * 16));
                            break;
                        }
                        h = (h + 1) & (T - 1);
                    }
                    s8 = inf.x;
                    secs = (int)((inf.y + 3u) / 4u);  // half-sectors holding elements
                    elems += inf.y;
                    const uint32_t hh = fhash(x);
                    atomicOr(&F[hh >> 5], 1u << (hh & 31));
                }
                carry = stage_rows(B, S, nr, carry, s8, secs, lane);
            }
            if (lane == 0) S[nr] = carry;
            __syncwarp();
            // ---- flattened walk of all rows b_j in 16-byte half-sectors:
            // one int4 per lane (rows are 32-byte aligned and padded with -1),
            // kUnrollHash loads in flight per lane, one row search per 4 slots
            const int nhalf = carry;
            int row = 0;
            for (int h0 = 0; h0 < nhalf; h0 += 32 * kUnrollHash) {
                int4 xs[kUnrollHash];
                int own[kUnrollHash];
                walk_owners<kUnrollHash>(S, nr, h0, row, lane, own);
#pragma unroll
                for (int u = 0; u < kUnrollHash; u++) {
                    const int h = h0 + u * 32 + (int)lane;
                    xs[u] = make_int4(-1, -1, -1, -1);
                    if (h < nhalf)
                        xs[u] = __ldg(reinterpret_cast<const int4 *>(uadj) +
                                      kQ * (int64_t)B[own[u]] + (h - S[own[u]]));
                }
#pragma unroll
                for (int u = 0; u < kUnrollHash; u++) {
                    const int32_t xv[4] = {xs[u].x, xs[u].y, xs[u].z, xs[u].w};
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const int32_t x = xv[i];
                        if (x < 0) continue;  // padding or past the end
                        const uint32_t hh = fhash(x);
                        if (F[hh >> 5] & (1u << (hh & 31))) {  // filter hit: hash probe
                            uint32_t h = ((uint32_t)x * 2654435761u) >> (32 - tbits);
                            for (;;) {
                                const int32_t key = HK[h];
                                if (key == x) {
                                    cnt += (HC[h >> 1] >> ((h & 1u) * 16)) & 0xFFFFu;
                                    break;
                                }
                                if (key == -1) break;
                                h = (h + 1) & (T - 1);
                            }
                        }
                    }
                }
            }
            __syncwarp();  // A/B/S/F are restaged for the next vertex
        }
    }
    cnt = warp_sum(cnt);
    elems = warp_sum(elems);
    if (lane == 0) {
        if (cnt) atomicAdd(&ctr->total, cnt);
        if (pairs) atomicAdd(&ctr->pairs, pairs);
        if (elems) atomicAdd(&ctr->elems, elems);
        if (abytes) atomicAdd(&ctr->abytes, abytes);
    }
}

// One CTA per vertex whose upper row exceeds the warp path (kA): the block
// builds an open-addressing hash table of A = N+(a) with multiplicities in
// dynamic shared memory (rows up to kHashMax; a membership hit -- on skewed
// graphs most probes are hits -- costs one probe instead of a binary
// search), or for longer rows stages A (up to kBigMax) with a
// kBigFilterBits filter; each warp takes 32 of A's b's at a time, loads
// their row descriptors with one coalesced read, and walks the flattened
// 16-byte half-sectors of their rows (owner by a 5-step shuffle search; a
// window bitmap of row starts, as in the warp path, measured slower here:
// 413 -> 460 ms on RMAT-24),
// one filter probe per element and a shared-memory binary search on a hit.
constexpr int kBigFilterBits = 1 << 17;  // 16 KB
constexpr int kBigFilterShift = 32 - 17;
constexpr int kBigMax = 48 * 1024;      // staged A entries (192 KB) -- beyond: global search
constexpr int kHashMax = 8 * 1024;      // rows up to this are hashed: 2^14 x (key, count) = 128 KB
// One CTA per SM (the shared table); 8 warps per vertex -- 32 warps
// measured slower (744 vs 534 ms on RMAT-24): the static 32-row batches
// leave more warps idle at each vertex's barrier.
#ifndef SP_TC_BIG_BLOCK
#define SP_TC_BIG_BLOCK 256
#endif
constexpr int kBigBlock = SP_TC_BIG_BLOCK;
#ifndef SP_TC_BIG_UNROLL
#define SP_TC_BIG_UNROLL 1  // RMAT-24: 1 -> 253 ms, 4 -> 264 ms
#endif
constexpr int kUnrollBig = SP_TC_BIG_UNROLL;  // 16-byte loads in flight per lane in k_tc_big

__global__ void __launch_bounds__(kBigBlock, 1) k_tc_big(const uint32_t *__restrict__ ustart8,
                                                      const int32_t *__restrict__ ulen,
                                                      const int32_t *__restrict__ uadj,
                                                      const uint2 *__restrict__ uinfo,
                                                      const int32_t *__restrict__ big,
                                                      int64_t nbig, const int32_t *__restrict__ order,
                                                      int64_t id0, int64_t id1,
                                                      int hash_max, int big_max, TcCounters *ctr,
                                                      int64_t hub_base, int hub_words,
                                                      int hub_bits) {
    extern __shared__ uint32_t smem[];
    uint32_t *F = smem;                                        // kBigFilterBits / 32 words
    int32_t *A = reinterpret_cast<int32_t *>(smem + kBigFilterBits / 32);
    // hashed form (na <= kHashMax): keys[T] then counts[T] from smem[0]
    int32_t *HK = reinterpret_cast<int32_t *>(smem);
    const unsigned lane = lane_id();
    unsigned long long cnt = 0, elems = 0, pairs = 0, abytes = 0;
    // Dynamic schedule (big[] is sorted by row length, longest first):
    // CTAs take vertices from a global cursor and warps take 32-row
    // batches of the vertex from a shared cursor -- longest-first
    // assignment keeps the hub tail short on skewed graphs.
    __shared__ long long s_bi;
    __shared__ int s_j;
    bool hub_clean = false;  // the hub array holds only row (prev_r0, prev_na)'s entries
    int64_t prev_r0 = 0;
    int prev_na = 0;
    for (;;) {
        __syncthreads();  // every warp is done with the previous vertex
        if (threadIdx.x == 0) {
            s_bi = (long long)atomicAdd(&ctr->big_next, 1ull);
            s_j = 0;
        }
        __syncthreads();
        const int64_t bi = s_bi;
        if (bi >= nbig) break;
        const int32_t a = big[bi];
        if (order && (__ldg(order + a) < id0 || __ldg(order + a) >= id1)) continue;  // block-uniform
        const int na = ulen[a];
        const int64_t r0 = kPad * (int64_t)ustart8[a];
        // hub rows (rank >= hub_base): every element of N+(a) and of every
        // N+(b) ranks above a, i.e. inside [hub_base, n) -- a direct-indexed
        // array of 16-bit multiplicities replaces the hash probes (one
        // shared load per element, no probe loop, no divergence)
        const bool hub = a >= hub_base && (hub_bits || na <= 65535);
        const bool staged = !hub && na <= big_max;
        const bool hashed = !hub && na <= hash_max;
        int tbits = 6;  // table of 2^tbits >= 2 na entries
        while ((1 << tbits) < 2 * na) tbits++;
        const int T = 1 << tbits;
        uint32_t *HC = reinterpret_cast<uint32_t *>(HK + T);
        // membership filter, 8T bits after the table: a non-member (most
        // probes) costs one bit test instead of ~2.5 linear-probe steps at
        // load factor 1/2; false positives ~ na / 8T <= 1/16
        uint32_t *HF = HC + T;
        const int fbits = tbits + 3;
        __syncthreads();  // previous vertex done with the shared structures
        uint32_t *HUB = smem;  // hub form: bits (or 16-bit counts), index x - hub_base
        if (hub) {
            if (hub_clean) {  // only the previous hub row's words are set: clear them
                for (int k = threadIdx.x; k < prev_na; k += blockDim.x) {
                    const int64_t i = (int64_t)uadj[prev_r0 + k] - hub_base;
                    HUB[hub_bits ? i >> 5 : i >> 1] = 0u;
                }
            } else {  // after a hash / staged row (or at the start): the whole array
                for (int k = threadIdx.x; k < hub_words; k += blockDim.x) HUB[k] = 0u;
            }
            __syncthreads();
            for (int k = threadIdx.x; k < na; k += blockDim.x) {
                const int64_t i = (int64_t)uadj[r0 + k] - hub_base;
                if (hub_bits)  // simple graph: multiplicities are 0 / 1
                    atomicOr(&HUB[i >> 5], 1u << (i & 31));
                else
                    atomicAdd(&HUB[i >> 1], 1u << ((i & 1) * 16));
            }
            __syncthreads();
        } else if (hashed) {
            for (int k = threadIdx.x; k < T; k += blockDim.x) {
                HK[k] = -1;
                HC[k] = 0u;
            }
            for (int k = threadIdx.x; k < T / 4; k += blockDim.x) HF[k] = 0u;
            __syncthreads();
            for (int k = threadIdx.x; k < na; k += blockDim.x) {
                const int32_t x = uadj[r0 + k];
                const uint32_t fb = ((uint32_t)x * 0x9E3779B1u) >> (32 - fbits);
                atomicOr(&HF[fb >> 5], 1u << (fb & 31));
                uint32_t h = ((uint32_t)x * 2654435761u) >> (32 - tbits);
                for (;;) {
                    const int32_t old = atomicCAS(&HK[h], -1, x);
                    if (old == -1 || old == x) {
                        atomicAdd(&HC[h], 1u);
                        break;
                    }
                    h = (h + 1) & (T - 1);
                }
            }
            __syncthreads();
        } else if (staged) {
            for (int k = threadIdx.x; k < kBigFilterBits / 32; k += blockDim.x) F[k] = 0u;
            __syncthreads();
            for (int k = threadIdx.x; k < na; k += blockDim.x) {
                const int32_t x = uadj[r0 + k];
                A[k] = x;
                const uint32_t hh = ((uint32_t)x * 2654435761u) >> kBigFilterShift;
                atomicOr(&F[hh >> 5], 1u << (hh & 31));
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            pairs += (unsigned long long)na;
            abytes += (unsigned long long)na * (unsigned long long)na;
        }
        // (block-uniform) the next hub row clears only this row's words
        hub_clean = hub;
        prev_r0 = r0;
        prev_na = na;
        for (;;) {
            int j0 = 0;
            if (lane == 0) j0 = atomicAdd(&s_j, 32);
            j0 = __shfl_sync(0xffffffffu, j0, 0);
            if (j0 >= na) break;
            const int j = j0 + (int)lane;
            uint2 inf = make_uint2(0u, 0u);
            if (j < na) inf = uinfo[r0 + j];
            elems += inf.y;
            const int secs = (int)((inf.y + 3u) / 4u);  // half-sectors holding elements
            int incl = secs;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)lane >= o) incl += t;
            }
            const int excl = incl - secs;
            const int nhalf = __shfl_sync(0xffffffffu, incl, 31);
            // kUnrollBig half-sectors per lane in flight (their owner searches
            // are independent); one load per lane measured latency-bound
            for (int h0 = 0; h0 < nhalf; h0 += 32 * kUnrollBig) {
                int4 xs[kUnrollBig];
#pragma unroll
                for (int u = 0; u < kUnrollBig; u++) {
                    const int h = h0 + u * 32 + (int)lane;
                    int lo = 0;  // owner lane: largest with excl <= h
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const int cand = lo + step;
                        const int ex = __shfl_sync(0xffffffffu, excl, cand & 31);
                        if (cand < 32 && ex <= h) lo = cand;
                    }
                    const int ex = __shfl_sync(0xffffffffu, excl, lo);
                    const uint32_t s8 = __shfl_sync(0xffffffffu, inf.x, lo);
                    xs[u] = h < nhalf ? __ldg(reinterpret_cast<const int4 *>(uadj) +
                                              kQ * (int64_t)s8 + (h - ex))
                                      : make_int4(-1, -1, -1, -1);
                }
#pragma unroll
                for (int u = 0; u < kUnrollBig; u++) {
                const int32_t xv[4] = {xs[u].x, xs[u].y, xs[u].z, xs[u].w};
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const int32_t x = xv[i];
                    if (x < 0) continue;
                    if (hub) {
                        const int64_t i = (int64_t)x - hub_base;
                        cnt += hub_bits ? (HUB[i >> 5] >> (i & 31)) & 1u
                                        : (HUB[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu;
                    } else if (hashed) {  // multiplicity of x in A
#ifndef SP_TC_BIG_NOFILTER
                        const uint32_t fb = ((uint32_t)x * 0x9E3779B1u) >> (32 - fbits);
                        if (!(HF[fb >> 5] & (1u << (fb & 31)))) continue;
#endif
                        uint32_t h = ((uint32_t)x * 2654435761u) >> (32 - tbits);
                        for (;;) {
                            const int32_t k = HK[h];
                            if (k == x) {
                                cnt += HC[h];
                                break;
                            }
                            if (k == -1) break;
                            h = (h + 1) & (T - 1);
                        }
                    } else if (staged) {
                        const uint32_t hh = ((uint32_t)x * 2654435761u) >> kBigFilterShift;
                        if (F[hh >> 5] & (1u << (hh & 31))) cnt += mult_s(A, na, x);
                    } else {
                        cnt += mult_g(uadj, r0, r0 + na, x);
                    }
                }
                }
            }
        }
    }
    cnt = warp_sum(cnt);
    elems = warp_sum(elems);
    if (lane == 0) {
        if (cnt) atomicAdd(&ctr->total, cnt);
        if (pairs) atomicAdd(&ctr->pairs, pairs);
        if (elems) atomicAdd(&ctr->elems, elems);
        if (abytes) atomicAdd(&ctr->abytes, abytes);
    }
}

// ---- literal middle-vertex form (directed) -----------------------------

__global__ void __launch_bounds__(kBlock, 1) k_tc_mid(const int64_t *__restrict__ off,
                                                   const int32_t *__restrict__ adj, int64_t v0,
                                                   int64_t v1, TcCounters *ctr) {
    __shared__ int32_t sA[kWarps][kA];
    __shared__ uint32_t sF[kWarps][kFilterWords];
    const unsigned lane = lane_id();
    const int wib = threadIdx.x >> 5;
    int32_t *A = sA[wib];
    uint32_t *F = sF[wib];
    unsigned long long cnt = 0, npairs = 0, elems = 0, abytes = 0;
    for (;;) {
        unsigned long long bt = 0;
        if (lane == 0) bt = atomicAdd(&ctr->next, (unsigned long long)kBatch);
        bt = __shfl_sync(0xffffffffu, bt, 0);
        const int64_t vb = v0 + (int64_t)bt;
        if (vb >= v1) break;
        const int64_t ve = min(v1, vb + kBatch);
        for (int64_t v = vb; v < ve; v++) {
            const int64_t r0 = off[v], r1 = off[v + 1];
            if (r1 - r0 < 2) continue;
            // A = [a0, r1) (slots > v); slots < v are [r0, ulast)
            const int64_t a0 = lower_bound_g(adj, r0, r1, (int32_t)v + 1);
            const int64_t na = r1 - a0;
            if (na == 0) continue;
            const int64_t ulast = lower_bound_g(adj, r0, a0, (int32_t)v);
            const int64_t nu = ulast - r0;
            if (nu == 0) continue;
            if (lane == 0) {
                npairs += (unsigned long long)nu;
                abytes += (unsigned long long)nu * (unsigned long long)na;
            }
            const bool staged = na <= kA;
            if (staged) stage_a(adj, a0, na, A, F, lane);
            for (int64_t k = r0 + lane; k < ulast; k += 32) {
                const int32_t u = adj[k];
                const int64_t u0 = off[u], u1 = off[u + 1];
                const int64_t b0 = u1 - u0 > 16 ? lower_bound_g(adj, u0, u1, (int32_t)v + 1) : u0;
                elems += (unsigned long long)(u1 - b0);
                for (int64_t e = b0; e < u1; e++) {
                    const int32_t x = __ldg(adj + e);
                    if (x <= (int32_t)v) continue;
                    if (staged) {
                        const uint32_t h = fhash(x);
                        if (F[h >> 5] & (1u << (h & 31))) cnt += mult_s(A, (int)na, x);
                    } else {
                        cnt += mult_g(adj, a0, r1, x);
                    }
                }
            }
            __syncwarp();
        }
    }
    cnt = warp_sum(cnt);
    elems = warp_sum(elems);
    if (lane == 0) {
        if (cnt) atomicAdd(&ctr->total, cnt);
        if (npairs) atomicAdd(&ctr->pairs, npairs);
        if (elems) atomicAdd(&ctr->elems, elems);
        if (abytes) atomicAdd(&ctr->abytes, abytes);
    }
}

}  // namespace

extern "C" int sp_tc(sp_graph *g, int64_t v0, int64_t v1, uint64_t *count, sp_stats *st) {
    SP_CHECK(g && count && v0 >= 0 && v0 <= v1 && v1 <= g->n, SP_ERR_ARG,
             "sp_tc: bad arguments");
    static const bool trace = getenv("SP_TC_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    Call c;
    SP_TRY(c.begin(g->device));
    if (!g->directed && g->n) SP_TRY(ensure_upper(g, c));
    if (trace) {
        cudaStreamSynchronize(c.stream);
        fprintf(stderr, "tc: begin + upper CSR %.2f ms\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                    .count());
    }
    TcCounters *ctr;
    SP_TRY(c.alloc(&ctr, 1));
    SP_CUDA(cudaMemsetAsync(ctr, 0, sizeof(TcCounters), c.stream));
    const int sms = num_sms(c.device);
    cudaEvent_t ka, kb;
    SP_CUDA(cudaEventCreate(&ka));
    SP_CUDA(cudaEventCreate(&kb));
    cudaEventRecord(ka, c.stream);
    // undirected rows are degree ranks: a partial vertex range filters rows
    // by their vertex id (uorder), the full range needs no filter
    const int64_t n = g->n;
    const int32_t *order = (!g->directed && (v0 != 0 || v1 != n)) ? g->uorder : nullptr;
    if (v1 > v0) {
        const int64_t rows = g->directed ? v1 - v0 : n;
        int64_t want = (rows + kBatch * kWarps - 1) / (kBatch * kWarps);
        int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
        if (g->directed) {
            k_tc_mid<<<grid, kBlock, 0, c.stream>>>(g->off, g->adj, v0, v1, ctr);
            c.launches++;
        } else {
            if (g->nbig > 0) {  // skewed: long upper rows exist, hits are frequent
                const size_t fsm = (size_t)kWarps * kFwdWarpWords * 4;
                SP_CUDA(cudaFuncSetAttribute(k_tc_fwd_hash,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));
                k_tc_fwd_hash<<<grid, kBlock, fsm, c.stream>>>(g->ustart8, g->ulen, g->uadj,
                                                               g->uinfo, 0, n, g->tc_warp_max,
                                                               ctr, order, v0, v1, g->tc_hub_base,
                                                               g->tc_hub_min);
            } else {
                k_tc_fwd_plain<<<grid, kBlock, 0, c.stream>>>(g->ustart8, g->ulen, g->uadj,
                                                              g->uinfo, 0, n, g->tc_warp_max,
                                                              ctr, order, v0, v1, g->tc_hub_base,
                                                              g->tc_hub_min);
            }
            c.launches++;
            if (g->nbig) {
                // row-form limits (SP_TC_HASH_MAX / SP_TC_BIG_MAX: tests, to reach the
                // staged and global-search forms on small graphs)
                const char *hm = getenv("SP_TC_HASH_MAX"), *bm = getenv("SP_TC_BIG_MAX");
                const int hash_max = hm ? std::max(1, std::min(kHashMax, atoi(hm))) : kHashMax;
                const int big_max = bm ? std::max(1, std::min(kBigMax, atoi(bm))) : kBigMax;
                int tb = 6;
                while ((1 << tb) < 2 * std::min<int64_t>(g->max_ulen, hash_max)) tb++;
                size_t smem = std::max<size_t>(
                    ((size_t)8 << tb) + ((size_t)1 << tb),  // hash keys + counts + filter
                    kBigFilterBits / 8 + 4 * (size_t)std::min<int64_t>(g->max_ulen, big_max));
                // hub rows: the top ranks whose 16-bit count array fits kHubSmem
                // (SP_TC_HUB=0: off; rows are ranks, so hubs are [hub_base, n))
                const char *he = getenv("SP_TC_HUB");
                // simple graphs (no multi-edges): one bit per hub rank, 8x the rows
                // (SP_TC_HUB=2: 16-bit counts, =0: the hash forms for every row)
                const int hub_bits = g->tc_simple && !(he && he[0] == '2') ? 1 : 0;
                int64_t hub_base = g->tc_hub_base;
                if (!hub_bits && g->tc_simple)  // 16-bit counts cover 16x fewer ranks
                    hub_base = std::max<int64_t>(hub_base, n - (int64_t)kHubSmem / 2);
                if (he && he[0] == '0') hub_base = n;
                const int64_t hub_n = n - hub_base;
                const int hub_words = (int)(hub_bits ? (hub_n + 31) / 32 : (hub_n + 1) / 2);
                if (hub_n) smem = std::max<size_t>(smem, (size_t)hub_words * 4);
                SP_CUDA(cudaFuncSetAttribute(k_tc_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
                int per_sm = 1;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tc_big, kBigBlock, smem);
                const int gb = (int)std::min<int64_t>(g->nbig,
                                                      (int64_t)sms * std::max(1, per_sm));
                k_tc_big<<<gb, kBigBlock, smem, c.stream>>>(g->ustart8, g->ulen, g->uadj, g->uinfo,
                                                         g->ubig, g->nbig, order, v0, v1,
                                                         hash_max, big_max, ctr, hub_base,
                                                         hub_words, hub_bits);
                c.launches++;
            }
        }
    }
    cudaEventRecord(kb, c.stream);
    SP_CUDA(cudaGetLastError());
    TcCounters *h;
    SP_TRY(c.host_as(&h));
    SP_CUDA(cudaMemcpyAsync(h, ctr, sizeof(TcCounters), cudaMemcpyDeviceToHost, c.stream));
    int rc = c.finish(st);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ka, kb);
    cudaEventDestroy(ka);
    cudaEventDestroy(kb);
    if (trace)
        fprintf(stderr, "tc: counting %.2f ms (device), call %.2f ms\n", ms,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                    .count());
    SP_TRY(rc);
    *count = (uint64_t)h->total;
    if (st) {
        st->iterations = 1;
        st->edges_visited = (int64_t)h->pairs;
        st->vertices_visited = v1 - v0;
        st->main_kernel_ms = ms;
        st->main_kernel_launches = v1 > v0 ? 1 : 0;
        // 8 B/vertex (offsets) + 4 B per stored slot + 4 B per
        // element of both intersected rows
        st->model_bytes = 8 * (v1 - v0) +
                          4 * (g->directed ? g->m : g->m / 2) +
                          4 * (int64_t)(h->abytes + h->elems);
    }
    return SP_OK;
}
