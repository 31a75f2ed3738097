// sp_fold.cuh -- ordered per-vertex folds over CSR rows (the `+=` reductions
// of interp.py:347-359/561-572 inside a forall over a vertex list).
//
// The reference folds left in iteration order.  k_fold keeps that order
// bit-exactly while loading with full-warp parallelism:
//   * a warp takes 32 listed vertices, prefix-sums their row lengths and
//     streams the flattened slots in kChunk-slot chunks; every lane computes
//     kChunk/32 terms (independent gathers in flight) into shared memory;
//   * each lane then folds the part of ITS row inside the chunk,
//     sequentially, in CSR order (a skipped slot contributes +0.0, which
//     leaves a non-negative running sum bit-identical).
// Deterministic mode: rows longer than hub_thr are deferred to k_fold_hub
// (one CTA per row, staged in 1024-slot chunks, folded sequentially:
// bit-exact).  Fast mode: rows longer than kShortRow are cut into
// kFoldSplit-slot chunks folded by whole warps (k_fold_chunks) and combined
// per row in chunk order (k_fold_combine): deterministic run to run, a few
// ulps from the left fold, and no lane folds a long row while its
// warp-mates idle.
// F supplies: double payload(int32_t v); int32_t key(int64_t slot) (the
//             slot's neighbour); double term(double pay, int32_t key);
//             void finish(int32_t v, double sum).
#pragma once

#include "sp_common.cuh"

namespace sp {

constexpr int kFoldBlock = 256;
constexpr int kFoldWarps = kFoldBlock / 32;
constexpr int kFoldChunk = 128;
constexpr int kHubFoldBlock = 256;
constexpr int kHubFoldChunk = 1024;

// Fast mode: rows longer than short_thr are cut into kFoldSplit-slot chunks.
// k_fold registers each such row (vertex, first chunk slot, chunk count) and
// publishes one work item per chunk; k_fold_chunks gives every chunk one
// warp (8 independent terms in flight per lane, fixed xor tree) and stores
// its partial; k_fold_combine adds a row's partials in chunk order (fixed
// shape: deterministic run to run) and finishes the row.
constexpr int kFoldSplit = 256;

struct FoldChunks {
    int32_t *reg_v;      // registered row vertex
    int64_t *reg_base;   // its first chunk slot
    int32_t *reg_nch;    // its chunk count
    uint4 *items;        // chunk slot -> {vertex, first slot lo, hi, slot count}
    double *csum;        // chunk slot -> partial sum
    unsigned long long *counts;  // [0] registered rows, [1] chunk slots used
};

template <class F>
__global__ void __launch_bounds__(kFoldBlock) k_fold(
    F f, const int64_t *__restrict__ rowoff, const int32_t *__restrict__ q, int64_t nq,
    int64_t hub_thr, int32_t *__restrict__ hubs, unsigned long long *nhubs, int64_t short_thr,
    FoldChunks fc) {
    __shared__ double stage[kFoldWarps][kFoldChunk];
    const unsigned lane = lane_id();
    double *buf = stage[threadIdx.x >> 5];
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * 32; base < nq; base += nwarps * 32) {
        const int64_t i = base + lane;
        int32_t v = -1;
        int64_t rs = 0, deg = 0;
        double pay = 0.0;
        if (i < nq) {
            v = q[i];
            rs = rowoff[v];
            deg = rowoff[v + 1] - rs;
            pay = f.payload(v);
        }
        const bool hub = deg > hub_thr;
        const bool mid = !hub && deg > short_thr;
        {
            int64_t slot = warp_append(hub, nhubs);
            if (hub) hubs[slot] = v;
        }
        if (short_thr < hub_thr) {  // fast mode: register the row's chunks
            const int64_t r = warp_append(mid, &fc.counts[0]);
            if (mid) {
                const int nch = (int)((deg + kFoldSplit - 1) / kFoldSplit);
                const int64_t base = (int64_t)atomicAdd(&fc.counts[1], (unsigned long long)nch);
                fc.reg_v[r] = v;
                fc.reg_base[r] = base;
                fc.reg_nch[r] = nch;
                for (int c = 0; c < nch; c++) {
                    const int64_t s0 = rs + (int64_t)c * kFoldSplit;
                    const int64_t len = min((int64_t)kFoldSplit, rs + deg - s0);
                    fc.items[base + c] = make_uint4((unsigned)v, (unsigned)(uint64_t)s0,
                                                    (unsigned)((uint64_t)s0 >> 32), (unsigned)len);
                }
            }
        }
        const bool deferred = hub || mid;
        if (deferred) deg = 0;
        int64_t incl = deg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += t;
        }
        const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
        const int64_t excl = incl - deg;
        double sum = 0.0;
        for (int64_t p0 = 0; p0 < total; p0 += kFoldChunk) {
#pragma unroll
            for (int j = 0; j < kFoldChunk / 32; j++) {
                const int64_t p = p0 + j * 32 + lane;
                int lo = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    int cand = lo + step;
                    int64_t ex = __shfl_sync(0xffffffffu, excl, cand & 31);
                    if (cand < 32 && ex <= p) lo = cand;
                }
                const int64_t ex = __shfl_sync(0xffffffffu, excl, lo);
                const int64_t b0 = __shfl_sync(0xffffffffu, rs, lo);
                const double pv = __shfl_sync(0xffffffffu, pay, lo);
                buf[j * 32 + lane] = p < total ? f.term(pv, f.key(b0 + (p - ex))) : 0.0;
            }
            __syncwarp();
            const int64_t a = max(excl, p0), b = min(excl + deg, p0 + (int64_t)kFoldChunk);
            for (int64_t p = a; p < b; p++) sum = __dadd_rn(sum, buf[p - p0]);
            __syncwarp();
        }
        if (i < nq && !deferred) f.finish(v, sum);
    }
}

// Keys (streamed slot loads) and payload of one chunk; count 0: all -1.
template <class F, int K>
__device__ __forceinline__ void fold_load_chunk(const F &f, const uint4 d, unsigned lane,
                                                int32_t (&key)[K], double &pay) {
    const int64_t s0 = (int64_t)(((uint64_t)d.z << 32) | d.y);
#pragma unroll
    for (int j = 0; j < K; j++) {
        const unsigned p = j * 32 + lane;
        key[j] = p < d.w ? f.key(s0 + p) : -1;
    }
    pay = d.w ? f.payload((int32_t)d.x) : 0.0;
}

// One warp per chunk, pipelined like expand_chunks_body: the descriptor two
// chunks ahead and the keys + payload of the next chunk load while the
// current chunk's terms (random record reads) are summed.
template <class F>
__global__ void __launch_bounds__(kFoldBlock) k_fold_chunks(F f, const int64_t *__restrict__ rowoff,
                                                            FoldChunks fc) {
    constexpr int kPer = kFoldSplit / 32;
    const unsigned lane = lane_id();
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nitems = (int64_t)__ldcg(&fc.counts[1]);
    const uint4 none = make_uint4(0, 0, 0, 0);
    int32_t key[kPer];
    double pay;
    fold_load_chunk(f, warp < nitems ? fc.items[warp] : none, lane, key, pay);
    uint4 d1 = warp + nwarps < nitems ? fc.items[warp + nwarps] : none;
    for (int64_t k = warp; k < nitems; k += nwarps) {
        const uint4 d2 = k + 2 * nwarps < nitems ? fc.items[k + 2 * nwarps] : none;
        int32_t keyn[kPer];
        double payn;
        fold_load_chunk(f, d1, lane, keyn, payn);
        double t[kPer];
#pragma unroll
        for (int j = 0; j < kPer; j++) t[j] = key[j] >= 0 ? f.term(pay, key[j]) : 0.0;
        double sum = 0.0;
#pragma unroll
        for (int j = 0; j < kPer; j++) sum = __dadd_rn(sum, t[j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum = __dadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, o));
        if (lane == 0) fc.csum[k] = sum;
#pragma unroll
        for (int j = 0; j < kPer; j++) key[j] = keyn[j];
        pay = payn;
        d1 = d2;
    }
}

template <class F>
__global__ void __launch_bounds__(kFoldBlock) k_fold_combine(F f, FoldChunks fc) {
    const unsigned lane = lane_id();
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nreg = (int64_t)__ldcg(&fc.counts[0]);
    for (int64_t r = warp; r < nreg; r += nwarps) {
        const int64_t base = fc.reg_base[r];
        const int nch = fc.reg_nch[r];
        double s = 0.0;
        for (int c0 = 0; c0 < nch; c0 += 32) {
            double t = c0 + (int)lane < nch ? fc.csum[base + c0 + lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, o));
            s = __dadd_rn(s, t);
        }
        if (lane == 0) f.finish(fc.reg_v[r], s);
    }
}

template <class F>
__global__ void __launch_bounds__(kHubFoldBlock) k_fold_hub(
    F f, const int64_t *__restrict__ rowoff, const int32_t *__restrict__ hubs,
    const unsigned long long *__restrict__ nhubs, int deterministic) {
    __shared__ double stage[kHubFoldChunk];
    __shared__ double red[kHubFoldBlock / 32];
    const int64_t nh = (int64_t)*nhubs;
    for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
        const int32_t v = hubs[h];
        const int64_t rs = rowoff[v], re = rowoff[v + 1];
        const double pay = f.payload(v);
        double acc = 0.0;  // meaningful in thread 0
        for (int64_t c0 = rs; c0 < re; c0 += kHubFoldChunk) {
            const int64_t len = min((int64_t)kHubFoldChunk, re - c0);
#pragma unroll
            for (int k = 0; k < kHubFoldChunk / kHubFoldBlock; k++) {
                const int j = threadIdx.x + k * kHubFoldBlock;
                stage[j] = j < len ? f.term(pay, f.key(c0 + j)) : 0.0;
            }
            __syncthreads();
            if (deterministic) {
                if (threadIdx.x == 0)
                    for (int64_t j = 0; j < len; j++) acc = __dadd_rn(acc, stage[j]);
            } else {
                constexpr int per = kHubFoldChunk / kHubFoldBlock;
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < per; k++) s = __dadd_rn(s, stage[threadIdx.x * per + k]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
                if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
                __syncthreads();
                if (threadIdx.x < 32) {
                    double t = threadIdx.x < kHubFoldBlock / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1)
                        t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, o));
                    if (threadIdx.x == 0) acc = __dadd_rn(acc, t);
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) f.finish(v, acc);
        __syncthreads();
    }
}

// Deferred-row buffers of a fold launch.
struct FoldLists {
    int32_t *hubs;                 // deterministic mode: rows > hub_thr (n)
    unsigned long long *counts;    // [0] hubs, [1] registered rows, [2] chunk slots
    FoldChunks chunks;             // fast mode: chunked rows
};

// Capacity of the chunk-slot buffers for a graph with m slots.
inline int64_t fold_chunk_capacity(int64_t m) { return m / kFoldSplit + m / 48 + 2; }

// Fast mode (!deterministic): rows longer than kShortRow are folded in
// kFoldSplit-slot chunks by whole warps; deterministic mode folds every row
// left to right (rows > hub_thr by k_fold_hub's thread 0).
constexpr int64_t kShortRow = 48;

template <class F>
inline void launch_fold(const F &f, const int64_t *rowoff, const int32_t *q, int64_t nq,
                        int64_t hub_thr, const FoldLists &fl, bool deterministic,
                        int64_t max_row, int sms, cudaStream_t s, int64_t *launches) {
    if (nq <= 0) return;
    const bool hubs = deterministic && max_row > hub_thr;
    const bool chunked = !deterministic && max_row > kShortRow;
    if (hubs || chunked) cudaMemsetAsync(fl.counts, 0, 3 * sizeof(unsigned long long), s);
    const int cap = sms * 8;
    int64_t want = (nq + kFoldBlock - 1) / kFoldBlock;
    int g = (int)(want < 1 ? 1 : (want > cap ? cap : want));
    FoldChunks fc = fl.chunks;
    fc.counts = fl.counts + 1;
    k_fold<F><<<g, kFoldBlock, 0, s>>>(f, rowoff, q, nq, hubs ? hub_thr : INT64_MAX, fl.hubs,
                                       fl.counts, chunked ? kShortRow : INT64_MAX, fc);
    ++*launches;
    if (chunked) {
        k_fold_chunks<F><<<cap, kFoldBlock, 0, s>>>(f, rowoff, fc);
        k_fold_combine<F><<<cap, kFoldBlock, 0, s>>>(f, fc);
        *launches += 2;
    }
    if (hubs) {
        k_fold_hub<F><<<sms * 2, kHubFoldBlock, 0, s>>>(f, rowoff, fl.hubs, fl.counts, 1);
        ++*launches;
    }
}

}  // namespace sp
