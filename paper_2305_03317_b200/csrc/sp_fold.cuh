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
// Rows longer than hub_thr are deferred to k_fold_hub: one CTA per row,
// staged in 1024-slot chunks; deterministic mode folds them sequentially
// (bit-exact), fast mode uses a fixed-shape tree per chunk (deterministic
// run to run, ~1e-16 relative from the left fold).
// F supplies: double payload(int32_t v); double term(double pay, int64_t slot);
//             void finish(int32_t v, double sum).
#pragma once

#include "sp_common.cuh"

namespace sp {

constexpr int kFoldBlock = 256;
constexpr int kFoldWarps = kFoldBlock / 32;
constexpr int kFoldChunk = 128;
constexpr int kHubFoldBlock = 256;
constexpr int kHubFoldChunk = 1024;

template <class F>
__global__ void __launch_bounds__(kFoldBlock) k_fold(
    F f, const int64_t *__restrict__ rowoff, const int32_t *__restrict__ q, int64_t nq,
    int64_t hub_thr, int32_t *__restrict__ hubs, unsigned long long *nhubs) {
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
        if (hub) {
            deg = 0;
        }
        {
            int64_t slot = warp_append(hub, nhubs);
            if (hub) hubs[slot] = v;
        }
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
                buf[j * 32 + lane] = p < total ? f.term(pv, b0 + (p - ex)) : 0.0;
            }
            __syncwarp();
            const int64_t a = max(excl, p0), b = min(excl + deg, p0 + (int64_t)kFoldChunk);
            for (int64_t p = a; p < b; p++) sum = __dadd_rn(sum, buf[p - p0]);
            __syncwarp();
        }
        if (i < nq && !hub) f.finish(v, sum);
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
                stage[j] = j < len ? f.term(pay, c0 + j) : 0.0;
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

template <class F>
inline void launch_fold(const F &f, const int64_t *rowoff, const int32_t *q, int64_t nq,
                        int64_t hub_thr, int32_t *hubs, unsigned long long *nhubs_dev,
                        bool deterministic, bool may_have_hubs, int sms, cudaStream_t s,
                        int64_t *launches) {
    if (nq <= 0) return;
    if (may_have_hubs) cudaMemsetAsync(nhubs_dev, 0, sizeof(unsigned long long), s);
    const int cap = sms * 8;
    int64_t want = (nq + kFoldBlock - 1) / kFoldBlock;
    int g = (int)(want < 1 ? 1 : (want > cap ? cap : want));
    k_fold<F><<<g, kFoldBlock, 0, s>>>(f, rowoff, q, nq, may_have_hubs ? hub_thr : INT64_MAX,
                                       hubs, nhubs_dev);
    ++*launches;
    if (may_have_hubs) {
        k_fold_hub<F><<<sms * 2, kHubFoldBlock, 0, s>>>(f, rowoff, hubs, nhubs_dev,
                                                        deterministic ? 1 : 0);
        ++*launches;
    }
}

}  // namespace sp
