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
// rank), outdeg int32[n], reverse CSR (roff int64, radj int32), the graph's
// non-empty-row index (nzrow int32, nzend int64: rows with in-degree > 0 and
// their ends), one f64 diff slot per iteration (max via atomicMax on the bit
// pattern of a non-negative double: exact and order-independent).
//
// Fast path (default) -- edge-balanced, one pass over radj per iteration:
//   k_pr_units: the slot range is cut into units of kUnit consecutive radj
//     slots; a warp takes a unit and streams it in kCh-slot chunks (8 slots
//     per lane: two 128-bit radj loads, eight independent contrib gathers).
//     Row ends inside a chunk are marked in a per-warp shared-memory bitmap
//     from a coalesced window of nzend; each lane folds its 8 values
//     left-to-right, a segmented Kogge-Stone warp scan carries partial sums
//     across lanes and a warp-uniform carry across chunks, and the lane
//     holding a row's last slot stores the row sum (sums[k], k = nz row).
//     Every warp does the same work whatever the degree mix (a 100K-slot hub
//     is just 50 units).
//   k_pr_epi: pr.sp:17-23 for every non-empty row, coalesced over k
//     (newRank, |delta| max, rank and contrib writes); a row that started
//     in an earlier unit is finished here first, its unit partials added
//     left to right (deterministic, fixed shape).
//   The iterations run as a device-side loop (CUDA graph with a conditional
//   WHILE node; k_pr_advance evaluates `diff < eps || iter >= maxIter` and
//   swaps the contrib buffers) unless a per-iteration callback is set.
//   k_pr_zero: rows with no in-edges have sum = 0, so newRank = (1-d)/n in
//     every iteration; they are written in iteration 1 only (identical bits
//     afterwards, |delta| = 0), into both contrib buffers.
//   Accumulation order: left fold inside each lane's 8 slots, then a fixed
//   Kogge-Stone tree across lanes/chunks/units.  Deterministic run to run;
//   differs from the interpreter's left fold by a few ulps (<= 1e-12
//   relative, tested; the north star allows 1e-6).
// Exact path (SP_FLAG_DETERMINISTIC): k_pull_exact -- a warp owns 32
//   consecutive vertices whose rows form one contiguous radj slab, streams it
//   through shared memory and every lane folds its own row sequentially in
//   CSR order: bit-identical to the interpreter, slower on hub rows.
// No FMA contraction anywhere: __dadd_rn/__dmul_rn are used explicitly.
#include <cub/cub.cuh>
#include <stdlib.h>

#include <algorithm>
#include <mutex>

#include "sp_common.cuh"

using namespace sp;

namespace {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kChunk = 128;     // exact path: slab slots staged per warp per step
constexpr int64_t kUnit = 768;   // fast path: radj slots per work unit (one warp); cfg2: 512/768/1024/2048/4096 -> 220/222/219/214/188 GTEPS
constexpr int kCh = 256;        // fast path: slots per warp chunk (8 per lane)
constexpr int kHotBlock = 1024;   // persistent hot-source variant: threads per block
constexpr int kHotMax = 20 * 1024;  // hot contrib values in shared memory (160 KB); cfg2: 16K/20K/24K/28K -> 232/233/221/154 GTEPS (more smem leaves less L1 for the cold gathers)
constexpr int kHotBit = 1 << 30;    // encoded radj: source is hot, low bits = hot index

__global__ void k_init(double *rank, double *contrib, const int32_t *__restrict__ outdeg,
                       int64_t v0, int64_t v1, double r0) {
    for (int64_t x = v0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < v1;
         x += (int64_t)gridDim.x * blockDim.x) {
        rank[x - v0] = r0;
        int d = outdeg[x];
        contrib[x - v0] = d > 0 ? __ddiv_rn(r0, (double)d) : 0.0;
    }
}

// ---------------------------------------------------------------- fast path

struct PrArgs {
    const int32_t *__restrict__ radj;
    const int64_t *__restrict__ nzend;
    const int32_t *__restrict__ nzrow;
    const int32_t *__restrict__ outdeg;
    const double *__restrict__ cin;  // full n-array, global ids
    double *__restrict__ rank;       // local (index v - v0)
    double *__restrict__ cout;       // local (index v - v0)
    double *__restrict__ sums;       // row sums, index k - K0 (nz row)
    int64_t v0;
    int64_t S0, S1;                  // radj slot range of the block
    int64_t K0, K1;                  // nz rows [K0, K1) lie in the block
    int64_t u0, nunits;              // global index of the first unit, count
    const int64_t *__restrict__ unit_row;  // first nz row with end > unit start
    double *__restrict__ hp;         // partial of a row that began before the unit
    double *__restrict__ tp;         // partial of the row still open at unit end
    double base, damping;
    double *diff_slot;
    struct PrLoop *loop;  // device loop state (cin/cout/slot come from it) or null
};

// Device-side fixedPoint loop state (pr.sp:10): contrib ping-pong and diff
// slots are picked by `cur`, so the captured kernels never change.
struct PrLoop {
    double *c[2];
    double *slot[2];
    int cur;
    int64_t iter, iters, max_iter, cap;
    double eps, diff;
    int status;  // 0 running/converged, 2 cap reached
};

__device__ __forceinline__ void pr_bind(PrArgs &a) {
    if (a.loop) {
        const int cur = a.loop->cur;
        a.cin = a.loop->c[cur];
        a.cout = a.loop->c[cur ^ 1];
        a.diff_slot = a.loop->slot[cur];
    }
}

// pr.sp:17-23 for one vertex; returns |newRank - rank|.
__device__ __forceinline__ double pr_apply(const PrArgs &a, int64_t v, double sum) {
    const double nr = __dadd_rn(a.base, __dmul_rn(a.damping, sum));
    const int64_t lv = v - a.v0;
    const double r = a.rank[lv];
    double d = __dsub_rn(nr, r);
    if (d < 0.0) d = __dsub_rn(0.0, d);
    a.rank[lv] = nr;
    const int od = __ldg(a.outdeg + v);
    a.cout[lv] = od > 0 ? __ddiv_rn(nr, (double)od) : 0.0;
    return d;
}

// One atomic per block (blockDim.x == 256): same-address atomics serialise.
__device__ __forceinline__ void block_diff(const PrArgs &a, double dmax) {
    __shared__ double red[8];
    __syncwarp();  // reconverge after divergent per-row work: the block barrier is .aligned
    dmax = warp_max(dmax);
    if (lane_id() == 0) red[threadIdx.x >> 5] = dmax;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = threadIdx.x < 8 ? red[threadIdx.x] : 0.0;
        t = warp_max(t);
        // read first: same-address atomics from thousands of blocks
        // serialise at one L2 slice (k_pr_zero: 16 K blocks, ~0.2 ms), and
        // most blocks do not raise the maximum (order-free: exact either way)
        if (threadIdx.x == 0 && t > 0.0 &&
            __double_as_longlong(t) > (long long)__ldcg(
                reinterpret_cast<const unsigned long long *>(a.diff_slot)))
            atomic_max_nonneg(a.diff_slot, t);
    }
}

// radj[c + 8*lane .. +8) clipped to s1 (-1 past it): two 128-bit loads
// when aligned and in range.
__device__ __forceinline__ void load_slab(const int32_t *__restrict__ radj, int64_t c, int64_t s1,
                                          unsigned lane, int (&idx)[8]) {
    const int64_t q = c + 8 * (int64_t)lane;
    if (q + 8 <= s1 && (q & 3) == 0) {
        const int4 x0 = __ldcs(reinterpret_cast<const int4 *>(radj + q));
        const int4 x1 = __ldcs(reinterpret_cast<const int4 *>(radj + q + 4));
        idx[0] = x0.x; idx[1] = x0.y; idx[2] = x0.z; idx[3] = x0.w;
        idx[4] = x1.x; idx[5] = x1.y; idx[6] = x1.z; idx[7] = x1.w;
    } else {
#pragma unroll
        for (int i = 0; i < 8; i++) idx[i] = q + i < s1 ? __ldcs(radj + q + i) : -1;
    }
}

// Row sums over edge-balanced units (see the file header).
template <bool kHot>
__device__ __forceinline__ void pr_units_body(const PrArgs &a, uint32_t *bm, const double *hot) {
    const unsigned lane = lane_id();
    if (lane < kCh / 32) bm[lane] = 0u;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = warp; u < a.nunits; u += nwarps) {
        const int64_t gu = a.u0 + u;
        const int64_t s0 = max(a.S0, gu * kUnit), s1 = min(a.S1, (gu + 1) * kUnit);
        int64_t rk = a.unit_row[u];
        const int64_t first_row = rk;
        // the unit's first row began in an earlier unit
        const bool head_spill = (rk > 0 ? __ldg(a.nzend + rk - 1) : 0) < s0;
        double carry = 0.0;
        int nxt[8];
        load_slab(a.radj, s0, s1, lane, nxt);
        for (int64_t c = s0; c < s1; c += kCh) {
            const int64_t lim = min(c + (int64_t)kCh, s1);
            // ---- radj slab: 8 consecutive slots per lane (prefetched one
            // chunk ahead so the DRAM latency overlaps this chunk's work)
            int idx[8];
#pragma unroll
            for (int i = 0; i < 8; i++) idx[i] = nxt[i];
            if (lim < s1) load_slab(a.radj, lim, s1, lane, nxt);
            // ---- row-end bitmap for this chunk from a window of nzend
            __syncwarp();
            const int64_t rk_chunk = rk;
            for (;;) {
                const int64_t k = rk + lane;
                const int64_t e = k < a.K1 ? __ldg(a.nzend + k) : INT64_MAX;
                const bool in = e <= lim;  // the row's last slot e-1 lies in [c, lim)
                if (in) {
                    const int b = (int)(e - 1 - c);
                    atomicOr(&bm[b >> 5], 1u << (b & 31));
                }
                const int cnt = __popc(__ballot_sync(0xffffffffu, in));
                rk += cnt;
                if (cnt < 32) break;
            }
            double val[8];
#pragma unroll
            for (int i = 0; i < 8; i++) {
                if constexpr (kHot) {  // hot sources: shared-memory copy
                    const int x = idx[i];
                    val[i] = x < 0 ? 0.0 : (x & kHotBit) ? hot[x & (kHotBit - 1)]
                                                         : __ldg(a.cin + x);
                } else {
                    val[i] = idx[i] >= 0 ? __ldg(a.cin + idx[i]) : 0.0;
                }
            }
            __syncwarp();
            const unsigned ends = (bm[lane >> 2] >> ((lane & 3) * 8)) & 0xFFu;
            __syncwarp();
            if (lane < kCh / 32) bm[lane] = 0u;
            // ---- lane-local fold: tail = sum after the last end (all 8 if none)
            double tail = 0.0;
#pragma unroll
            for (int i = 0; i < 8; i++) {
                tail = __dadd_rn(tail, val[i]);
                if ((ends >> i) & 1u) tail = 0.0;
            }
            // ---- segmented inclusive scan of (has_end, tail), plus end counts
            bool f = ends != 0u;
            double v = tail;
            int ne = __popc(ends);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const bool fo = __shfl_up_sync(0xffffffffu, f, o);
                const double vo = __shfl_up_sync(0xffffffffu, v, o);
                const int no = __shfl_up_sync(0xffffffffu, ne, o);
                if ((int)lane >= o) {
                    if (!f) v = __dadd_rn(vo, v);
                    f = f || fo;
                    ne += no;
                }
            }
            // exclusive values for this lane
            bool fe = __shfl_up_sync(0xffffffffu, f, 1);
            double ve = __shfl_up_sync(0xffffffffu, v, 1);
            int nbefore = __shfl_up_sync(0xffffffffu, ne, 1);
            if (lane == 0) { fe = false; ve = 0.0; nbefore = 0; }
            const double carry_in = fe ? ve : __dadd_rn(carry, ve);
            const bool f31 = __shfl_sync(0xffffffffu, f, 31);
            const double v31 = __shfl_sync(0xffffffffu, v, 31);
            carry = f31 ? v31 : __dadd_rn(carry, v31);
            // ---- rows whose last slot this lane holds: store their sums
            if (ends) {
                double run = 0.0;
                int j = 0;
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    run = __dadd_rn(run, val[i]);
                    if ((ends >> i) & 1u) {
                        const double total = j == 0 ? __dadd_rn(carry_in, run) : run;
                        const int64_t row = rk_chunk + nbefore + j;
                        if (head_spill && row == first_row) {
                            a.hp[u] = total;  // finished by k_pr_epi
                        } else {
                            a.sums[row - a.K0] = total;
                        }
                        j++;
                        run = 0.0;
                    }
                }
            }
        }
        if (lane == 0) a.tp[u] = carry;
    }
}

__global__ void __launch_bounds__(kBlock, 4) k_pr_units(PrArgs a) {
    pr_bind(a);
    __shared__ uint32_t bitmap[kWarps][kCh / 32];
    pr_units_body<false>(a, bitmap[threadIdx.x >> 5], nullptr);
}

// hotc[h] = contrib of the h-th hot source (one gather per iteration)
__global__ void k_pr_hot_gather(PrArgs a, const int32_t *__restrict__ hot_ids, int H,
                                double *__restrict__ hotc) {
    pr_bind(a);
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x)
        hotc[h] = __ldg(a.cin + hot_ids[h]);
}

// Persistent variant (one 1024-thread block per SM): the block copies the H
// hot contrib values into shared memory once per iteration, then its warps
// walk their units; a gather whose (encoded) source carries kHotBit reads
// the shared copy -- the same value, so the sums are bit-identical.
__global__ void __launch_bounds__(kHotBlock, 1) k_pr_units_hot(PrArgs a, const double *hotc,
                                                             int H) {
    pr_bind(a);
    extern __shared__ double hot_smem[];
    uint32_t *bitmaps = reinterpret_cast<uint32_t *>(hot_smem + H);
    const int4 *src = reinterpret_cast<const int4 *>(hotc);
    int4 *dst = reinterpret_cast<int4 *>(hot_smem);
    for (int i = threadIdx.x; i < (H + 1) / 2; i += blockDim.x) dst[i] = __ldcg(src + i);
    __syncthreads();
    pr_units_body<true>(a, bitmaps + (threadIdx.x >> 5) * (kCh / 32), hot_smem);
}

// pr.sp:17-23 for every non-empty row of the block (coalesced over k).
// Each thread takes kEpi rows strided by the block size: all loads of a
// thread are issued before any store (memory-level parallelism).
// A row whose first and last slots lie in different units (a "spill" row)
// was not summed by k_pr_units: its partials are added here left to right,
// tp of every unit it crosses, then hp of the unit holding its end.
constexpr int kEpi = 1;  // rows per thread; cfg2: 1/2/4/8 -> 239/237/234/221 GTEPS (more blocks beat per-thread MLP)
__global__ void __launch_bounds__(256) k_pr_epi(PrArgs a) {
    pr_bind(a);
    const int64_t nk = a.K1 - a.K0;
    const int64_t base_k = blockIdx.x * (int64_t)(256 * kEpi) + threadIdx.x;
    int32_t v[kEpi];
    double sum[kEpi], r[kEpi];
    int od[kEpi];
#pragma unroll
    for (int j = 0; j < kEpi; j++) {
        const int64_t k = base_k + j * 256;
        v[j] = k < nk ? __ldcs(a.nzrow + a.K0 + k) : -1;
        sum[j] = 0.0;
        const int64_t kk = a.K0 + k;
        // row k starts where row k-1 ends: the previous lane's end (lane 0 loads it)
        const int64_t end = k < nk ? __ldg(a.nzend + kk) : 0;
        int64_t start = __shfl_up_sync(0xffffffffu, end, 1);
        if ((threadIdx.x & 31) == 0) start = (k < nk && kk > 0) ? __ldg(a.nzend + kk - 1) : 0;
        if (k < nk) {
            const int64_t us = start / kUnit, ue = (end - 1) / kUnit;
            if (us == ue) {
                sum[j] = __ldcs(a.sums + k);
            } else {
                double acc = 0.0;
                for (int64_t w = us; w < ue; w++) acc = __dadd_rn(acc, a.tp[w - a.u0]);
                sum[j] = __dadd_rn(acc, a.hp[ue - a.u0]);
            }
        }
    }
#pragma unroll
    for (int j = 0; j < kEpi; j++) {
        r[j] = v[j] >= 0 ? a.rank[v[j] - a.v0] : 0.0;
        od[j] = v[j] >= 0 ? __ldg(a.outdeg + v[j]) : 0;
    }
    double dmax = 0.0;
#pragma unroll
    for (int j = 0; j < kEpi; j++) {
        if (v[j] < 0) continue;
        const double nr = __dadd_rn(a.base, __dmul_rn(a.damping, sum[j]));
        double d = __dsub_rn(nr, r[j]);
        if (d < 0.0) d = __dsub_rn(0.0, d);
        dmax = fmax(dmax, d);
        a.rank[v[j] - a.v0] = nr;
        a.cout[v[j] - a.v0] = od[j] > 0 ? __ddiv_rn(nr, (double)od[j]) : 0.0;
    }
    block_diff(a, dmax);
}

// Rows without in-edges: newRank = base (sum = 0).  cout2 (optional) is the
// other contrib buffer of the single-GPU ping-pong.
__global__ void __launch_bounds__(256) k_pr_zero(PrArgs a, const int32_t *__restrict__ indeg,
                                                 int64_t v1, double *cout2) {
    pr_bind(a);
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double dmax = 0.0;
    if (i < v1 - a.v0 && __ldcs(indeg + a.v0 + i) == 0) {
        dmax = pr_apply(a, a.v0 + i, 0.0);
        if (cout2) cout2[i] = a.cout[i];
    }
    block_diff(a, dmax);
}

// unit_row[u] = first nz row in [K0, K1) whose end exceeds the unit start.
__global__ void k_pr_setup(const int64_t *__restrict__ nzend, int64_t K0, int64_t K1, int64_t S0,
                           int64_t u0, int64_t nunits, int64_t *unit_row) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nunits;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s0 = max(S0, (u0 + u) * kUnit);
        int64_t lo = K0, hi = K1;
        while (lo < hi) {
            const int64_t mid = lo + ((hi - lo) >> 1);
            if (nzend[mid] <= s0) lo = mid + 1; else hi = mid;
        }
        unit_row[u] = lo;
    }
}

// out = {roff[v0], roff[v1], K0, K1}: the block's slot range and its nz
// rows (first index in nzrow with nzrow[k] >= v0 / v1).
__global__ void k_pr_bounds(const int64_t *__restrict__ roff, const int32_t *__restrict__ nzrow,
                            int64_t nnz, int64_t v0, int64_t v1, int64_t *out) {
    const int t = threadIdx.x;
    if (t < 2) {
        out[t] = roff[t == 0 ? v0 : v1];
    } else if (t < 4) {
        const int64_t want = t == 2 ? v0 : v1;
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = lo + ((hi - lo) >> 1);
            if (nzrow[mid] < want) lo = mid + 1; else hi = mid;
        }
        out[t] = lo;
    }
}

// ---- hot-source set (per graph, built once) ---------------------------

std::mutex g_hot_mu;
constexpr int64_t kHotMinSlots = 1 << 20;  // smaller graphs keep the plain kernel
constexpr double kHotMinCover = 0.25;  // hot sources must cover >= 25% of the slots (RMAT-24 at 0.307: 9.54 -> 8.83 ms)

__global__ void k_hot_keys(const int32_t *__restrict__ outdeg, int64_t n, uint32_t *key,
                           int32_t *id, int32_t *hot_idx) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        key[v] = (uint32_t)outdeg[v];
        id[v] = (int32_t)v;
        hot_idx[v] = -1;
    }
}

__global__ void k_hot_scatter(const int32_t *__restrict__ ids, int H, int32_t *hot_idx) {
    for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x)
        hot_idx[ids[h]] = h;
}

__global__ void k_hot_encode(const int32_t *__restrict__ radj, int64_t m,
                             const int32_t *__restrict__ hot_idx, int32_t *out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t u = radj[k];
        const int32_t h = hot_idx[u];
        out[k] = h >= 0 ? (kHotBit | h) : u;
    }
}

// Hot-set selection: the H sources of largest out-degree, if they cover at
// least kHotMinCover of the slots.  On success g->pr_hot_ids is set (H
// resident ids), *hot_idx (call scratch, n entries: hot index or -1) and *H_out
// are returned; otherwise *H_out = 0.
int pr_hot_select(sp_graph *g, Call &c, const int32_t *outdeg, int64_t max_outdeg,
                  int32_t **hot_idx_out, int *H_out) {
    *H_out = 0;
    *hot_idx_out = nullptr;
    const int64_t n = g->n, m = g->m;
    const char *ce = getenv("SP_PR_HOT_COVER");  // tuning override of kHotMinCover
    const double min_cover = ce ? atof(ce) : kHotMinCover;
    // free upper bound on the coverage: H sources of at most max_outdeg
    // slots each (a grid decides here, without the sort)
    if (m < kHotMinSlots || n >= kHotBit ||
        (double)std::min<int64_t>(kHotMax, n) * (double)max_outdeg < min_cover * (double)m)
        return SP_OK;
    const int H = (int)std::min<int64_t>(kHotMax, n);
    uint32_t *key, *key_s;
    int32_t *id, *id_s, *hot_idx;
    SP_TRY(c.alloc(&key, n));
    SP_TRY(c.alloc(&key_s, n));
    SP_TRY(c.alloc(&id, n));
    SP_TRY(c.alloc(&id_s, n));
    SP_TRY(c.alloc(&hot_idx, n));
    k_hot_keys<<<grid_for(n, 256, c.device, 16), 256, 0, c.stream>>>(outdeg, n, key, id, hot_idx);
    size_t tmp = 0;
    SP_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, key, key_s, id, id_s, n, 0,
                                                      32, c.stream));
    void *dt = nullptr;
    SP_TRY(scratch_alloc(&dt, tmp, c.stream));
    cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(dt, tmp, key, key_s, id, id_s, n,
                                                              0, 32, c.stream);
    scratch_free(dt, c.stream);
    SP_CUDA(e);
    // coverage: share of the slots whose source is hot (sum of the top H
    // out-degrees); below kHotMinCover the per-iteration refill of the shared
    // copies costs more than the gathers it saves
    unsigned long long *cov;
    SP_TRY(c.alloc(&cov, 1));
    tmp = 0;
    SP_CUDA(cub::DeviceReduce::Sum(nullptr, tmp, key_s, cov, H, c.stream));
    SP_TRY(scratch_alloc(&dt, tmp, c.stream));
    e = cub::DeviceReduce::Sum(dt, tmp, key_s, cov, H, c.stream);
    scratch_free(dt, c.stream);
    SP_CUDA(e);
    unsigned long long *hcov;
    SP_TRY(c.host_as(&hcov));
    SP_CUDA(cudaMemcpyAsync(hcov, cov, 8, cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    if (getenv("SP_PR_HOT_VERBOSE"))
        fprintf(stderr, "pr hot set: top %d sources cover %.3f of the slots\n", H,
                (double)hcov[0] / (double)m);
    if ((double)hcov[0] < min_cover * (double)m) return SP_OK;
    int32_t *ids = nullptr;
    SP_TRY(resident_alloc((void **)&ids, (size_t)H * sizeof(int32_t)));
    SP_CUDA(cudaMemcpyAsync(ids, id_s, (size_t)H * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                            c.stream));
    k_hot_scatter<<<grid_for(H, 256, c.device), 256, 0, c.stream>>>(ids, H, hot_idx);
    c.launches += 3;
    SP_CUDA(cudaGetLastError());
    g->pr_hot_ids = ids;
    *hot_idx_out = hot_idx;
    *H_out = H;
    return SP_OK;
}

int ensure_pr_hot(sp_graph *g, Call &c) {
    std::lock_guard<std::mutex> lk(g_hot_mu);
    if (g->pr_H >= 0) return SP_OK;
    // Built on the graph's second fast PR call: the encoding (a sort of the
    // out-degrees + one pass over radj, ~0.9 ms at cfg2) costs more than it
    // saves in a single run (~0.4 ms), so a one-shot run on a fresh graph
    // keeps the plain kernel (same sums either way).  A large directed graph
    // uploaded with from_csr gets it during the upload (sp_graph.cu).
    const char *ce = getenv("SP_PR_HOT_COVER");
    const double min_cover = ce ? atof(ce) : kHotMinCover;
    if (g->m < kHotMinSlots || g->n >= kHotBit ||
        (double)std::min<int64_t>(kHotMax, g->n) * (double)g->max_outdeg <
            min_cover * (double)g->m) {
        g->pr_H = 0;
        return SP_OK;
    }
    if (g->pr_fast_calls++ == 0) return SP_OK;
    int32_t *hot_idx = nullptr;
    int H = 0;
    SP_TRY(pr_hot_select(g, c, g->outdeg, g->max_outdeg, &hot_idx, &H));
    if (H == 0) {
        g->pr_H = 0;
        return SP_OK;
    }
    int32_t *enc = nullptr;
    SP_TRY(resident_alloc((void **)&enc, (size_t)g->m * sizeof(int32_t)));
    k_hot_encode<<<grid_for(g->m, 256, c.device, 16), 256, 0, c.stream>>>(g->radj, g->m, hot_idx,
                                                                          enc);
    c.launches++;
    SP_CUDA(cudaGetLastError());
    SP_CUDA(cudaStreamSynchronize(c.stream));
    g->pr_radj_hot = enc;
    g->pr_H = H;
    return SP_OK;
}

// Per-call state of the fast path for a vertex block [v0, v1).
struct FastPlan {
    PrArgs a{};
    int grid_units = 1, grid_epi = 1, grid_zero = 1;
    // hot-source variant
    int H = 0, grid_hot = 0;
    size_t hot_smem = 0;
    const int32_t *hot_ids = nullptr;
    double *hotc = nullptr;
};

int plan_fast(sp_graph *g, Call &c, int64_t v0, int64_t v1, double damping, FastPlan &p) {
    int64_t S[2] = {0, g->m}, K[2] = {0, g->nnz_rows};  // the whole graph: known on the host
    if (v0 != 0 || v1 != g->n) {  // a vertex block (multi-GPU): slot and row bounds
        int64_t *kb, *hb;
        SP_TRY(c.alloc(&kb, 4));
        SP_TRY(c.host_as(&hb));
        k_pr_bounds<<<1, 32, 0, c.stream>>>(g->roff, g->nzrow, g->nnz_rows, v0, v1, kb);
        c.launches++;
        SP_CUDA(cudaMemcpyAsync(hb + 8, kb, 32, cudaMemcpyDeviceToHost, c.stream));
        SP_CUDA(cudaStreamSynchronize(c.stream));
        S[0] = hb[8];
        S[1] = hb[9];
        K[0] = hb[10];
        K[1] = hb[11];
    }
    PrArgs &a = p.a;
    a.radj = g->radj;
    a.nzend = g->nzend;
    a.nzrow = g->nzrow;
    a.outdeg = g->outdeg;
    a.v0 = v0;
    a.S0 = S[0];
    a.S1 = S[1];
    a.K0 = K[0];
    a.K1 = K[1];
    a.u0 = S[0] / kUnit;
    a.nunits = S[1] > S[0] ? (S[1] - 1) / kUnit - a.u0 + 1 : 0;
    a.base = (1.0 - damping) / (double)g->n;  // pr.sp:17, no FMA on host either
    a.damping = damping;
    const int64_t nu = std::max<int64_t>(1, a.nunits);
    int64_t *ur;
    SP_TRY(c.alloc(&ur, nu));
    double *hp, *tp, *sums;
    SP_TRY(c.alloc(&sums, std::max<int64_t>(1, a.K1 - a.K0)));
    a.sums = sums;
    SP_TRY(c.alloc(&hp, nu));
    SP_TRY(c.alloc(&tp, nu));
    a.hp = hp;
    a.tp = tp;
    a.unit_row = ur;
    if (a.nunits) {
        k_pr_setup<<<grid_for(a.nunits, 256, c.device), 256, 0, c.stream>>>(
            g->nzend, a.K0, a.K1, a.S0, a.u0, a.nunits, ur);
        c.launches++;
    }
    // one unit per warp, no cap: the block scheduler balances the tail
    p.grid_units = (int)std::max<int64_t>(1, (a.nunits + kWarps - 1) / kWarps);
    SP_TRY(ensure_pr_hot(g, c));
    if (g->pr_H > 0) {
        p.H = g->pr_H;
        p.hot_ids = g->pr_hot_ids;
        a.radj = g->pr_radj_hot;  // encoded slots
        double *hotc;
        SP_TRY(c.alloc(&hotc, p.H + 1));
        p.hotc = hotc;
        p.hot_smem = (size_t)p.H * sizeof(double) + (kHotBlock / 32) * (kCh / 32) * 4;
        SP_CUDA(cudaFuncSetAttribute(k_pr_units_hot, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)p.hot_smem));
        p.grid_hot = num_sms(c.device);
    }
    p.grid_epi = (int)std::max<int64_t>(1, (a.K1 - a.K0 + 256 * kEpi - 1) / (256 * kEpi));
    p.grid_zero = (int)std::max<int64_t>(1, (v1 - v0 + 255) / 256);
    SP_CUDA(cudaGetLastError());
    return SP_OK;
}

// The row-sum kernel of one iteration (hot-source variant when built).
void launch_units(Call &c, const FastPlan &p, const PrArgs &a) {
    if (p.H > 0) {
        k_pr_hot_gather<<<grid_for(p.H, 256, c.device), 256, 0, c.stream>>>(a, p.hot_ids, p.H,
                                                                            p.hotc);
        k_pr_units_hot<<<p.grid_hot, kHotBlock, p.hot_smem, c.stream>>>(a, p.hotc, p.H);
        c.launches += 2;
    } else {
        k_pr_units<<<p.grid_units, kBlock, 0, c.stream>>>(a);
        c.launches++;
    }
}

// One fast iteration; `zero` says whether zero-in-degree rows are written.
int launch_fast(Call &c, FastPlan &p, sp_graph *g, int64_t v1, const double *cin, double *rank,
                double *cout, double *cout2, bool zero, double *diff_slot, cudaEvent_t ka,
                cudaEvent_t kb) {
    PrArgs a = p.a;
    a.cin = cin;
    a.rank = rank;
    a.cout = cout;
    a.diff_slot = diff_slot;
    if (ka) cudaEventRecord(ka, c.stream);
    if (a.nunits) {
        launch_units(c, p, a);
        k_pr_epi<<<p.grid_epi, 256, 0, c.stream>>>(a);
        c.launches += 1;
    }
    if (kb) cudaEventRecord(kb, c.stream);
    if (zero) {
        k_pr_zero<<<p.grid_zero, 256, 0, c.stream>>>(a, g->indeg, v1, cout2);
        c.launches++;
    }
    SP_CUDA(cudaGetLastError());
    return SP_OK;
}

__global__ void k_pr_advance(PrLoop *L, cudaGraphConditionalHandle h) {
    const int cur = L->cur;
    const double diff = *L->slot[cur];
    L->diff = diff;
    L->iter++;
    L->iters++;
    int go = !(diff < L->eps || L->iter >= L->max_iter);  // pr.sp:10
    if (go && L->iters >= L->cap) {
        L->status = 2;
        go = 0;
    }
    *L->slot[cur ^ 1] = 0.0;
    L->cur = cur ^ 1;
    cudaGraphSetConditional(h, go);
}

// Iterations 2.. of the fast path as one graph launch (no host round trip
// per iteration).  `hL` receives the final loop state.
int pr_device_loop(Call &c, FastPlan &p, double *rank, double *c0, double *c1, double *s0,
                   double *s1, int64_t iter0, int64_t iters0, int64_t max_iter, int64_t cap,
                   double eps, PrLoop *hL, float *kernel_ms) {
    PrLoop *L;
    SP_TRY(c.alloc(&L, 1));
    PrLoop init{};
    init.c[0] = c0;
    init.c[1] = c1;
    init.slot[0] = s0;
    init.slot[1] = s1;
    init.iter = iter0;
    init.iters = iters0;
    init.max_iter = max_iter;
    init.cap = cap;
    init.eps = eps;
    SP_CUDA(cudaMemcpyAsync(L, &init, sizeof(PrLoop), cudaMemcpyHostToDevice, c.stream));
    SP_CUDA(cudaMemsetAsync(s0, 0, sizeof(double), c.stream));
    PrArgs a = p.a;
    a.rank = rank;
    a.loop = L;
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
    if (a.nunits) {
        launch_units(c, p, a);
        k_pr_epi<<<p.grid_epi, 256, 0, c.stream>>>(a);
    }
    k_pr_advance<<<1, 1, 0, c.stream>>>(L, h);
    SP_CUDA(cudaStreamEndCapture(c.stream, &body));
    cudaEvent_t ka, kb;
    SP_CUDA(cudaEventCreate(&ka));
    SP_CUDA(cudaEventCreate(&kb));
    cudaEventRecord(ka, c.stream);
    SP_TRY(launch_cached_graph(graph, p.a.radj, kLoopPr, c.stream));
    cudaEventRecord(kb, c.stream);
    SP_CUDA(cudaMemcpyAsync(hL, L, sizeof(PrLoop), cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    cudaEventElapsedTime(kernel_ms, ka, kb);
    cudaEventDestroy(ka);
    cudaEventDestroy(kb);
    c.launches += (hL->iters - iters0) * 3;
    return SP_OK;
}

// ---------------------------------------------------------------- exact path

// One PageRank iteration for vertices [v0, v1), bit-identical to the
// interpreter's left fold.  contrib_in: full n-array (global ids);
// rank/contrib_out: local, index v-v0.
__global__ void __launch_bounds__(kBlock) k_pull_exact(
    const int64_t *__restrict__ roff, const int32_t *__restrict__ radj,
    const int32_t *__restrict__ outdeg, const double *__restrict__ contrib_in,
    double *__restrict__ rank, double *__restrict__ contrib_out, int64_t v0, int64_t v1,
    double base, double damping, double *diff_slot) {
    __shared__ double stage[kWarps][kChunk];
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
        const int64_t deg = re - rs;
        // the tile's rows are one contiguous slab radj[roff[t0] .. roff[t0+32])
        int64_t incl = deg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t tt = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)lane >= o) incl += tt;
        }
        const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
        const int64_t excl = incl - deg;
        const int64_t sb = __shfl_sync(0xffffffffu, rs, 0);
        double sum = 0.0;
        for (int64_t p0 = 0; p0 < total; p0 += kChunk) {
#pragma unroll
            for (int j = 0; j < kChunk / 32; j++) {
                const int64_t p = p0 + j * 32 + lane;
                buf[j * 32 + lane] = p < total ? contrib_in[radj[sb + p]] : 0.0;
            }
            __syncwarp();
            // sequential left fold of this lane's slice of the chunk
            int64_t lo = max(excl, p0), hi = min(excl + deg, p0 + (int64_t)kChunk);
            for (int64_t p = lo; p < hi; p++) sum = __dadd_rn(sum, buf[p - p0]);
            __syncwarp();
        }
        if (live) {
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
    if (lane == 0 && dmax > 0.0) atomic_max_nonneg(diff_slot, dmax);
}

int launch_exact(sp_graph *g, Call &c, int64_t v0, int64_t v1, double damping, const double *cin,
                 double *rank, double *cout, double *diff_slot, cudaEvent_t ka, cudaEvent_t kb) {
    const double base = (1.0 - damping) / (double)g->n;  // pr.sp:17
    int64_t tiles = (v1 - v0 + 31) / 32;
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>((tiles + kWarps - 1) / kWarps,
                                                           (int64_t)num_sms(c.device) * 8));
    if (ka) cudaEventRecord(ka, c.stream);
    k_pull_exact<<<grid, kBlock, 0, c.stream>>>(g->roff, g->radj, g->outdeg, cin, rank, cout, v0,
                                                v1, base, damping, diff_slot);
    if (kb) cudaEventRecord(kb, c.stream);
    c.launches++;
    SP_CUDA(cudaGetLastError());
    return SP_OK;
}

}  // namespace

namespace sp {
int pr_hot_prepare(sp_graph *g, Call &c, const int32_t *outdeg, int64_t max_outdeg,
                   int32_t **hot_idx, int *H) {
    static_assert(kHotBit == kPrHotBit, "hot-slot encoding");
    return pr_hot_select(g, c, outdeg, max_outdeg, hot_idx, H);
}
}  // namespace sp

extern "C" int sp_pagerank(sp_graph *g, double damping, double epsilon, int64_t max_iter,
                           int64_t cap, unsigned flags, double *rank_out, int mem,
                           int64_t *iter_out, double *diff_out, int64_t *iters_out,
                           sp_iter_cb cb, void *user, sp_stats *st) {
    SP_CHECK(g && (rank_out || g->n == 0), SP_ERR_ARG, "sp_pagerank: bad arguments");
    Call c;
    SP_TRY(c.begin(g->device));
    const int64_t n = g->n;
    const bool exact = flags & SP_FLAG_DETERMINISTIC;
    double *rank, *ca, *cb2, *diffs;
    SP_TRY(c.alloc(&rank, n));
    SP_TRY(c.alloc(&ca, n));
    SP_TRY(c.alloc(&cb2, n));
    const int64_t kSlots = 1024;  // diff slots, recycled in a ring
    SP_TRY(c.alloc(&diffs, kSlots));
    SP_CUDA(cudaMemsetAsync(diffs, 0, kSlots * sizeof(double), c.stream));
    double *hdiff = nullptr;
    SP_TRY(c.host_as(&hdiff));
    FastPlan plan;
    if (n && !exact) SP_TRY(plan_fast(g, c, 0, n, damping, plan));
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
            rc = exact ? launch_exact(g, c, 0, n, damping, ca, rank, cb2, slot, ka, kb)
                       : launch_fast(c, plan, g, n, ca, rank, cb2, ca, iters == 0, slot, ka, kb);
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
        const char *hostloop = getenv("SP_HOSTLOOP");  // ncu cannot profile conditional graphs
        if (!cb && !exact && n && !(hostloop && hostloop[0] == '1')) {
            // the remaining iterations on the device: contrib to read is ca
            PrLoop *hL;
            SP_TRY(c.host_as(&hL));
            float ms = 0.f;
            SP_TRY(pr_device_loop(c, plan, rank, ca, cb2, diffs, diffs + 1, iter, iters,
                                  max_iter, cap, epsilon, hL, &ms));
            kernel_ms += ms;
            iter = hL->iter;
            iters = hL->iters;
            diff = hL->diff;
            if (hL->status == 2) {
                set_error("fixedPoint 'converged' did not converge within %lld iterations",
                          (long long)cap);
                rc = SP_ERR_NONCONV;
            }
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
        // per iteration 12 B per slot (radj 4 + contrib gather 8)
        // + 36 B per vertex (roff 8, rank r/w 16, contrib write 8, outdeg 4)
        st->model_bytes = iters * (12 * g->m + 36 * n);
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
    double *slot;
    SP_TRY(c.alloc(&slot, 1));
    SP_CUDA(cudaMemsetAsync(slot, 0, sizeof(double), c.stream));
    if (v1 > v0) {
        if (flags & SP_FLAG_DETERMINISTIC) {
            SP_TRY(launch_exact(g, c, v0, v1, damping, contrib_in, rank_local, contrib_out, slot,
                                nullptr, nullptr));
        } else {
            FastPlan plan;
            SP_TRY(plan_fast(g, c, v0, v1, damping, plan));
            // contrib_out is a single persistent buffer here: zero rows are
            // rewritten every step (cheap: one indeg pass over the block)
            SP_TRY(launch_fast(c, plan, g, v1, contrib_in, rank_local, contrib_out, nullptr, true,
                               slot, nullptr, nullptr));
        }
    }
    SP_CUDA(cudaMemcpyAsync(diff, slot, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    SP_TRY(c.finish(st));
    return SP_OK;
}
