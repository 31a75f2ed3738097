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
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <stdlib.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <mutex>
#include <utility>

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
    // multi-GPU shards: every contrib this block computes is also stored at
    // peers[q][v] (v global) -- the other ranks' contrib arrays, mapped over
    // NVLink (CUDA IPC): the exchange rides on the producing kernel
    double *const *peers;
    int npeers;
};

__device__ __forceinline__ void pr_store_contrib(const PrArgs &a, int64_t v, double c) {
    a.cout[v - a.v0] = c;
    for (int q = 0; q < a.npeers; q++) a.peers[q][v] = c;
}

// Device-side fixedPoint loop state (pr.sp:10), one per call, in the
// argument block of the thread's cached executable (ArgExec): every per-call
// value lives here, so the captured kernels never change.  Contrib buffers:
// c0 holds rank0/outdeg (iteration 1 reads it); c1/c2 ping-pong from
// iteration 2 on (iteration i writes c1 when i is odd, c2 when even).  Rows
// without in-edges are constant from iteration 1 on, so k_pr_init writes
// their final rank and contrib (in c1 and c2) up front, and their
// |delta| = |base - rank0| into iteration 1's diff slot.
struct PrLoop {
    double *c0, *c1, *c2;
    double *rank, *sums, *hp, *tp;
    double *rank_out;  // relabelled layout: the final ranks in vertex order
    double base, damping, eps;
    double slot[2];  // diff of odd / even iterations
    int64_t iter, iters, max_iter, cap;
    double diff;
    int status;  // 0 running/converged, 2 cap reached
};

// pr.sp:10 after an iteration: diff, iter++, stop test; the next
// iteration's diff slot is cleared.  In a graph, sets the WHILE condition.
__device__ __forceinline__ void pr_advance(PrLoop *L, cudaGraphConditionalHandle h, bool in_graph) {
    const int64_t i = L->iters + 1;  // the iteration just computed
    const double diff = __longlong_as_double(
        (long long)__ldcg(reinterpret_cast<const unsigned long long *>(L->slot + (i & 1))));
    L->diff = diff;
    L->iter++;
    L->iters = i;
    int go = !(diff < L->eps || L->iter >= L->max_iter);  // pr.sp:10
    if (go && L->iters >= L->cap) {
        L->status = 2;
        go = 0;
    }
    L->slot[(i + 1) & 1] = 0.0;
    if (in_graph) cudaGraphSetConditional(h, go);
}

// Programmatic dependent launch: the kernels of one iteration are launched
// with programmatic stream serialisation (launch_pdl), so a kernel's blocks
// become resident while its predecessor drains; they wait here until the
// predecessor's writes are visible (a no-op for ordinary launches).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void pr_bind(PrArgs &a) {
    griddep_wait();
    if (a.loop) {
        const PrLoop *L = a.loop;
        const int64_t i = L->iters + 1;  // the iteration being computed (1-based)
        const bool odd = i & 1;
        a.cin = i == 1 ? L->c0 : odd ? L->c2 : L->c1;
        a.cout = odd ? L->c1 : L->c2;
        a.diff_slot = a.loop->slot + (odd ? 1 : 0);
        a.rank = L->rank;
        a.sums = L->sums;
        a.hp = L->hp;
        a.tp = L->tp;
        a.base = L->base;
        a.damping = L->damping;
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
    pr_store_contrib(a, v, od > 0 ? __ddiv_rn(nr, (double)od) : 0.0);
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
// kMode: kPlain (every gather from cin), kEnc (radj slots carry kHotBit |
// hot index for the hot sources), kRel (relabelled layout: sources are
// ranked by out-degree, the hot ones are exactly the ids below relH).
enum { kPlain = 0, kEnc = 1, kRel = 2, kEnc2 = 3 };
// kEnc2: a hot set split over a CTA pair (thread-block cluster): hot index
// h lives in CTA h / relH's shared memory -- this CTA's (rank `my`) or the
// peer's, read through distributed shared memory (`peer`).
template <int kMode>
__device__ __forceinline__ void pr_units_body(const PrArgs &a, uint32_t *bm, const double *hot,
                                              int relH = 0, const double *peer = nullptr,
                                              int my = 0) {
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
                if constexpr (kMode == kEnc) {  // hot sources: shared-memory copy
                    const int x = idx[i];
                    val[i] = x < 0 ? 0.0 : (x & kHotBit) ? hot[x & (kHotBit - 1)]
                                                         : __ldg(a.cin + x);
                } else if constexpr (kMode == kRel) {
                    const int x = idx[i];
                    val[i] = x < 0 ? 0.0 : x < relH ? hot[x] : __ldg(a.cin + x);
                } else if constexpr (kMode == kEnc2) {
                    const int x = idx[i];
                    if (x < 0) {
                        val[i] = 0.0;
                    } else if (x & kHotBit) {
                        const int h = x & (kHotBit - 1);
                        const int ow = h >= relH ? 1 : 0;
                        const int off = h - ow * relH;
                        val[i] = ow == my ? hot[off] : peer[off];
                    } else {
                        val[i] = __ldg(a.cin + x);
                    }
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
    pr_units_body<kPlain>(a, bitmap[threadIdx.x >> 5], nullptr);
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
    pr_units_body<kEnc>(a, bitmaps + (threadIdx.x >> 5) * (kCh / 32), hot_smem);
}

// Cluster variant (hot sets beyond one CTA's shared memory, SP_PR_HOT_MAX):
// CTA pairs, each holding half of the H hot contribs; a gather whose hot
// index lies in the peer's half reads it through distributed shared memory.
// The pair synchronises after the refill (the peer's half is complete) and
// before exiting (its shared memory stays readable until the peer is done).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kHotBlock, 1)
    k_pr_units_hot2(PrArgs a, const double *hotc, int H) {
    pr_bind(a);
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ double hot_smem[];
    const int Hl = ((H + 1) / 2 + 1) & ~1;  // even: int4 refills
    const int my = (int)cl.block_rank();
    uint32_t *bitmaps = reinterpret_cast<uint32_t *>(hot_smem + Hl);
    const int lo = my * Hl, cnt = min(Hl, H - lo);
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) hot_smem[i] = __ldcg(hotc + lo + i);
    cl.sync();
    const double *peer = cl.map_shared_rank(hot_smem, my ^ 1);
    pr_units_body<kEnc2>(a, bitmaps + (threadIdx.x >> 5) * (kCh / 32), hot_smem, Hl, peer, my);
    cl.sync();
}

// Relabelled layout: the hot contribs are cin[0, H) -- one contiguous copy
// into shared memory per block, no gather kernel.
__global__ void __launch_bounds__(kHotBlock, 1) k_pr_units_rel(PrArgs a, int H) {
    pr_bind(a);
    extern __shared__ double hot_smem[];
    uint32_t *bitmaps = reinterpret_cast<uint32_t *>(hot_smem + H);
    const int4 *src = reinterpret_cast<const int4 *>(a.cin);
    int4 *dst = reinterpret_cast<int4 *>(hot_smem);
    for (int i = threadIdx.x; i < H / 2; i += blockDim.x) dst[i] = __ldcg(src + i);
    __syncthreads();
    pr_units_body<kRel>(a, bitmaps + (threadIdx.x >> 5) * (kCh / 32), hot_smem, H);
}

// pr.sp:17-23 for every non-empty row of the block (coalesced over k).
// Each thread takes kEpi rows strided by the block size: all loads of a
// thread are issued before any store (memory-level parallelism).
// A row whose first and last slots lie in different units (a "spill" row)
// was not summed by k_pr_units: its partials are added here left to right,
// tp of every unit it crosses, then hp of the unit holding its end.
#ifndef SP_PR_EPI_ROWS
#define SP_PR_EPI_ROWS 2
#endif
// rows per thread; round 1 cfg2: 1/2/4/8 -> 239/237/234/221 GTEPS; round 2
// (unrolled init, same box): 1 -> 2.90 / 7.85 ms, 2 -> 2.87 / 7.80 ms,
// 4 -> 2.90 / 7.86 ms (cfg2 / RMAT-24 per run)
constexpr int kEpi = SP_PR_EPI_ROWS;
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
        pr_store_contrib(a, v[j], od[j] > 0 ? __ddiv_rn(nr, (double)od[j]) : 0.0);
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

// Hot-set size: kHotMax (one CTA's shared memory); SP_PR_HOT_MAX up to
// 2 x kHotMax splits the set over a CTA pair (k_pr_units_hot2).
static int hot_max() {
    static const int h = [] {
        const char *e = getenv("SP_PR_HOT_MAX");
        const int v = e ? atoi(e) : kHotMax;
        return std::max(2, std::min(2 * kHotMax - 4, v)) & ~1;
    }();
    return h;
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
        (double)std::min<int64_t>(hot_max(), n) * (double)max_outdeg < min_cover * (double)m)
        return SP_OK;
    const int H = (int)std::min<int64_t>(hot_max(), n);
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

static int hot_build_locked(sp_graph *g, Call &c, bool now);

int pr_hot_build_impl(sp_graph *g, Call &c) {
    std::lock_guard<std::mutex> lk(g_hot_mu);
    if (g->pr_H >= 0) return SP_OK;
    return hot_build_locked(g, c, true);
}

int ensure_pr_hot(sp_graph *g, Call &c) {
    std::lock_guard<std::mutex> lk(g_hot_mu);
    if (g->pr_H >= 0) return SP_OK;
    return hot_build_locked(g, c, false);
}

static int hot_build_locked(sp_graph *g, Call &c, bool now) {
    // Built on the graph's second fast PR call: the encoding (a sort of the
    // out-degrees + one pass over radj, ~0.9 ms at cfg2) costs more than it
    // saves in a single run (~0.4 ms), so a one-shot run on a fresh graph
    // keeps the plain kernel (same sums either way).  A large directed graph
    // uploaded with from_csr gets it during the upload (sp_graph.cu).
    const char *ce = getenv("SP_PR_HOT_COVER");
    const double min_cover = ce ? atof(ce) : kHotMinCover;
    if (g->m < kHotMinSlots || g->n >= kHotBit ||
        (double)std::min<int64_t>(hot_max(), g->n) * (double)g->max_outdeg <
            min_cover * (double)g->m) {
        g->pr_H = 0;
        return SP_OK;
    }
    if (!now && g->pr_fast_calls++ == 0) return SP_OK;
    prep_mark(g, kPrepPrHot, 0, c.stream);
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
    prep_mark(g, kPrepPrHot, 1, c.stream);
    c.launches++;
    SP_CUDA(cudaGetLastError());
    SP_CUDA(cudaStreamSynchronize(c.stream));
    g->pr_radj_hot = enc;
    g->pr_H = H;
    return SP_OK;
}

// ---- relabelled layout (per graph, built once) ---------------------------
//
// The pull's cost is one L1/shared-memory wavefront per distinct line or
// bank group a warp's gather instruction touches, and random source ids put
// every lane of an instruction on its own line.  Ranking the vertices by
// out-degree packs the sources that are gathered most into a dense prefix
// (the hot ones, ranks < H, are a contiguous shared-memory copy), and each
// row's sources are stored as ascending ranks, placed within every 256-slot
// chunk so that load instruction i of lane l (slot 8l + i) reads the row's
// (32i + l)-th element: one instruction reads 32 consecutive ranks of the
// row -- conflict-free shared-memory banks for the hot part, shared lines
// for the dense warm part.  Same per-row multiset of contribs, so the same
// fast-mode sums up to the association order (fast mode only).

__global__ void k_rel_rank(const int32_t *__restrict__ order, const uint32_t *__restrict__ deg_s,
                           int64_t n, int32_t *perm, int32_t *rel_outdeg,
                           const int32_t *__restrict__ indeg, int32_t *rel_indeg) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = order[r];
        perm[v] = (int32_t)r;
        rel_outdeg[r] = (int32_t)deg_s[r];
        rel_indeg[r] = indeg[v];
    }
}

__global__ void k_rel_rowmark(const int64_t *__restrict__ roff, int64_t n, uint32_t *mark) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x)
        if (roff[v + 1] > roff[v]) mark[roff[v]] = (uint32_t)v;
}

__global__ void k_rel_keys(const uint32_t *__restrict__ rowof, const int32_t *__restrict__ radj,
                           const int32_t *__restrict__ perm, int64_t m, int b, uint64_t *key) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
         k += (int64_t)gridDim.x * blockDim.x)
        key[k] = ((uint64_t)(uint32_t)perm[rowof[k]] << b) | (uint32_t)perm[radj[k]];
}

// roff[x] = first slot whose row (key >> b) is >= x, x in [0, n]
__global__ void k_rel_offsets(const uint64_t *__restrict__ key, int64_t m, int64_t n, int b,
                              int64_t *roff) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t prev = e == 0 ? -1 : (int64_t)(key[e - 1] >> b);
        const int64_t cur = e == m ? n : (int64_t)(key[e] >> b);
        for (int64_t x = prev + 1; x <= cur; x++) roff[x] = e;
    }
}

__global__ void k_rel_nzend(const int64_t *__restrict__ roff, const int32_t *__restrict__ nzrow,
                            const int64_t *__restrict__ cnt, int64_t *nzend) {
    const int64_t k1 = *cnt;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < k1;
         k += (int64_t)gridDim.x * blockDim.x)
        nzend[k] = roff[nzrow[k] + 1];
}

// number of q in [0, x) with q % 8 == r
__device__ __forceinline__ int64_t rel_cnt(int64_t x, int r) { return x > r ? (x - r + 7) >> 3 : 0; }

// Within the part [a, b) of a row that lies in one 256-slot chunk, the
// positions are filled in the order (q % 8, q / 8) of their chunk offset q:
// the element of sorted rank k goes to the k-th position in that order.
__global__ void k_rel_place(const uint64_t *__restrict__ key, int64_t m, int b,
                            const int64_t *__restrict__ roff, int32_t *out) {
    const uint64_t mask = (uint64_t(1) << b) - 1;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = (int64_t)(key[p] >> b);
        const int64_t c0 = p & ~int64_t(kCh - 1);
        const int64_t a = max(roff[row], c0), e = min(roff[row + 1], c0 + kCh);
        const int64_t lo = a - c0, hi = e - c0, pp = p - c0;
        const int rp = (int)(pp & 7);
        int64_t k = rel_cnt(pp, rp) - rel_cnt(lo, rp);
        for (int r = 0; r < rp; r++) k += rel_cnt(hi, r) - rel_cnt(lo, r);
        out[p] = (int32_t)(key[a + k] & mask);
    }
}

struct NonEmptyRank {
    const int32_t *deg;
    __device__ __forceinline__ bool operator()(int32_t x) const { return deg[x] > 0; }
};

struct MaxRow {
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const {
        return a > b ? a : b;
    }
};

int bits_for_n(int64_t n) {
    int b = 1;
    while (b < 62 && ((int64_t)1 << b) < n) b++;
    return b;
}

// Builds the relabelled layout when the hot-source criterion holds (the
// graph is skewed enough for a shared-memory hot set); otherwise pr_rel = 0.
int ensure_pr_rel(sp_graph *g, Call &c) {
    std::lock_guard<std::mutex> lk(g_hot_mu);
    if (g->pr_rel >= 0) return SP_OK;
    const char *re = getenv("SP_PR_REL");
    const char *ce = getenv("SP_PR_HOT_COVER");
    const double min_cover = ce ? atof(ce) : kHotMinCover;
    const int64_t n = g->n, m = g->m;
    // Where it pays (measured, B200, RMAT ef16, ms per run rel / encoded):
    // the contrib array 8n must exceed the L2 (the ranking then keeps the
    // gathered sources' lines L2-resident: RMAT-24 7.68 / 8.26) but not by
    // far (RMAT-26: 38.3 / 32.4 -- the final unpermute pass and the
    // scattered rank-order rows cost more); an L2-resident contrib gains
    // nothing (RMAT-22: 2.98 / 2.92).  SP_PR_REL=1 forces it, =0 disables.
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, c.device);
    const bool in_band = 8.0 * (double)n > (double)l2 && 8.0 * (double)n <= 2.5 * (double)l2;
    const bool force = re && re[0] == '1';
    if ((re && re[0] == '0') || (!force && !in_band) || m < kHotMinSlots || n >= kHotBit ||
        2 * bits_for_n(n) > 64 ||
        (double)std::min<int64_t>(kHotMax, n) * (double)g->max_outdeg < min_cover * (double)m) {
        g->pr_rel = 0;
        return SP_OK;
    }
    const int b = bits_for_n(n);
    prep_mark(g, kPrepPrRel, 0, c.stream);
    // out-degree ranking (stable: ties by id) and the hot coverage
    uint32_t *key, *key_s;
    int32_t *id, *id_s;
    SP_TRY(c.alloc(&key, n));
    SP_TRY(c.alloc(&key_s, n));
    SP_TRY(c.alloc(&id, n));
    SP_TRY(c.alloc(&id_s, n));
    int32_t *hot_dummy;
    SP_TRY(c.alloc(&hot_dummy, n));
    k_hot_keys<<<grid_for(n, 256, c.device, 16), 256, 0, c.stream>>>(g->outdeg, n, key, id,
                                                                     hot_dummy);
    size_t tmp = 0;
    SP_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, key, key_s, id, id_s, n, 0,
                                                      32, c.stream));
    void *dt = nullptr;
    SP_TRY(scratch_alloc(&dt, tmp, c.stream));
    cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(dt, tmp, key, key_s, id, id_s, n,
                                                              0, 32, c.stream);
    scratch_free(dt, c.stream);
    SP_CUDA(e);
    const int H = (int)(std::min<int64_t>(kHotMax, n) & ~int64_t(1));
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
    if ((double)hcov[0] < min_cover * (double)m) {
        g->pr_rel = 0;
        return SP_OK;
    }
    int32_t *perm = nullptr, *radj = nullptr, *outd = nullptr, *ind = nullptr, *nzrow = nullptr;
    int64_t *nzend = nullptr, *ur = nullptr;
    struct Guard {  // frees the resident arrays unless the build completes
        int32_t **a[5];
        int64_t **b[2];
        bool ok = false;
        ~Guard() {
            if (ok) return;
            for (auto p : a) resident_free(*p);
            for (auto p : b) resident_free(*p);
        }
    } guard{{&perm, &radj, &outd, &ind, &nzrow}, {&nzend, &ur}};
    SP_TRY(resident_alloc((void **)&perm, (size_t)n * 4 + 16));
    SP_TRY(resident_alloc((void **)&radj, (size_t)m * 4 + 16));
    SP_TRY(resident_alloc((void **)&outd, (size_t)n * 4 + 16));
    SP_TRY(resident_alloc((void **)&ind, (size_t)n * 4 + 16));
    SP_TRY(resident_alloc((void **)&nzrow, (size_t)n * 4 + 16));
    SP_TRY(resident_alloc((void **)&nzend, (size_t)n * 8 + 16));
    k_rel_rank<<<grid_for(n, 256, c.device, 16), 256, 0, c.stream>>>(id_s, key_s, n, perm, outd,
                                                                     g->indeg, ind);
    // the reverse CSR in rank order: sort (rank of row, rank of source)
    uint32_t *rowof;
    uint64_t *k0, *k1;
    SP_TRY(c.alloc(&rowof, m));
    SP_TRY(c.alloc(&k0, m));
    SP_TRY(c.alloc(&k1, m));
    SP_CUDA(cudaMemsetAsync(rowof, 0, (size_t)m * 4, c.stream));
    k_rel_rowmark<<<grid_for(n, 256, c.device, 16), 256, 0, c.stream>>>(g->roff, n, rowof);
    tmp = 0;
    SP_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tmp, rowof, rowof, MaxRow(), m,
                                           c.stream));
    SP_TRY(scratch_alloc(&dt, tmp, c.stream));
    e = cub::DeviceScan::InclusiveScan(dt, tmp, rowof, rowof, MaxRow(), m,
                                       c.stream);
    scratch_free(dt, c.stream);
    SP_CUDA(e);
    k_rel_keys<<<grid_for(m, 256, c.device, 16), 256, 0, c.stream>>>(rowof, g->radj, perm, m, b,
                                                                     k0);
    tmp = 0;
    SP_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, k0, k1, m, 0, 2 * b, c.stream));
    SP_TRY(scratch_alloc(&dt, tmp, c.stream));
    e = cub::DeviceRadixSort::SortKeys(dt, tmp, k0, k1, m, 0, 2 * b, c.stream);
    scratch_free(dt, c.stream);
    SP_CUDA(e);
    int64_t *roff2;
    SP_TRY(c.alloc(&roff2, n + 1));
    k_rel_offsets<<<grid_for(m + 1, 256, c.device, 16), 256, 0, c.stream>>>(k1, m, n, b, roff2);
    k_rel_place<<<grid_for(m, 256, c.device, 16), 256, 0, c.stream>>>(k1, m, b, roff2, radj);
    // non-empty rows in rank order and their ends
    int64_t *nsel;
    SP_TRY(c.alloc(&nsel, 1));
    NonEmptyRank pred{ind};
    tmp = 0;
    SP_CUDA(cub::DeviceSelect::If(nullptr, tmp, thrust::counting_iterator<int32_t>(0), nzrow, nsel,
                                  n, pred, c.stream));
    SP_TRY(scratch_alloc(&dt, tmp, c.stream));
    e = cub::DeviceSelect::If(dt, tmp, thrust::counting_iterator<int32_t>(0), nzrow, nsel, n, pred,
                              c.stream);
    scratch_free(dt, c.stream);
    SP_CUDA(e);
    k_rel_nzend<<<grid_for(n, 256, c.device, 16), 256, 0, c.stream>>>(roff2, nzrow, nsel, nzend);
    int64_t *hn;
    SP_TRY(c.host_as(&hn));
    SP_CUDA(cudaMemcpyAsync(hn, nsel, 8, cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    const int64_t nnz = hn[0];
    const int64_t nunits = m ? (m - 1) / kUnit + 1 : 0;
    SP_TRY(resident_alloc((void **)&ur, (size_t)std::max<int64_t>(1, nunits) * 8 + 16));
    if (nunits)
        k_pr_setup<<<grid_for(nunits, 256, c.device), 256, 0, c.stream>>>(nzend, 0, nnz, 0, 0,
                                                                          nunits, ur);
    c.launches += 12;
    SP_CUDA(cudaGetLastError());
    SP_CUDA(cudaStreamSynchronize(c.stream));  // other threads' streams read the layout
    g->rel_perm = perm;
    g->rel_radj = radj;
    g->rel_outdeg = outd;
    g->rel_indeg = ind;
    g->rel_nzrow = nzrow;
    g->rel_nzend = nzend;
    g->rel_unit_row = ur;
    g->rel_nnz = nnz;
    g->rel_nunits = nunits;
    g->rel_H = H;
    prep_mark(g, kPrepPrRel, 1, c.stream);
    g->pr_rel = 1;
    guard.ok = true;
    return SP_OK;
}

// rank[v] = rank'[rank of v]: the relabelled run's ranks in vertex order
__global__ void k_pr_unperm(const PrLoop *L, const int32_t *__restrict__ perm, int64_t n) {
    const double *rr = L->rank;
    double *out = L->rank_out;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < n; v0 += 4 * stride) {
        int32_t p[4];
#pragma unroll
        for (int j = 0; j < 4; j++) p[j] = v0 + j * stride < n ? __ldcs(perm + v0 + j * stride) : 0;
        double r[4];
#pragma unroll
        for (int j = 0; j < 4; j++) r[j] = v0 + j * stride < n ? __ldcs(rr + p[j]) : 0.0;
#pragma unroll
        for (int j = 0; j < 4; j++)
            if (v0 + j * stride < n) out[v0 + j * stride] = r[j];
    }
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
    // relabelled layout (whole graph only): rows and sources are ranks
    bool rel = false;
    const int32_t *init_outdeg = nullptr, *init_indeg = nullptr;  // k_pr_init's view
};

// The whole-graph plan over the relabelled layout (ensure_pr_rel built it).
int plan_rel(sp_graph *g, Call &c, double damping, FastPlan &p) {
    PrArgs &a = p.a;
    a.radj = g->rel_radj;
    a.nzend = g->rel_nzend;
    a.nzrow = g->rel_nzrow;
    a.outdeg = g->rel_outdeg;
    a.v0 = 0;
    a.S0 = 0;
    a.S1 = g->m;
    a.K0 = 0;
    a.K1 = g->rel_nnz;
    a.u0 = 0;
    a.nunits = g->rel_nunits;
    a.base = (1.0 - damping) / (double)g->n;  // pr.sp:17
    a.damping = damping;
    a.unit_row = g->rel_unit_row;
    const int64_t nu = std::max<int64_t>(1, a.nunits);
    double *hp, *tp, *sums;
    SP_TRY(c.alloc(&sums, std::max<int64_t>(1, a.K1)));
    SP_TRY(c.alloc(&hp, nu));
    SP_TRY(c.alloc(&tp, nu));
    a.sums = sums;
    a.hp = hp;
    a.tp = tp;
    p.rel = true;
    p.H = g->rel_H;
    p.hot_smem = (size_t)p.H * sizeof(double) + (kHotBlock / 32) * (kCh / 32) * 4;
    SP_CUDA(cudaFuncSetAttribute(k_pr_units_rel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)p.hot_smem));
    p.grid_hot = num_sms(c.device);
    p.grid_units = (int)std::max<int64_t>(1, (a.nunits + kWarps - 1) / kWarps);
    p.grid_epi = (int)std::max<int64_t>(1, (a.K1 + 256 * kEpi - 1) / (256 * kEpi));
    p.init_outdeg = g->rel_outdeg;
    p.init_indeg = g->rel_indeg;
    return SP_OK;
}

// hotc_ext: caller-owned buffer of >= pr_H + 1 doubles for the hot copies
// (the cached device loop keeps it in its argument block), or null.
int plan_fast(sp_graph *g, Call &c, int64_t v0, int64_t v1, double damping, FastPlan &p,
              double *hotc_ext = nullptr, bool hot_settled = false) {
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
    const bool whole = v0 == 0 && v1 == g->n;
    int64_t *ur = nullptr;
    if (whole) {  // the whole graph's unit index: built once, resident
        std::lock_guard<std::mutex> lk(g_hot_mu);
        if (g->pr_nunits < 0) {
            SP_TRY(resident_alloc((void **)&g->pr_unit_row, (size_t)nu * sizeof(int64_t)));
            if (a.nunits) {
                k_pr_setup<<<grid_for(a.nunits, 256, c.device), 256, 0, c.stream>>>(
                    g->nzend, a.K0, a.K1, a.S0, a.u0, a.nunits, g->pr_unit_row);
                c.launches++;
            }
            SP_CUDA(cudaStreamSynchronize(c.stream));  // other threads' streams read it
            g->pr_nunits = a.nunits;
        }
        ur = g->pr_unit_row;
    } else {
        SP_TRY(c.alloc(&ur, nu));
        if (a.nunits) {
            k_pr_setup<<<grid_for(a.nunits, 256, c.device), 256, 0, c.stream>>>(
                g->nzend, a.K0, a.K1, a.S0, a.u0, a.nunits, ur);
            c.launches++;
        }
    }
    double *hp, *tp, *sums;
    SP_TRY(c.alloc(&sums, std::max<int64_t>(1, a.K1 - a.K0)));
    a.sums = sums;
    SP_TRY(c.alloc(&hp, nu));
    SP_TRY(c.alloc(&tp, nu));
    a.hp = hp;
    a.tp = tp;
    a.unit_row = ur;
    // one unit per warp, no cap: the block scheduler balances the tail
    p.grid_units = (int)std::max<int64_t>(1, (a.nunits + kWarps - 1) / kWarps);
    if (!hot_settled) SP_TRY(ensure_pr_hot(g, c));
    if (g->pr_H > 0) {
        p.H = g->pr_H;
        p.hot_ids = g->pr_hot_ids;
        a.radj = g->pr_radj_hot;  // encoded slots
        if (!hotc_ext) {
            double *hotc;
            SP_TRY(c.alloc(&hotc, p.H + 1));
            p.hotc = hotc;
        } else {
            p.hotc = hotc_ext;
        }
        if (p.H > kHotMax) {  // split over a CTA pair
            const int Hl = ((p.H + 1) / 2 + 1) & ~1;
            p.hot_smem = (size_t)Hl * sizeof(double) + (kHotBlock / 32) * (kCh / 32) * 4;
            SP_CUDA(cudaFuncSetAttribute(k_pr_units_hot2,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)p.hot_smem));
            p.grid_hot = num_sms(c.device) & ~1;
        } else {
            p.hot_smem = (size_t)p.H * sizeof(double) + (kHotBlock / 32) * (kCh / 32) * 4;
            SP_CUDA(cudaFuncSetAttribute(k_pr_units_hot,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)p.hot_smem));
            p.grid_hot = num_sms(c.device);
        }
    }
    p.grid_epi = (int)std::max<int64_t>(1, (a.K1 - a.K0 + 256 * kEpi - 1) / (256 * kEpi));
    p.grid_zero = (int)std::max<int64_t>(1, (v1 - v0 + 255) / 256);
    p.init_outdeg = g->outdeg;
    p.init_indeg = g->indeg;
    SP_CUDA(cudaGetLastError());
    return SP_OK;
}

template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                Args &&...args) {
    // opt-in (SP_PR_PDL=1): measured neutral on B200 (RMAT-22 2.921 vs
    // 2.922 ms per run; RMAT-24 relabelled 7.89 vs 7.70 ms)
    static const bool off = [] {
        const char *e = getenv("SP_PR_PDL");
        return !(e && e[0] == '1');
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = off ? 0 : 1;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// The row-sum kernel of one iteration (hot-source variant when built).
void launch_units(Call &c, const FastPlan &p, const PrArgs &a) {
    if (p.rel) {
        launch_pdl(k_pr_units_rel, p.grid_hot, kHotBlock, p.hot_smem, c.stream, a, p.H);
        c.launches++;
    } else if (p.H > 0) {
        launch_pdl(k_pr_hot_gather, grid_for(p.H, 256, c.device), 256, 0, c.stream, a, p.hot_ids,
                   p.H, p.hotc);
        if (p.H > kHotMax)
            launch_pdl(k_pr_units_hot2, p.grid_hot, kHotBlock, p.hot_smem, c.stream, a,
                       (const double *)p.hotc, p.H);
        else
            launch_pdl(k_pr_units_hot, p.grid_hot, kHotBlock, p.hot_smem, c.stream, a,
                       (const double *)p.hotc, p.H);
        c.launches += 2;
    } else {
        launch_pdl(k_pr_units, p.grid_units, kBlock, 0, c.stream, a);
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

#ifndef SP_PR_INIT_U
#define SP_PR_INIT_U 4
#endif
constexpr int kInitU = SP_PR_INIT_U;
// Loop-path init (pr.sp:5-8 plus iteration 1 of the zero-in-degree rows):
// rank = 1/n and c0 = rank/outdeg for every vertex; rows with no in-edges
// get their final rank = base now, c1 = c2 = base/outdeg, and contribute
// |base - 1/n| to iteration 1's diff (exactly what iteration 1 computes for
// them: sum = 0).
__global__ void __launch_bounds__(256) k_pr_init(PrLoop *L, const int32_t *__restrict__ outdeg,
                                                 const int32_t *__restrict__ indeg, int64_t n,
                                                 double r0) {
    const double base = L->base;
    double *rank = L->rank, *c0 = L->c0, *c1 = L->c1, *c2 = L->c2;
    double dmax = 0.0;
    // kInitU vertices per thread and step, their loads issued first: the
    // stream needs that many bytes in flight per SM (RMAT-24: 194 -> 169 us)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t x0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x0 < n;
         x0 += stride * kInitU) {
        int d[kInitU], in[kInitU];
#pragma unroll
        for (int j = 0; j < kInitU; j++) {
            const int64_t x = x0 + j * stride;
            d[j] = x < n ? __ldcs(outdeg + x) : 0;
            in[j] = x < n ? __ldcs(indeg + x) : 1;
        }
#pragma unroll
        for (int j = 0; j < kInitU; j++) {
            const int64_t x = x0 + j * stride;
            if (x >= n) break;
            c0[x] = d[j] > 0 ? __ddiv_rn(r0, (double)d[j]) : 0.0;
            if (in[j] == 0) {
                rank[x] = base;
                const double cz = d[j] > 0 ? __ddiv_rn(base, (double)d[j]) : 0.0;
                c1[x] = cz;
                c2[x] = cz;
                double t = __dsub_rn(base, r0);
                if (t < 0.0) t = __dsub_rn(0.0, t);
                dmax = fmax(dmax, t);
            } else {
                rank[x] = r0;
            }
        }
    }
    dmax = warp_max(dmax);
    // the same value from every block: read first, so at most a few atomics
    if (lane_id() == 0 && dmax > 0.0 &&
        __double_as_longlong(dmax) >
            (long long)__ldcg(reinterpret_cast<const unsigned long long *>(L->slot + 1)))
        atomic_max_nonneg(L->slot + 1, dmax);
}

// The loop step as its own launch (graphs without non-empty rows).
__global__ void k_pr_advance(PrLoop *L, cudaGraphConditionalHandle h, int in_graph) {
    griddep_wait();
    pr_advance(L, h, in_graph != 0);
}


// The body of one fast iteration on the call's stream.
// One iteration and the loop step (in a graph: sets the WHILE flag).  (A
// last-block-done step inside k_pr_epi measured slower: thousands of
// same-address counter atomics serialise at one L2 slice.)
void launch_iteration(Call &c, const FastPlan &p, const PrArgs &a, bool in_graph,
                      cudaGraphConditionalHandle cond) {
    if (a.nunits) {
        launch_units(c, p, a);
        launch_pdl(k_pr_epi, p.grid_epi, 256, 0, c.stream, a);
        c.launches++;
    }
    launch_pdl(k_pr_advance, 1, 1, 0, c.stream, a.loop, cond, in_graph ? 1 : 0);
    c.launches++;
}

// Instantiate the whole fast run as one graph: k_pr_init, then a WHILE node
// over { [hot gather,] units, epilogue, advance }.  Every per-call value is
// read from L, so the executable is reused by every later call of this
// thread on this graph (arg_exec_get): no capture, no update, no host round
// trip per iteration.
// A reused entry of another graph (same kind, same argument layout) is
// refreshed with cudaGraphExecUpdate instead of a new instantiation: a graph
// created per request (from_csr -> run) then costs one capture, not an
// instantiation.
int pr_build_exec(sp_graph *g, Call &c, const FastPlan &p, PrLoop *L, cudaGraphExec_t *exec) {
    cudaGraph_t graph = nullptr;
    struct GraphFree {
        cudaGraph_t *g;
        ~GraphFree() {
            if (*g) cudaGraphDestroy(*g);
        }
    } gf{&graph};
    SP_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h;
    SP_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
    // k_pr_init as the first node (captured into the top-level graph)
    SP_CUDA(cudaStreamBeginCaptureToGraph(c.stream, graph, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
    const double r0 = 1.0 / (double)g->n;  // pr.sp:6
    k_pr_init<<<grid_for(g->n, 256, c.device), 256, 0, c.stream>>>(L, p.init_outdeg, p.init_indeg,
                                                                   g->n, r0);
    SP_CUDA(cudaStreamEndCapture(c.stream, &graph));
    size_t nn = 0;
    SP_CUDA(cudaGraphGetNodes(graph, nullptr, &nn));
    SP_CHECK(nn == 1, SP_ERR_CUDA, "pr graph: unexpected init capture");
    cudaGraphNode_t init;
    SP_CUDA(cudaGraphGetNodes(graph, &init, &nn));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    SP_CUDA(cudaGraphAddNode(&node, graph, &init, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    SP_CUDA(cudaStreamBeginCaptureToGraph(c.stream, body, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
    PrArgs a = p.a;
    a.loop = L;
    launch_iteration(c, p, a, true, h);
    SP_CUDA(cudaStreamEndCapture(c.stream, &body));
    if (p.rel) {  // the ranks back in vertex order, after the loop
        SP_CUDA(cudaStreamBeginCaptureToGraph(c.stream, graph, &node, nullptr, 1,
                                              cudaStreamCaptureModeThreadLocal));
        k_pr_unperm<<<grid_for(g->n, 256, c.device, 16), 256, 0, c.stream>>>(L, g->rel_perm, g->n);
        SP_CUDA(cudaStreamEndCapture(c.stream, &graph));
    }
    if (*exec) {
        cudaGraphExecUpdateResultInfo info;
        if (cudaGraphExecUpdate(*exec, graph, &info) == cudaSuccess) return SP_OK;
        cudaGetLastError();
        cudaGraphExecDestroy(*exec);
        *exec = nullptr;
    }
    SP_CUDA(cudaGraphInstantiate(exec, graph, 0));
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
int pr_hot_build(sp_graph *g, Call &c) { return pr_hot_build_impl(g, c); }
int pr_hot_prepare(sp_graph *g, Call &c, const int32_t *outdeg, int64_t max_outdeg,
                   int32_t **hot_idx, int *H) {
    static_assert(kHotBit == kPrHotBit, "hot-slot encoding");
    return pr_hot_select(g, c, outdeg, max_outdeg, hot_idx, H);
}
}  // namespace sp

namespace {

// The default (fast) path: one cached graph launch per call (see
// pr_build_exec), or -- with a per-iteration callback or SP_HOSTLOOP=1 (ncu
// cannot profile conditional graphs) -- the same kernels driven from the
// host with one flag read per iteration.
int pr_fast_run(sp_graph *g, Call &c, double damping, double epsilon, int64_t max_iter,
                int64_t cap, sp_iter_cb cb, void *user, double *rank, PrLoop *hL,
                float *kernel_ms) {
    const int64_t n = g->n;
    const char *hl = getenv("SP_HOSTLOOP");
    const bool hostloop = cb || (hl && hl[0] == '1');
    // SP_PR_TRACE: host time of the call's phases (diagnostics; syncs)
    static const bool trace = getenv("SP_PR_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char *what) {
        if (!trace) return;
        cudaStreamSynchronize(c.stream);
        fprintf(stderr, "pr: %-14s %7.3f ms\n", what,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                    .count());
    };
    // the layout must be settled before the executable is chosen: the
    // relabelled one from the graph's second fast call on (its build costs
    // about two runs), else the hot-encoded or plain one
    int runs;
    {
        std::lock_guard<std::mutex> lk(g_hot_mu);
        runs = g->pr_runs++;
    }
    if (runs > 0) SP_TRY(ensure_pr_rel(g, c));
    const bool rel = g->pr_rel == 1;
    if (!rel) SP_TRY(ensure_pr_hot(g, c));
    const int H = rel ? 0 : std::max(0, g->pr_H);
    const size_t hot_off = (sizeof(PrLoop) + 255) & ~size_t(255);
    const size_t bytes = hot_off + (size_t)(H + 1) * sizeof(double);
    ArgExec *e = nullptr;
    bool fresh = false;
    PrLoop *L;
    double *hotc = nullptr;
    if (!hostloop) {
        SP_TRY(arg_exec_get(g->uid, rel ? kArgPrRel : H > 0 ? kArgPrHot : kArgPr, bytes, c.device,
                            &e, &fresh));
        L = static_cast<PrLoop *>(e->args);
        hotc = reinterpret_cast<double *>(static_cast<char *>(e->args) + hot_off);
    } else {
        char *blk;
        SP_TRY(c.alloc(&blk, bytes));
        L = reinterpret_cast<PrLoop *>(blk);
        hotc = reinterpret_cast<double *>(blk + hot_off);
    }
    mark("layout+exec");
    FastPlan plan;
    if (rel) {
        SP_TRY(plan_rel(g, c, damping, plan));
    } else {
        SP_TRY(plan_fast(g, c, 0, n, damping, plan, hotc, true));
    }
    mark("plan");
    double *c0, *c1, *c2, *rank_rel = nullptr;
    if (rel) SP_TRY(c.alloc(&rank_rel, n));
    SP_TRY(c.alloc(&c0, n));
    SP_TRY(c.alloc(&c1, n));
    SP_TRY(c.alloc(&c2, n));
    char *pin;
    SP_TRY(c.host_as(&pin));
    static_assert(2048 + sizeof(PrLoop) <= kPinnedBlock, "pinned block layout");
    PrLoop *init = reinterpret_cast<PrLoop *>(pin + 2048);  // hL is at the block's start
    *init = PrLoop{};
    init->c0 = c0;
    init->c1 = c1;
    init->c2 = c2;
    init->rank = rel ? rank_rel : rank;
    init->rank_out = rank;
    init->sums = plan.a.sums;
    init->hp = plan.a.hp;
    init->tp = plan.a.tp;
    init->base = plan.a.base;
    init->damping = damping;
    init->eps = epsilon;
    init->max_iter = max_iter;
    init->cap = cap;
    SP_CUDA(cudaMemcpyAsync(L, init, sizeof(PrLoop), cudaMemcpyHostToDevice, c.stream));
    const int per_it = (plan.a.nunits ? (H > 0 ? 3 : 2) : 0) + 1;
    cudaEvent_t ka, kb;
    SP_CUDA(cudaEventCreate(&ka));
    SP_CUDA(cudaEventCreate(&kb));
    struct EvFree {
        cudaEvent_t a, b;
        ~EvFree() {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } ef{ka, kb};
    if (!hostloop) {
        if (fresh) {
            const int64_t l0 = c.launches;
            static const bool verbose = getenv("SP_PR_VERBOSE") != nullptr;
            if (verbose)
                fprintf(stderr, "pr exec: %s (graph %llu)\n",
                        e->exec ? "capture + update" : "capture + instantiate",
                        (unsigned long long)g->uid);
            mark("allocs+init");
            int rc = pr_build_exec(g, c, plan, L, &e->exec);
            c.launches = l0;
            if (rc != SP_OK) {
                e->exec = nullptr;
                return rc;
            }
            mark("capture+update");
        }
        SP_CUDA(cudaEventRecord(ka, c.stream));
        SP_CUDA(cudaGraphLaunch(e->exec, c.stream));
        SP_CUDA(cudaEventRecord(kb, c.stream));
        SP_CUDA(cudaMemcpyAsync(hL, L, sizeof(PrLoop), cudaMemcpyDeviceToHost, c.stream));
        SP_CUDA(cudaStreamSynchronize(c.stream));
        mark("loop");
        c.launches += 1 + hL->iters * per_it + (rel ? 1 : 0);
    } else {
        PrArgs a = plan.a;
        a.loop = L;
        const double r0 = 1.0 / (double)n;
        SP_CUDA(cudaEventRecord(ka, c.stream));
        k_pr_init<<<grid_for(n, 256, c.device), 256, 0, c.stream>>>(L, plan.init_outdeg,
                                                                    plan.init_indeg, n, r0);
        c.launches++;
        for (;;) {
            launch_iteration(c, plan, a, false, cudaGraphConditionalHandle{});
            SP_CUDA(cudaMemcpyAsync(hL, L, sizeof(PrLoop), cudaMemcpyDeviceToHost, c.stream));
            SP_CUDA(cudaStreamSynchronize(c.stream));
            if (cb && cb(hL->iters, user)) {
                set_error("aborted by the fixedPoint iteration callback");
                return SP_ERR_ABORTED;
            }
            if (hL->status == 2 || hL->diff < epsilon || hL->iter >= max_iter) break;
        }
        if (rel) {
            k_pr_unperm<<<grid_for(n, 256, c.device, 16), 256, 0, c.stream>>>(L, g->rel_perm, n);
            c.launches++;
        }
        SP_CUDA(cudaEventRecord(kb, c.stream));
    }
    SP_CUDA(cudaGetLastError());
    SP_CUDA(cudaEventSynchronize(kb));
    cudaEventElapsedTime(kernel_ms, ka, kb);
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
    const bool exact = flags & SP_FLAG_DETERMINISTIC;
    // results land in the caller's buffer directly when it is device memory
    double *rank = nullptr;
    if (mem == SP_MEM_DEVICE && n) {
        rank = rank_out;
    } else {
        SP_TRY(c.alloc(&rank, n));
    }
    float kernel_ms = 0.f;
    int64_t iter = 0, iters = 0;
    double diff = 0.0;
    int rc = SP_OK;
    if (n && !exact) {
        PrLoop *hL;
        SP_TRY(c.host_as(&hL));
        rc = pr_fast_run(g, c, damping, epsilon, max_iter, cap, cb, user, rank, hL, &kernel_ms);
        if (rc == SP_OK) {
            iter = hL->iter;
            iters = hL->iters;
            diff = hL->diff;
            if (hL->status == 2) {
                set_error("fixedPoint 'converged' did not converge within %lld iterations",
                          (long long)cap);
                rc = SP_ERR_NONCONV;
            }
        }
    } else {
        // exact path (and n == 0): host loop, one diff read per iteration
        double *ca, *cb2, *diffs;
        SP_TRY(c.alloc(&ca, n));
        SP_TRY(c.alloc(&cb2, n));
        const int64_t kSlots = 1024;  // diff slots, recycled in a ring
        SP_TRY(c.alloc(&diffs, kSlots));
        SP_CUDA(cudaMemsetAsync(diffs, 0, kSlots * sizeof(double), c.stream));
        double *hdiff = nullptr;
        SP_TRY(c.host_as(&hdiff));
        const double r0 = n ? 1.0 / (double)n : 0.0;  // pr.sp:6
        if (n) {
            k_init<<<grid_for(n, 256, c.device), 256, 0, c.stream>>>(rank, ca, g->outdeg, 0, n, r0);
            c.launches++;
        }
        cudaEvent_t ka, kb;
        SP_CUDA(cudaEventCreate(&ka));
        SP_CUDA(cudaEventCreate(&kb));
        for (;;) {
            double *slot = diffs + (iters % kSlots);
            if (n) {
                rc = launch_exact(g, c, 0, n, damping, ca, rank, cb2, slot, ka, kb);
                if (rc) break;
                SP_CUDA(cudaMemcpyAsync(hdiff, slot, sizeof(double), cudaMemcpyDeviceToHost,
                                        c.stream));
                SP_CUDA(cudaMemsetAsync(diffs + ((iters + 1) % kSlots), 0, sizeof(double),
                                        c.stream));
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
    }
    if (rc == SP_OK && n && rank != rank_out)
        SP_TRY(from_device(rank_out, rank, n * 8, mem, c.stream));
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

// ---- vertex-block shards (multi-GPU, graph.py:226-249 ownership) --------
// A shard is planned once per run (the block's slot and row bounds, unit
// index, scratch, hot sources): a step only launches the pull over the
// block and writes the block's max |delta| into a caller device double, on
// the caller's stream (`stream`, e.g. torch's current stream, so the
// exchange collectives order after it without a host sync; NULL: the
// library's per-thread stream, synchronised per step).
struct sp_pagerank_shard {
    sp_graph *g = nullptr;
    int64_t v0 = 0, v1 = 0;
    double damping = 0.0;
    bool det = false;
    cudaStream_t stream = nullptr;
    FastPlan plan;
    void *keep[32];
    int nkeep = 0;
    double **peers = nullptr;  // device: nsets x npeers contrib-array pointers
    int npeers = 0, nsets = 0;
};

// Deterministic-mode form of the peer stores: the block's contribs to every
// peer's array (the exact kernel writes contrib_out only).
__global__ void k_pr_scatter_peers(const double *__restrict__ cout, int64_t v0, int64_t nb,
                                   double *const *peers, int npeers) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double c = cout[i];
        for (int q = 0; q < npeers; q++) peers[q][v0 + i] = c;
    }
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

extern "C" int sp_pagerank_shard_create(sp_graph *g, int64_t v0, int64_t v1, double damping,
                                        unsigned flags, void *stream, sp_pagerank_shard **out) {
    SP_CHECK(g && out && v0 >= 0 && v0 <= v1 && v1 <= g->n, SP_ERR_ARG, "bad vertex block");
    *out = nullptr;
    Call c;
    SP_TRY(c.begin(g->device));
    sp_pagerank_shard *h = new sp_pagerank_shard;
    h->g = g;
    h->v0 = v0;
    h->v1 = v1;
    h->damping = damping;
    h->det = (flags & SP_FLAG_DETERMINISTIC) != 0;
    h->stream = static_cast<cudaStream_t>(stream);
    int rc = SP_OK;
    if (!h->det && v1 > v0) rc = plan_fast(g, c, v0, v1, damping, h->plan);
    // the plan's scratch outlives this call: the shard owns it
    for (int i = 0; i < c.nbufs && h->nkeep < 32; i++) h->keep[h->nkeep++] = c.bufs[i];
    c.nbufs = 0;
    if (rc == SP_OK) rc = c.finish(nullptr);
    if (rc != SP_OK) {
        cudaDeviceSynchronize();
        for (int i = 0; i < h->nkeep; i++) scratch_free(h->keep[i], nullptr);
        delete h;
        return rc;
    }
    *out = h;
    return SP_OK;
}

extern "C" int sp_pagerank_shard_peers(sp_pagerank_shard *h, int nsets, int npeers,
                                       double *const *peers) {
    SP_CHECK(h && nsets >= 1 && npeers >= 1 && npeers <= 1024 && peers, SP_ERR_ARG,
             "sp_pagerank_shard_peers: bad arguments");
    Call c;
    SP_TRY(c.begin(h->g->device));
    double **d = nullptr;
    SP_TRY(resident_alloc((void **)&d, (size_t)nsets * npeers * sizeof(double *)));
    SP_CUDA(cudaMemcpyAsync(d, peers, (size_t)nsets * npeers * sizeof(double *),
                            cudaMemcpyHostToDevice, c.stream));
    SP_TRY(c.finish(nullptr));
    if (h->peers) resident_free(h->peers);
    h->peers = d;
    h->npeers = npeers;
    h->nsets = nsets;
    return SP_OK;
}

static int shard_step(sp_pagerank_shard *h, const double *contrib_in, double *rank_local,
                      double *contrib_out, double *diff, int set);

extern "C" int sp_pagerank_shard_step_peers(sp_pagerank_shard *h, const double *contrib_in,
                                            double *rank_local, double *contrib_out,
                                            double *diff, int set) {
    SP_CHECK(h && h->peers && set >= 0 && set < h->nsets, SP_ERR_ARG,
             "sp_pagerank_shard_step_peers: no peer set %d", set);
    return shard_step(h, contrib_in, rank_local, contrib_out, diff, set);
}

extern "C" int sp_pagerank_shard_step(sp_pagerank_shard *h, const double *contrib_in,
                                      double *rank_local, double *contrib_out, double *diff) {
    return shard_step(h, contrib_in, rank_local, contrib_out, diff, -1);
}

static int shard_step(sp_pagerank_shard *h, const double *contrib_in, double *rank_local,
                      double *contrib_out, double *diff, int set) {
    SP_CHECK(h && contrib_in && rank_local && contrib_out && diff, SP_ERR_ARG,
             "sp_pagerank_shard_step: bad arguments");
    sp_graph *g = h->g;
    Call c;
    if (h->stream) SP_TRY(c.begin_external(g->device, h->stream));
    else SP_TRY(c.begin(g->device));
    SP_CUDA(cudaMemsetAsync(diff, 0, sizeof(double), c.stream));
    double *const *peers = set >= 0 ? h->peers + (size_t)set * h->npeers : nullptr;
    const int np = set >= 0 ? h->npeers : 0;
    if (h->v1 > h->v0) {
        if (h->det) {
            SP_TRY(launch_exact(g, c, h->v0, h->v1, h->damping, contrib_in, rank_local,
                                contrib_out, diff, nullptr, nullptr));
            if (np) {
                k_pr_scatter_peers<<<grid_for(h->v1 - h->v0, 256, c.device), 256, 0, c.stream>>>(
                    contrib_out, h->v0, h->v1 - h->v0, peers, np);
                c.launches++;
            }
        } else {
            // contrib_out is a single persistent buffer here: zero rows are
            // rewritten every step (cheap: one indeg pass over the block);
            // with peers, the epilogue also stores every contrib into them
            FastPlan plan = h->plan;
            plan.a.peers = peers;
            plan.a.npeers = np;
            SP_TRY(launch_fast(c, plan, g, h->v1, contrib_in, rank_local, contrib_out, nullptr,
                               true, diff, nullptr, nullptr));
        }
    }
    SP_CUDA(cudaGetLastError());
    if (!h->stream) SP_TRY(c.finish(nullptr));
    return SP_OK;
}

extern "C" void sp_pagerank_shard_destroy(sp_pagerank_shard *h) {
    if (!h) return;
    cudaSetDevice(h->g->device);
    cudaDeviceSynchronize();
    for (int i = 0; i < h->nkeep; i++) scratch_free(h->keep[i], nullptr);
    if (h->peers) resident_free(h->peers);
    cudaDeviceSynchronize();
    delete h;
}

// ---- peer-mapped buffers (CUDA IPC: other processes' GPUs over NVLink) ----
extern "C" int sp_peer_alloc(int device, int64_t bytes, void **ptr, void *handle) {
    SP_CHECK(ptr && handle && bytes > 0, SP_ERR_ARG, "sp_peer_alloc: bad arguments");
    SP_CUDA(cudaSetDevice(device));
    // plain cudaMalloc: IPC handles need it (not the stream-ordered pool)
    SP_CUDA(cudaMalloc(ptr, (size_t)bytes));
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, *ptr);
    if (e != cudaSuccess) {
        cudaFree(*ptr);
        *ptr = nullptr;
        SP_CUDA(e);
    }
    memcpy(handle, &h, sizeof(h));
    return SP_OK;
}

extern "C" int sp_peer_open(int device, const void *handle, void **ptr) {
    SP_CHECK(ptr && handle, SP_ERR_ARG, "sp_peer_open: bad arguments");
    SP_CUDA(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    SP_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return SP_OK;
}

extern "C" void sp_peer_free(void *ptr, int opened) {
    if (!ptr) return;
    cudaDeviceSynchronize();
    if (opened) cudaIpcCloseMemHandle(ptr);
    else cudaFree(ptr);
}
