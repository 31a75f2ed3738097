// sp_expand.cuh -- load-balanced frontier expansion (the `forall nbr in
// g.neighbors(v)` of a filtered outer forall, interp.py:373-399), shared by
// SSSP relaxation and BFS discovery.
//
//  * k_expand: a warp takes up to 32 frontier vertices, prefix-sums their
//    degrees in registers and walks the flattened edge list kRounds x 32
//    slots at a time: coalesced adj loads, every lane busy whatever the
//    degree mix;
//  * rows longer than kSplit are not walked there; they are cut into
//    kSplit-slot chunks (vertex, chunk) and k_expand_chunks gives each chunk
//    one warp (kSplit/32 slots per lane), so one 100K-degree hub cannot
//    serialise a warp;
//  * small frontiers get fewer vertices per warp (down to one), so a
//    frontier of a few hundred long rows still fills the GPU;
//  * every slot's work is split into a load-only probe and an apply step
//    (the atomics); all probes of a lane are issued before any apply, so
//    several random L2 round trips are in flight per lane instead of one
//    dependent chain per slot;
//  * visited vertices are staged in a per-warp shared-memory buffer and
//    appended to the next frontier kStage at a time, one global atomic per
//    batch: a single global counter shared by every warp serialises at one
//    L2 slice, and waiting for its return was the top stall.
// Op supplies:  Payload payload(int32_t v)             -- per-source-vertex value
//               Probe probe(int64_t e, int32_t x)      -- loads only
//               bool apply(Payload, int64_t e, int32_t x, Probe) -- true => push x
//               (`using Payload` / `using Probe` declare the types)
#pragma once

#include <type_traits>
#include <utility>

#include "sp_common.cuh"

namespace sp {

constexpr int kExpandBlock = 256;
constexpr int kSplit = 256;  // rows longer than this are cut into kSplit-slot chunks
constexpr int kRounds = 4;   // 32-slot rounds in flight per warp in k_expand

// A hub-chunk work item: {vertex, first slot (lo, hi), slot count}.  The
// slot range is resolved when the chunk is published, so the chunk kernel's
// first dependent load is the adjacency itself.
using ChunkItem = uint4;

struct ExpandCounters {
    unsigned long long next_size;  // appended frontier entries
    unsigned long long scanned;    // slots scanned
    unsigned long long chunks;     // hub chunk work items published
    unsigned long long flag;       // op-specific error flag
};

// Optional Op extensions (detected at compile time):
//   bool keep(int32_t v, Payload pay)  -- false: skip v's row (stale entry)
//   apply() returning 2 = push x to the far queue (Op::kFar == true; the
//   far queue and its counter come from op.far_q / op.far_n)
template <class Op, class = void>
struct HasFar : std::false_type {};
template <class Op>
struct HasFar<Op, std::void_t<decltype(Op::kFar)>> : std::integral_constant<bool, Op::kFar> {};
// Optional phased apply (Op::kPhased): the returning atomics of all of a
// lane's slots are issued before any result is examined, so their round
// trips overlap instead of chaining slot after slot:
//   int a = apply(pay, e, x, probe)         -- phase 1 (predicated atomics)
//   int b = settle(a, x, pay, probe)        -- phase 2 (predicated atomics)
//   int r = result(a, b, x, pay, probe)     -- pure
// x < 0 marks an empty slot (its probe is unset); the Op must ignore it.
template <class Op, class = void>
struct IsPhased : std::false_type {};
template <class Op>
struct IsPhased<Op, std::void_t<decltype(Op::kPhased)>> : std::integral_constant<bool, Op::kPhased> {};

template <class Op, int K, class PayArr>
__device__ __forceinline__ void apply_all(const Op &op, int (&res)[K], const int32_t (&x)[K],
                                          const int64_t (&e)[K], const PayArr &pay,
                                          const typename Op::Probe (&pr)[K]) {
    if constexpr (IsPhased<Op>::value) {
        int a[K], b[K];
#pragma unroll
        for (int u = 0; u < K; u++) a[u] = op.apply(pay[u], e[u], x[u], pr[u]);
#pragma unroll
        for (int u = 0; u < K; u++) b[u] = op.settle(a[u], x[u], pay[u], pr[u]);
#pragma unroll
        for (int u = 0; u < K; u++) res[u] = op.result(a[u], b[u], x[u], pay[u], pr[u]);
    } else {
#pragma unroll
        for (int u = 0; u < K; u++)
            res[u] = x[u] >= 0 ? (int)op.apply(pay[u], e[u], x[u], pr[u]) : 0;
    }
}

// Predicated returning atomics (inline PTX, no branch around them): the
// result register is only written when p holds.
__device__ __forceinline__ int atom_min_if(bool p, int32_t *a, int v) {
    int old;
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %1, 0; @q atom.global.min.s32 %0, [%2], %3; }"
                 : "=r"(old)
                 : "r"((unsigned)p), "l"(a), "r"(v)
                 : "memory");
    return old;
}
__device__ __forceinline__ int atom_exch_if(bool p, int32_t *a, int v) {
    int old;
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %1, 0; @q atom.global.exch.b32 %0, [%2], %3; }"
                 : "=r"(old)
                 : "r"((unsigned)p), "l"(a), "r"(v)
                 : "memory");
    return old;
}

template <class Op, class = void>
struct HasKeep : std::false_type {};
template <class Op>
struct HasKeep<Op, std::void_t<decltype(std::declval<const Op &>().keep(0, typename Op::Payload()))>>
    : std::true_type {};

constexpr int kStage = 256;  // staged queue entries per warp (shared memory)

// The warp's staging buffers for the next frontier (and the far pile).
struct ExpandStage {
    WarpStage<kStage> near, far;
};

__device__ __forceinline__ ExpandStage make_stage() {
    __shared__ int32_t s_near[kExpandBlock / 32][kStage];
    __shared__ int32_t s_far[kExpandBlock / 32][kStage];
    ExpandStage st;
    st.near.buf = s_near[threadIdx.x >> 5];
    st.far.buf = s_far[threadIdx.x >> 5];
    return st;
}

template <class Op, int K>
__device__ __forceinline__ void append_results(const Op &op, const int (&res)[K],
                                               const int32_t (&x)[K], ExpandCounters *cnt,
                                               int32_t *qn, ExpandStage &st) {
    bool near[K];
#pragma unroll
    for (int u = 0; u < K; u++) near[u] = res[u] == 1;
    st.near.push<K>(near, x, &cnt->next_size, qn);
    if constexpr (HasFar<Op>::value) {
        bool far[K];
#pragma unroll
        for (int u = 0; u < K; u++) far[u] = res[u] == 2;
        st.far.push<K>(far, x, op.far_n, op.far_q, op.far_cap);
    }
}

template <class Op>
__device__ __forceinline__ void flush_stage(const Op &op, ExpandCounters *cnt, int32_t *qn,
                                            ExpandStage &st) {
    st.near.flush(&cnt->next_size, qn);
    if constexpr (HasFar<Op>::value) st.far.flush(op.far_n, op.far_q, op.far_cap);
}

// One batch: lane-held frontier vertex v (-1: none) expanded by the warp.
template <class Op>
__device__ __forceinline__ void expand_batch(const Op &op, const int64_t *__restrict__ off,
                                             const int32_t *__restrict__ adj, int32_t v,
                                             int32_t *__restrict__ qn, ChunkItem *__restrict__ chunks,
                                             ExpandCounters *cnt, ExpandStage &st,
                                             unsigned long long &scanned) {
    using P = typename Op::Payload;
    using Pr = typename Op::Probe;
    const unsigned lane = lane_id();
    int64_t beg = 0, deg = 0;
    P pay = P(0);
    if (v >= 0) {
        beg = off[v];
        deg = off[v + 1] - beg;
        pay = op.payload(v);
        if constexpr (HasKeep<Op>::value) {
            if (!op.keep(v, pay)) deg = 0;
        }
    }
    if (deg > kSplit) {  // hub row -> chunk work items
        int64_t nch = (deg + kSplit - 1) / kSplit;
        unsigned long long s = atomicAdd(&cnt->chunks, (unsigned long long)nch);
        for (int64_t c = 0; c < nch; c++) {
            const int64_t e0 = beg + c * kSplit;
            const int64_t len = min((int64_t)kSplit, beg + deg - e0);
            chunks[s + c] = make_uint4((unsigned)v, (unsigned)(uint64_t)e0,
                                       (unsigned)((uint64_t)e0 >> 32), (unsigned)len);
        }
        deg = 0;
    }
    int64_t incl = deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl += t;
    }
    const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
    const int64_t excl = incl - deg;
    scanned += total;
    for (int64_t p0 = 0; p0 < total; p0 += 32 * kRounds) {
        int64_t e[kRounds];
        int32_t x[kRounds];
        P pv[kRounds];
        Pr pr[kRounds];
#pragma unroll
        for (int u = 0; u < kRounds; u++) {
            const int64_t p = p0 + u * 32 + lane;
            // owner = largest lane with excl <= p (always a lane with deg > 0)
            int lo = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                int cand = lo + step;
                int64_t ex = __shfl_sync(0xffffffffu, excl, cand & 31);
                if (cand < 32 && ex <= p) lo = cand;
            }
            const int64_t ex = __shfl_sync(0xffffffffu, excl, lo);
            const int64_t b0 = __shfl_sync(0xffffffffu, beg, lo);
            pv[u] = __shfl_sync(0xffffffffu, pay, lo);
            e[u] = p < total ? b0 + (p - ex) : -1;
            x[u] = e[u] >= 0 ? __ldcs(adj + e[u]) : -1;  // streamed: evict first
        }
#pragma unroll
        for (int u = 0; u < kRounds; u++)
            if (e[u] >= 0) pr[u] = op.probe(e[u], x[u]);
        int res[kRounds];
        apply_all(op, res, x, e, pv, pr);
        append_results<Op, kRounds>(op, res, x, cnt, qn, st);
    }
}

// kHops > 0 (thin graphs, persistent loops): after its share of the
// frontier, a warp keeps expanding the near entries it has just produced,
// up to kHops hops, before the grid-wide barrier.  Those entries are still
// flushed to the next frontier as usual; the local expansion is
// speculative extra work that Op::keep() (distance dropped since the last
// expansion?) makes idempotent, so correctness never depends on it.
template <class Op, int kHops = 0>
__device__ __forceinline__ void expand_body(
    const Op &op, const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
    const int32_t *__restrict__ q, int64_t nq, int32_t *__restrict__ qn,
    ChunkItem *__restrict__ chunks, ExpandCounters *cnt, int vpw) {
    // vpw = frontier vertices per warp (32 normally; fewer for small
    // frontiers, so that every SM gets work)
    const unsigned lane = lane_id();
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long scanned = 0;
    ExpandStage st = make_stage();
    for (int64_t base = warp * vpw; base < nq; base += nwarps * vpw) {
        const int64_t i = base + lane;
        const int32_t v = ((int)lane < vpw && i < nq) ? q[i] : -1;
        expand_batch(op, off, adj, v, qn, chunks, cnt, st, scanned);
    }
    if constexpr (kHops > 0) {
        __shared__ int32_t s_local[kExpandBlock / 32][kStage];
        int32_t *lq = s_local[threadIdx.x >> 5];
        for (int hop = 0; hop < kHops && st.near.n > 0; hop++) {
            const int nl = st.near.n;
            for (int k = lane; k < nl; k += 32) lq[k] = st.near.buf[k];
            __syncwarp();
            st.near.flush(&cnt->next_size, qn);  // the global frontier gets them too
            for (int b = 0; b < nl; b += 32) {
                const int32_t v = b + (int)lane < nl ? lq[b + lane] : -1;
                expand_batch(op, off, adj, v, qn, chunks, cnt, st, scanned);
            }
            __syncwarp();
        }
    }
    flush_stage(op, cnt, qn, st);
    // `scanned` is warp-uniform (every lane added the same totals)
    if (lane == 0 && scanned) atomicAdd(&cnt->scanned, scanned);
}

template <class Op>
__global__ void __launch_bounds__(kExpandBlock, 4) k_expand(
    Op op, const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
    const int32_t *__restrict__ q, int64_t nq, int32_t *__restrict__ qn,
    ChunkItem *__restrict__ chunks, ExpandCounters *cnt, int vpw) {
    expand_body(op, off, adj, q, nq, qn, chunks, cnt, vpw);
}

// Largest power of two <= 32 that still gives every one of `warps` warps a
// share of an nq-vertex frontier (host and device use the same rule).
__host__ __device__ __forceinline__ int expand_vpw(int64_t nq, int64_t warps) {
    int vpw = 32;
    while (vpw > 1 && (nq + vpw - 1) / vpw < warps) vpw >>= 1;
    return vpw;
}

// Slots (adjacency, streamed) and payload of one chunk; len 0: all -1.
template <class Op, int K>
__device__ __forceinline__ void load_chunk(const Op &op, const int32_t *__restrict__ adj,
                                           const ChunkItem d, unsigned lane, int32_t (&x)[K],
                                           typename Op::Payload &pay, int64_t &e0) {
    e0 = (int64_t)(((uint64_t)d.z << 32) | d.y);
#pragma unroll
    for (int j = 0; j < K; j++) {
        const unsigned p = j * 32 + lane;
        x[j] = p < d.w ? __ldcs(adj + e0 + p) : -1;  // streamed: evict first
    }
    pay = d.w ? op.payload((int32_t)d.x) : typename Op::Payload(0);
}

// One warp per chunk, software-pipelined across the warp's chunks: the
// descriptor two chunks ahead and the slots + payload of the next chunk are
// in flight while the current chunk's probes and atomics run, so a chunk
// costs about one random round trip instead of descriptor -> slots ->
// probe in series.
template <class Op>
__device__ __forceinline__ void expand_chunks_body(
    const Op &op, const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
    const ChunkItem *__restrict__ chunks, int32_t *__restrict__ qn, ExpandCounters *cnt) {
    using P = typename Op::Payload;
    using Pr = typename Op::Probe;
    constexpr int kPer = kSplit / 32;
    const unsigned lane = lane_id();
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nch = (int64_t)__ldcg(&cnt->chunks);
    const ChunkItem none = make_uint4(0, 0, 0, 0);
    unsigned long long scanned = 0;
    ExpandStage st = make_stage();
    int32_t x[kPer];
    P pay;
    int64_t e0;
    const ChunkItem d0 = warp < nch ? chunks[warp] : none;
    unsigned len = d0.w;
    load_chunk(op, adj, d0, lane, x, pay, e0);
    ChunkItem d1 = warp + nwarps < nch ? chunks[warp + nwarps] : none;
    for (int64_t w = warp; w < nch; w += nwarps) {
        const ChunkItem d2 = w + 2 * nwarps < nch ? chunks[w + 2 * nwarps] : none;
        int32_t xn[kPer];
        P payn;
        int64_t e0n;
        load_chunk(op, adj, d1, lane, xn, payn, e0n);
        Pr pr[kPer];
#pragma unroll
        for (int j = 0; j < kPer; j++)
            if (x[j] >= 0) pr[j] = op.probe(e0 + j * 32 + lane, x[j]);
        int res[kPer];
        int64_t ej[kPer];
        P pj[kPer];
#pragma unroll
        for (int j = 0; j < kPer; j++) {
            ej[j] = e0 + j * 32 + lane;
            pj[j] = pay;
        }
        apply_all(op, res, x, ej, pj, pr);
        append_results<Op, kPer>(op, res, x, cnt, qn, st);
        scanned += len;
#pragma unroll
        for (int j = 0; j < kPer; j++) x[j] = xn[j];
        pay = payn;
        e0 = e0n;
        len = d1.w;
        d1 = d2;
    }
    flush_stage(op, cnt, qn, st);
    if (lane == 0 && scanned) atomicAdd(&cnt->scanned, scanned);  // warp-uniform
}

#ifndef SP_EXPCHUNK_MINB
#define SP_EXPCHUNK_MINB 3  // blocks/SM k_expand_chunks is compiled for
#endif
template <class Op>
__global__ void __launch_bounds__(kExpandBlock, SP_EXPCHUNK_MINB) k_expand_chunks(
    Op op, const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
    const ChunkItem *__restrict__ chunks, int32_t *__restrict__ qn, ExpandCounters *cnt) {
    expand_chunks_body(op, off, adj, chunks, qn, cnt);
}

// Chunk buffer capacity for a graph with m slots.
inline int64_t expand_chunk_capacity(int64_t m) { return 2 * (m / kSplit) + 2; }

// Launch both expansion kernels for one frontier.
template <class Op>
inline void launch_expand(const Op &op, const int64_t *off, const int32_t *adj, const int32_t *q,
                          int64_t nq, int32_t *qn, ChunkItem *chunks, ExpandCounters *cnt, int sms,
                          bool has_big_rows, cudaStream_t s, int64_t *launches) {
    const int cap = sms * 8;
    const int64_t warps_full = (int64_t)cap * (kExpandBlock / 32);
    const int vpw = expand_vpw(nq, warps_full);
    int64_t want = ((nq + vpw - 1) / vpw + 7) / 8;  // 8 warps per block
    int g1 = (int)(want < 1 ? 1 : (want > cap ? cap : want));
    k_expand<Op><<<g1, kExpandBlock, 0, s>>>(op, off, adj, q, nq, qn, chunks, cnt, vpw);
    ++*launches;
    if (has_big_rows) {
        k_expand_chunks<Op><<<cap, kExpandBlock, 0, s>>>(op, off, adj, chunks, qn, cnt);
        ++*launches;
    }
}

}  // namespace sp
