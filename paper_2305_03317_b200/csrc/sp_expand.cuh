// sp_expand.cuh -- load-balanced frontier expansion (the `forall nbr in
// g.neighbors(v)` of a filtered outer forall, interp.py:373-399), shared by
// SSSP relaxation and BFS discovery.
//
//  * k_expand: a warp takes 32 frontier vertices, prefix-sums their degrees
//    in registers and walks the flattened edge list 32 slots at a time:
//    coalesced adj / weight loads, every lane busy whatever the degree mix.
//  * rows longer than kSplit are not walked there; they are cut into
//    kSplit-slot chunks (vertex, chunk) and k_expand_chunks spreads the
//    chunks over all warps, so one 100K-degree hub cannot serialise a warp;
//  * small frontiers get fewer vertices per warp (down to one), so a
//    frontier of a few hundred long rows still fills the GPU.
//  * visited vertices are appended to the next frontier with one atomic per
//    warp (ballot + popc).
// Op supplies:  Payload payload(int32_t v)      -- per-source-vertex value
//               bool visit(Payload pay, int64_t e, int32_t x) -- true => push x
//               (Payload defaults to int; an Op may declare `using Payload`)
#pragma once

#include <type_traits>

#include "sp_common.cuh"

namespace sp {

constexpr int kExpandBlock = 256;

template <class Op, class = void>
struct PayloadOf { using type = int; };
template <class Op>
struct PayloadOf<Op, std::void_t<typename Op::Payload>> { using type = typename Op::Payload; };
constexpr int kSplit = 256;  // rows longer than this are cut into kSplit-slot chunks

struct ExpandCounters {
    unsigned long long next_size;  // appended frontier entries
    unsigned long long scanned;    // slots scanned
    unsigned long long chunks;     // hub chunk work items published
    unsigned long long flag;       // op-specific error flag
};

template <class Op>
__global__ void __launch_bounds__(kExpandBlock) k_expand(
    Op op, const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
    const int32_t *__restrict__ q, int64_t nq, int32_t *__restrict__ qn,
    uint2 *__restrict__ chunks, ExpandCounters *cnt, int vpw) {
    // vpw = frontier vertices per warp (32 normally; fewer for small
    // frontiers, so that every SM gets work)
    const unsigned lane = lane_id();
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long scanned = 0;
    for (int64_t base = warp * vpw; base < nq; base += nwarps * vpw) {
        int64_t i = base + lane;
        using P = typename PayloadOf<Op>::type;
        int32_t v = -1;
        int64_t beg = 0, deg = 0;
        P pay = P(0);
        if ((int)lane < vpw && i < nq) {
            v = q[i];
            beg = off[v];
            deg = off[v + 1] - beg;
            pay = op.payload(v);
        }
        if (deg > kSplit) {  // hub row -> chunk work items
            int64_t nch = (deg + kSplit - 1) / kSplit;
            unsigned long long s = atomicAdd(&cnt->chunks, (unsigned long long)nch);
            for (int64_t c = 0; c < nch; c++) chunks[s + c] = make_uint2((unsigned)v, (unsigned)c);
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
        for (int64_t p0 = 0; p0 < total; p0 += 32) {
            const int64_t p = p0 + lane;
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
            const P pv = __shfl_sync(0xffffffffu, pay, lo);
            bool push = false;
            int32_t x = 0;
            if (p < total) {
                const int64_t e = b0 + (p - ex);
                x = adj[e];
                push = op.visit(pv, e, x);
            }
            int64_t slot = warp_append(push, &cnt->next_size);
            if (push) qn[slot] = x;
        }
    }
    // `scanned` is warp-uniform (every lane added the same totals)
    if (lane == 0 && scanned) atomicAdd(&cnt->scanned, scanned);
}

template <class Op>
__global__ void __launch_bounds__(kExpandBlock) k_expand_chunks(
    Op op, const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
    const uint2 *__restrict__ chunks, int32_t *__restrict__ qn, ExpandCounters *cnt) {
    const unsigned lane = lane_id();
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nch = (int64_t)__ldcg(&cnt->chunks);
    unsigned long long scanned = 0;
    for (int64_t w = warp; w < nch; w += nwarps) {
        const uint2 ch = chunks[w];
        const int32_t v = (int32_t)ch.x;
        const int64_t end = off[v + 1];
        const int64_t e0 = off[v] + (int64_t)ch.y * kSplit;
        const int64_t e1 = min(end, e0 + kSplit);
        const auto pay = op.payload(v);
        scanned += e1 - e0;
        for (int64_t e = e0; e < e1; e += 32) {
            const int64_t ee = e + lane;
            bool push = false;
            int32_t x = 0;
            if (ee < e1) {
                x = adj[ee];
                push = op.visit(pay, ee, x);
            }
            int64_t slot = warp_append(push, &cnt->next_size);
            if (push) qn[slot] = x;
        }
    }
    if (lane == 0 && scanned) atomicAdd(&cnt->scanned, scanned);  // warp-uniform
}

// Chunk buffer capacity for a graph with m slots.
inline int64_t expand_chunk_capacity(int64_t m) { return 2 * (m / kSplit) + 2; }

// Launch both expansion kernels for one frontier.
template <class Op>
inline void launch_expand(const Op &op, const int64_t *off, const int32_t *adj, const int32_t *q,
                          int64_t nq, int32_t *qn, uint2 *chunks, ExpandCounters *cnt, int sms,
                          bool has_big_rows, cudaStream_t s, int64_t *launches) {
    const int cap = sms * 8;
    const int64_t warps_full = (int64_t)cap * (kExpandBlock / 32);
    int vpw = 32;
    while (vpw > 1 && (nq + vpw - 1) / vpw < warps_full) vpw >>= 1;
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
