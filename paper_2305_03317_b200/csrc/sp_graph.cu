// sp_graph.cu -- device CSR builder, device generators, graph handle.
//
// Replaces trident/graph.py:68-116 (_build_csr / from_edges) and the
// CsrGraph storage (graph.py:18-65).  The build runs entirely on the GPU:
//   slots (graph.py:107-113: edge, then its mirror if undirected and u != v)
//   -> 2b-bit keys (src << b | dst), values = slot index
//   -> stable LSD radix sort (CUB)  == Python's stable sort by (src, dst)
//   -> offsets from run boundaries, weights gathered through the permutation
//   -> w_eff (weight of the first slot of each equal-dst run; get_edge's
//      bisect_left, graph.py:56-62)
//   -> reverse CSR: stable sort of forward slots by (dst << b | src), which
//      yields graph.py:92's (dst, src, eid) order.
// Arrays stay resident; nothing is copied back unless the host asks for a
// view (sp_graph_download).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <mutex>
#include <new>

#include "sp_common.cuh"

using namespace sp;

namespace {

std::mutex g_lazy_mu;  // guards lazy reverse-eid construction

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

int bits_for(int64_t n) {
    int b = 1;
    while (b < 62 && ((int64_t)1 << b) < n) b++;
    return b;
}

__global__ void k_id_range(const int32_t *__restrict__ u, const int32_t *__restrict__ v,
                           int64_t ne, int *mn, int *mx) {
    int lo = 0x7fffffff, hi = -1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ne;
         i += (int64_t)gridDim.x * blockDim.x) {
        int a = u[i], b = v[i];
        lo = min(lo, min(a, b));
        hi = max(hi, max(a, b));
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mn, lo);
        atomicMax(mx, hi);
    }
}

__global__ void k_nonloop(const int32_t *__restrict__ u, const int32_t *__restrict__ v,
                          int64_t ne, int64_t *flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ne;
         i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = (u[i] != v[i]);
}

// Fill slot keys (src << b | dst) in graph.py:107-113 append order.
template <class IdxT>
__global__ void k_fill_slots(const int32_t *__restrict__ u, const int32_t *__restrict__ v,
                             const int32_t *__restrict__ w, int64_t ne,
                             const int64_t *__restrict__ excl, int directed, int b,
                             uint64_t *key, IdxT *val, int32_t *sw) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ne;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = directed ? i : i + excl[i];
        uint64_t a = (uint32_t)u[i], c = (uint32_t)v[i];
        key[p] = (a << b) | c;
        val[p] = (IdxT)p;
        sw[p] = w[i];
        if (!directed && a != c) {
            key[p + 1] = (c << b) | a;
            val[p + 1] = (IdxT)(p + 1);
            sw[p + 1] = w[i];
        }
    }
}

template <class IdxT>
__global__ void k_iota(IdxT *val, int64_t m) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        val[i] = (IdxT)i;
}

// Offsets from the sorted key's high part: off[x] = first e with src(e) >= x.
__global__ void k_offsets(const uint64_t *__restrict__ key, int64_t m, int64_t n, int b,
                          int64_t *off) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= m;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t prev = e == 0 ? -1 : (int64_t)(key[e - 1] >> b);
        int64_t cur = e == m ? n : (int64_t)(key[e] >> b);
        for (int64_t x = prev + 1; x <= cur; x++) off[x] = e;
    }
}

template <class IdxT>
__global__ void k_forward(const uint64_t *__restrict__ key, const IdxT *__restrict__ perm,
                          const int32_t *__restrict__ sw, int64_t m, int b,
                          int32_t *adj, int32_t *w, int64_t *runstart) {
    uint64_t mask = (1ull << b) - 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = key[e];
        adj[e] = (int32_t)(k & mask);
        w[e] = sw[perm[e]];
        runstart[e] = (e == 0 || key[e - 1] != k) ? e : 0;
    }
}

struct MaxOp {
    __device__ __forceinline__ int64_t operator()(int64_t a, int64_t b) const { return a > b ? a : b; }
};

__global__ void k_weff(const int32_t *__restrict__ w, const int64_t *__restrict__ runstart,
                       int64_t m, int32_t *weff) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x)
        weff[e] = w[runstart[e]];
}

__global__ void k_deg(const int64_t *__restrict__ off, int64_t n, int32_t *deg,
                      unsigned long long *maxdeg) {
    unsigned long long mx = 0;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        int64_t d = off[x + 1] - off[x];
        deg[x] = (int32_t)(d > 0x7fffffff ? 0x7fffffff : d);
        mx = max(mx, (unsigned long long)d);
    }
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxdeg, mx);
}

struct NonEmpty {
    const int32_t *deg;
    __device__ __forceinline__ bool operator()(int32_t x) const { return deg[x] > 0; }
};

__global__ void k_nzend(const int64_t *__restrict__ roff, const int32_t *__restrict__ nzrow,
                        const int64_t *__restrict__ cnt, int64_t *nzend) {
    const int64_t k1 = *cnt;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < k1;
         k += (int64_t)gridDim.x * blockDim.x)
        nzend[k] = roff[nzrow[k] + 1];
}

__global__ void k_wrange(const int32_t *__restrict__ w, int64_t m, int32_t *r) {
    int lo = 0x7fffffff, hi = (int)0x80000000;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        lo = min(lo, w[e]);
        hi = max(hi, w[e]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&r[0], lo);
        atomicMax(&r[1], hi);
    }
}

// w_eff of a forward CSR: weight of the first slot of each run of equal
// destinations within a row (get_edge's bisect_left, graph.py:56-62).
__global__ void k_weff_csr(const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
                           const int32_t *__restrict__ w, int64_t n, int32_t *weff) {
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t x = warp; x < n; x += nw) {
        const int64_t r0 = off[x], r1 = off[x + 1];
        for (int64_t e = r0 + lane_id(); e < r1; e += 32) {
            const int32_t d = adj[e];
            int64_t s = e;
            while (s > r0 && adj[s - 1] == d) s--;  // duplicates are rare and short
            weff[e] = w[s];
        }
    }
}

// Row id of every forward slot: the row starts are scattered (row x with
// slots marks off[x] with x), then an inclusive max-scan fills the rows.
// from_csr input checks (graph.py:18-36 invariants the device build relies
// on): off[0] == 0, off[n] == m, rows non-decreasing; every adj id in [0, n).
// bad[0] |= 1 for bad offsets, bad[0] |= 2 for an id out of range.
__global__ void k_check_off(const int64_t *__restrict__ off, int64_t n, int64_t m, int *bad) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x <= n;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = off[x];
        const bool ok = (x == 0 ? o == 0 : o >= off[x - 1]) && (x < n || o == m) && o <= m;
        if (!ok) atomicOr(bad, 1);
    }
}

__global__ void k_check_ids(const int32_t *__restrict__ adj, int64_t m, int64_t n, int *bad) {
    bool ok = true;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x)
        ok &= (uint32_t)adj[e] < (uint64_t)n;
    if (__any_sync(0xffffffffu, !ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 2);
}

__global__ void k_row_starts(const int64_t *__restrict__ off, int64_t n, uint32_t *mark) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x)
        if (off[x + 1] > off[x]) mark[off[x]] = (uint32_t)x;
}

struct MaxU32 {
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const {
        return a > b ? a : b;
    }
};

__global__ void k_fill_w(int32_t *w, int64_t m, int32_t v) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x)
        w[e] = v;
}

// off[x] = first e with key[e] >= x (sorted 32-bit keys).
__global__ void k_offsets32(const uint32_t *__restrict__ key, int64_t m, int64_t n, int64_t *off) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= m;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t prev = e == 0 ? -1 : (int64_t)key[e - 1];
        int64_t cur = e == m ? n : (int64_t)key[e];
        for (int64_t x = prev + 1; x <= cur; x++) off[x] = e;
    }
}

// Reverse keys from forward CSR: key2[e] = dst << b | src, in forward order.
__global__ void k_rev_keys(const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
                           int64_t n, int b, uint64_t *key2) {
    // one warp per source row
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t x = warp; x < n; x += nw)
        for (int64_t e = off[x] + lane_id(); e < off[x + 1]; e += 32)
            key2[e] = ((uint64_t)(uint32_t)adj[e] << b) | (uint64_t)x;
}

template <class IdxT>
__global__ void k_rev_out(const uint64_t *__restrict__ key2, const IdxT *__restrict__ perm,
                          int64_t m, int b, int32_t *radj, int64_t *reid) {
    uint64_t mask = (1ull << b) - 1;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (radj) radj[k] = (int32_t)(key2[k] & mask);
        if (reid) reid[k] = (int64_t)perm[k];
    }
}

// ---- device generators (bit-identical to paper_2305_03317_b200/gen.py) ----
__global__ void k_gen_rmat(int64_t ne, int scale, uint64_t sk, int ta, int tb, int tc,
                           int undirected, uint64_t *key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ne;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t u = 0, v = 0;
        int ngroups = (scale + 3) / 4;
        for (int g = 0; g < ngroups; g++) {
            uint64_t h = splitmix64(sk ^ (((uint64_t)i << 4) | (uint64_t)g));
#pragma unroll
            for (int j = 0; j < 4; j++) {
                int lvl = g * 4 + j;
                if (lvl >= scale) break;
                uint32_t r = (uint32_t)((h >> (16 * j)) & 0xFFFFu);
                uint64_t bu = r >= (uint32_t)tb;
                uint64_t bv = (r >= (uint32_t)ta && r < (uint32_t)tb) || r >= (uint32_t)tc;
                u |= bu << (scale - 1 - lvl);
                v |= bv << (scale - 1 - lvl);
            }
        }
        if (undirected && u > v) { uint64_t t = u; u = v; v = t; }
        key[i] = (u == v) ? ~0ull : ((u << 32) | v);
    }
}

__global__ void k_gen_uniform(int64_t ne, uint64_t n, uint64_t sk, int undirected, uint64_t *key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ne;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t h = splitmix64(sk ^ (uint64_t)i);
        uint64_t u = ((h >> 32) * n) >> 32;
        uint64_t v = ((h & 0xFFFFFFFFull) * n) >> 32;
        if (undirected && u > v) { uint64_t t = u; u = v; v = t; }
        key[i] = (u == v) ? ~0ull : ((u << 32) | v);
    }
}

__global__ void k_keys_to_edges(const uint64_t *__restrict__ key, int64_t ne, uint64_t wsk,
                                int32_t *u, int32_t *v, int32_t *w) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ne;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = key[i];
        u[i] = (int32_t)(k >> 32);
        v[i] = (int32_t)(k & 0xFFFFFFFFull);
        w[i] = (int32_t)(1 + splitmix64(k ^ wsk) % 100ull);
    }
}

__global__ void k_gen_grid(int64_t rows, int64_t cols, uint64_t wsk, int32_t *u, int32_t *v,
                           int32_t *w) {
    // cell c = r*cols + col emits right (if col+1<cols) then down (if r+1<rows);
    // slot index = 2*c - (#missing edges before c) computed in closed form.
    int64_t ncell = rows * cols;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell;
         c += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = c / cols, q = c % cols;
        // edges before cell c: full rows r*(2*cols-1) plus q*2 in this row
        // (each earlier cell in row r has right edge; down exists if r+1<rows)
        int64_t before = r * ((cols - 1) + cols) + q * (1 + (r + 1 < rows ? 1 : 0));
        int64_t p = before;
        if (q + 1 < cols) {
            uint64_t k = ((uint64_t)c << 32) | (uint64_t)(c + 1);
            u[p] = (int32_t)c; v[p] = (int32_t)(c + 1);
            w[p] = (int32_t)(1 + splitmix64(k ^ wsk) % 100ull);
            p++;
        }
        if (r + 1 < rows) {
            uint64_t k = ((uint64_t)c << 32) | (uint64_t)(c + cols);
            u[p] = (int32_t)c; v[p] = (int32_t)(c + cols);
            w[p] = (int32_t)(1 + splitmix64(k ^ wsk) % 100ull);
        }
    }
}

template <class F>
int cub_call(Call &c, F f) {
    size_t tmp = 0;
    SP_CUDA(f(nullptr, tmp));
    void *d = nullptr;
    SP_TRY(scratch_alloc(&d, tmp, c.stream));
    cudaError_t e = f(d, tmp);
    scratch_free(d, c.stream);
    SP_CUDA(e);
    return SP_OK;
}

int gridN(int64_t work, int dev) { return grid_for(work, 256, dev, 16); }

void free_graph(sp_graph *g) {
    if (!g) return;
    cudaSetDevice(g->device);
    resident_free(g->off);
    resident_free(g->adj);
    resident_free(g->w);
    resident_free(g->weff);
    if (g->directed) resident_free(g->rweff);
    resident_free(g->ell);
    resident_free(g->ell2);
    resident_free(g->outdeg);
    if (g->directed) {
        resident_free(g->roff);
        resident_free(g->radj);
        resident_free(g->indeg);
    }
    resident_free(g->reid);
    resident_free(g->nzrow);
    resident_free(g->nzend);
    resident_free(g->ustart8);
    resident_free(g->ulen);
    resident_free(g->uadj);
    resident_free(g->uinfo);
    resident_free(g->ubig);
    resident_free(g->uorder);
    resident_free(g->pr_hot_ids);
    resident_free(g->pr_radj_hot);
    resident_free(g->pr_unit_row);
    resident_free(g->rel_perm);
    resident_free(g->rel_radj);
    resident_free(g->rel_outdeg);
    resident_free(g->rel_indeg);
    resident_free(g->rel_nzrow);
    resident_free(g->rel_nzend);
    resident_free(g->rel_unit_row);
    resident_free(g->wrange);
    for (auto &ev : g->prep_ev)
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
    delete g;
}


template <class T>
int dalloc(T **p, size_t count) {
    void *q = nullptr;
    SP_TRY(resident_alloc(&q, count * sizeof(T) + 16));
    *p = static_cast<T *>(q);
    return SP_OK;
}

// Reverse CSR from the forward arrays (graph.py:84-96).
template <class IdxT>
int build_reverse_t(sp_graph *g, Call &c, bool want_adj, bool want_eid) {
    int64_t n = g->n, m = g->m;
    int b = bits_for(n);
    uint64_t *k2, *k2s;
    IdxT *vi, *vo;
    SP_TRY(c.alloc(&k2, m));
    SP_TRY(c.alloc(&k2s, m));
    SP_TRY(c.alloc(&vi, m));
    SP_TRY(c.alloc(&vo, m));
    k_rev_keys<<<gridN(n * 32, c.device), 256, 0, c.stream>>>(g->off, g->adj, n, b, k2);
    k_iota<IdxT><<<gridN(m, c.device), 256, 0, c.stream>>>(vi, m);
    if (m)
        SP_TRY(cub_call(c, [&](void *t, size_t &sz) {
            return cub::DeviceRadixSort::SortPairs(t, sz, k2, k2s, vi, vo, m, 0, 2 * b, c.stream);
        }));
    if (want_adj) {
        SP_TRY(dalloc(&g->roff, n + 1));
        SP_TRY(dalloc(&g->radj, m));
        k_offsets<<<gridN(m + 1, c.device), 256, 0, c.stream>>>(k2s, m, n, b, g->roff);
    }
    if (want_eid) SP_TRY(dalloc(&g->reid, m));
    k_rev_out<IdxT><<<gridN(m, c.device), 256, 0, c.stream>>>(
        k2s, vo, m, b, want_adj ? g->radj : nullptr, want_eid ? g->reid : nullptr);
    SP_CUDA(cudaGetLastError());
    return SP_OK;
}

// Reverse adjacency only (the algorithm path): a stable LSD radix sort of
// the b-bit destination keys carrying the source ids.  The input is in
// forward slot order, i.e. (src, eid) order, so the stable sort yields
// graph.py:92's (dst, src, eid) order with b/8 passes over 32-bit keys.
int build_reverse_adj(sp_graph *g, Call &c) {
    const int64_t n = g->n, m = g->m;
    const int b = bits_for(n);
    uint32_t *dks, *sv;
    SP_TRY(c.alloc(&dks, m));
    SP_TRY(c.alloc(&sv, m));
    SP_TRY(dalloc(&g->roff, n + 1));
    SP_TRY(dalloc(&g->radj, m));
    // source of every slot (slots are in (src, eid) order): scatter + max-scan
    SP_CUDA(cudaMemsetAsync(sv, 0, m * sizeof(uint32_t), c.stream));
    k_row_starts<<<gridN(n, c.device), 256, 0, c.stream>>>(g->off, n, sv);
    if (m)
        SP_TRY(cub_call(c, [&](void *t, size_t &sz) {
            return cub::DeviceScan::InclusiveScan(t, sz, sv, sv, MaxU32(), m, c.stream);
        }));
    // the destinations are the forward adj itself (the sort keys)
    const uint32_t *dk = reinterpret_cast<const uint32_t *>(g->adj);
    if (m)
        SP_TRY(cub_call(c, [&](void *t, size_t &sz) {
            return cub::DeviceRadixSort::SortPairs(t, sz, dk, dks, sv,
                                                   reinterpret_cast<uint32_t *>(g->radj), m, 0,
                                                   b, c.stream);
        }));
    k_offsets32<<<gridN(m + 1, c.device), 256, 0, c.stream>>>(dks, m, n, g->roff);
    SP_CUDA(cudaGetLastError());
    return SP_OK;
}

// ---- pipelined upload + reverse build (host CSR input, directed) -------
// The adjacency crosses PCIe in kUpChunks pieces on a copy stream; each
// piece is stably sorted by destination (carrying its source ids, which
// come from the offsets alone) while the next one is in flight, and its
// row starts start_i[x] = #(keys < x in piece i) are recorded.  Then
// roff[x] = sum_i start_i[x], and element j of piece i with destination x
// lands at roff[x] + sum_{i' < i} cnt_i'(x) + (j - start_i[x]) -- the
// (dst, src) order of graph.py:92, with one scatter after the last piece
// instead of a full sort behind the whole upload.
constexpr int kUpChunks = 8;
constexpr int64_t kUpMinSlots = int64_t(1) << 23;  // smaller graphs: one copy + one sort

// start[x] = first j with key[j] >= x, x in [0, n] (key sorted, mc keys)
// An id outside [0, n) (caller error, reported after the build) is clamped
// to n here and skipped by k_up_scatter: no out-of-range writes.
__global__ void k_start32(const uint32_t *__restrict__ key, int64_t mc, int64_t n,
                          uint32_t *start, int *bad) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= mc;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t prev = e == 0 ? -1 : min((int64_t)key[e - 1], n);
        int64_t cur = n;
        if (e < mc) {
            cur = (int64_t)key[e];
            if (cur >= n) {
                atomicOr(bad, 2);
                cur = n;
            }
        }
        for (int64_t x = prev + 1; x <= cur; x++) start[x] = (uint32_t)e;
    }
}

// roff[x] and base_i[x] = roff[x] + sum_{i'<i} cnt_i'(x) - start_i[x]
__global__ void k_up_bases(const uint32_t *__restrict__ start, int C, int64_t n, int64_t *roff,
                           int64_t *base) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x <= n;
         x += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = 0;
        for (int i = 0; i < C; i++) r += start[(int64_t)i * (n + 1) + x];
        roff[x] = r;
        if (x == n) continue;
        int64_t before = 0;
        for (int i = 0; i < C; i++) {
            const int64_t si = start[(int64_t)i * (n + 1) + x];
            base[(int64_t)i * n + x] = r + before - si;
            before += (int64_t)start[(int64_t)i * (n + 1) + x + 1] - si;
        }
    }
}

// radj (and, when the PR hot set exists, its hot-encoded copy) in one pass
__global__ void k_up_scatter(const uint32_t *__restrict__ dks, const uint32_t *__restrict__ svs,
                             int64_t mc, int64_t n, int64_t m, const int64_t *__restrict__ base,
                             int32_t *radj,
                             const int32_t *__restrict__ hot_idx, int32_t *enc) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < mc;
         j += (int64_t)gridDim.x * blockDim.x) {
        if ((int64_t)dks[j] >= n) continue;  // bad id (k_start32 flagged it)
        const int64_t pos = base[dks[j]] + j;
        if ((uint64_t)pos >= (uint64_t)m) continue;  // only with bad ids elsewhere
        const int32_t u = (int32_t)svs[j];
        radj[pos] = u;
        if (enc) {
            const int32_t h = hot_idx[u];
            enc[pos] = h >= 0 ? (kPrHotBit | h) : u;
        }
    }
}

__global__ void k_outdeg(const int64_t *__restrict__ off, int64_t n, int32_t *deg,
                         unsigned long long *mx) {
    unsigned long long best = 0;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = off[x + 1] - off[x];
        deg[x] = (int32_t)d;
        best = best > (unsigned long long)d ? best : (unsigned long long)d;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
        best = best > t ? best : t;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(mx, best);
}

int upload_adj_build_reverse(sp_graph *g, Call &c, const int32_t *adj_host, int *bad) {
    const int64_t n = g->n, m = g->m;
    const int b = bits_for(n);
    const int C = kUpChunks;
    uint32_t *sv, *dks, *svs, *start;
    int64_t *base;
    SP_TRY(c.alloc(&sv, m));
    SP_TRY(c.alloc(&dks, m));
    SP_TRY(c.alloc(&svs, m));
    SP_TRY(c.alloc(&start, (int64_t)C * (n + 1)));
    SP_TRY(c.alloc(&base, (int64_t)C * n + 1));
    SP_TRY(dalloc(&g->roff, n + 1));
    SP_TRY(dalloc(&g->radj, m));
    cudaStream_t cs = nullptr;
    cudaEvent_t ev[kUpChunks] = {}, ready = nullptr;
    struct Res {
        cudaStream_t *s;
        cudaEvent_t *e;
        cudaEvent_t *r;
        ~Res() {
            for (int i = 0; i < kUpChunks; i++)
                if (e[i]) cudaEventDestroy(e[i]);
            if (*r) cudaEventDestroy(*r);
            if (*s) cudaStreamDestroy(*s);
        }
    } res{&cs, ev, &ready};
    SP_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    SP_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    for (int i = 0; i < C; i++) SP_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    // the copies may only start once the call's stream has allocated g->adj
    SP_CUDA(cudaEventRecord(ready, c.stream));
    SP_CUDA(cudaStreamWaitEvent(cs, ready, 0));
    int64_t cut[kUpChunks + 1];
    for (int i = 0; i <= C; i++) cut[i] = m * i / C;
    for (int i = 0; i < C; i++) {
        SP_CUDA(cudaMemcpyAsync(g->adj + cut[i], adj_host + cut[i],
                                (cut[i + 1] - cut[i]) * sizeof(int32_t), cudaMemcpyHostToDevice,
                                cs));
        SP_CUDA(cudaEventRecord(ev[i], cs));
    }
    // source of every slot, from the offsets only (overlaps the copies)
    SP_CUDA(cudaMemsetAsync(sv, 0, m * sizeof(uint32_t), c.stream));
    k_row_starts<<<gridN(n, c.device), 256, 0, c.stream>>>(g->off, n, sv);
    SP_TRY(cub_call(c, [&](void *t, size_t &sz) {
        return cub::DeviceScan::InclusiveScan(t, sz, sv, sv, MaxU32(), m, c.stream);
    }));
    // PageRank hot sources, chosen from the offsets alone while the copies
    // run: the scatter below then writes the hot-encoded radj too, so the
    // first PR call on the graph already has it (sp_pagerank.cu)
    int32_t *hot_idx = nullptr, *enc = nullptr;
    int H = 0;
    if (!getenv("SP_UPLOAD_NO_HOT")) {
        int32_t *deg;
        unsigned long long *mx;
        SP_TRY(c.alloc(&deg, n));
        SP_TRY(c.alloc(&mx, 1));
        SP_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned long long), c.stream));
        k_outdeg<<<gridN(n, c.device), 256, 0, c.stream>>>(g->off, n, deg, mx);
        unsigned long long *hm;
        SP_TRY(c.host_as(&hm));
        SP_CUDA(cudaMemcpyAsync(hm, mx, 8, cudaMemcpyDeviceToHost, c.stream));
        SP_CUDA(cudaStreamSynchronize(c.stream));  // the copies continue on their stream
        SP_TRY(pr_hot_prepare(g, c, deg, (int64_t)hm[0], &hot_idx, &H));
        if (H > 0 && dalloc(&enc, m) != SP_OK) {  // optional: no memory -> no hot set
            cudaGetLastError();
            resident_free(g->pr_hot_ids);
            g->pr_hot_ids = nullptr;
            enc = nullptr;
            hot_idx = nullptr;
            H = 0;
        }
    }
    const uint32_t *dk = reinterpret_cast<const uint32_t *>(g->adj);
    for (int i = 0; i < C; i++) {
        const int64_t e0 = cut[i], mc = cut[i + 1] - cut[i];
        SP_CUDA(cudaStreamWaitEvent(c.stream, ev[i], 0));
        if (mc)
            SP_TRY(cub_call(c, [&](void *t, size_t &sz) {
                return cub::DeviceRadixSort::SortPairs(t, sz, dk + e0, dks + e0, sv + e0,
                                                       svs + e0, mc, 0, b, c.stream);
            }));
        k_start32<<<gridN(mc + 1, c.device), 256, 0, c.stream>>>(
            dks + e0, mc, n, start + (int64_t)i * (n + 1), bad);
    }
    k_up_bases<<<gridN(n + 1, c.device), 256, 0, c.stream>>>(start, C, n, g->roff, base);
    for (int i = 0; i < C; i++) {
        const int64_t e0 = cut[i], mc = cut[i + 1] - cut[i];
        if (mc)
            k_up_scatter<<<gridN(mc, c.device), 256, 0, c.stream>>>(
                dks + e0, svs + e0, mc, n, m, base + (int64_t)i * n, g->radj, hot_idx, enc);
    }
    SP_CUDA(cudaGetLastError());
    if (H > 0) {
        g->pr_radj_hot = enc;
        g->pr_H = H;
    }
    return SP_OK;
}

int build_reverse(sp_graph *g, Call &c, bool want_adj, bool want_eid) {
    if (want_adj && !want_eid) return build_reverse_adj(g, c);
    if (g->m < (int64_t)0xFFFFFFFFll) return build_reverse_t<uint32_t>(g, c, want_adj, want_eid);
    return build_reverse_t<uint64_t>(g, c, want_adj, want_eid);
}

int finish_graph(sp_graph *g, Call &c, bool unit_weights = false) {
    int64_t n = g->n, m = g->m;
    unsigned long long *cnt;
    SP_TRY(c.alloc(&cnt, 4));
    SP_CUDA(cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), c.stream));
    SP_TRY(dalloc(&g->outdeg, n));
    k_deg<<<gridN(n, c.device), 256, 0, c.stream>>>(g->off, n, g->outdeg, cnt + 0);
    if (g->directed) {
        if (!g->roff) SP_TRY(build_reverse(g, c, true, false));  // else built while uploading
        SP_TRY(dalloc(&g->indeg, n));
        k_deg<<<gridN(n, c.device), 256, 0, c.stream>>>(g->roff, n, g->indeg, cnt + 1);
    } else {
        g->roff = g->off;
        g->radj = g->adj;
        g->indeg = g->outdeg;
    }
    // non-empty in-rows, order-preserving compaction (ascending v)
    SP_TRY(dalloc(&g->nzrow, n));
    SP_TRY(dalloc(&g->nzend, n));
    if (n) {
        int64_t *nsel = reinterpret_cast<int64_t *>(cnt + 2);
        NonEmpty pred{g->indeg};
        SP_TRY(cub_call(c, [&](void *t, size_t &sz) {
            return cub::DeviceSelect::If(t, sz, thrust::counting_iterator<int32_t>(0), g->nzrow,
                                         nsel, (int64_t)n, pred, c.stream);
        }));
        k_nzend<<<gridN(n, c.device), 256, 0, c.stream>>>(g->roff, g->nzrow, nsel, g->nzend);
    }
    SP_TRY(dalloc(&g->wrange, 2));
    int32_t init[2] = {0x7fffffff, (int32_t)0x80000000};
    SP_CUDA(cudaMemcpyAsync(g->wrange, init, sizeof(init), cudaMemcpyHostToDevice, c.stream));
    if (m && unit_weights) {  // every slot weight 1: no pass over w
        const int32_t one[2] = {1, 1};
        SP_CUDA(cudaMemcpyAsync(g->wrange, one, sizeof(one), cudaMemcpyHostToDevice, c.stream));
    } else if (m) {
        k_wrange<<<gridN(m, c.device), 256, 0, c.stream>>>(g->w, m, g->wrange);
    }
    unsigned long long h[4];
    int32_t wr[2] = {0, 0};
    SP_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    if (m) SP_CUDA(cudaMemcpyAsync(wr, g->wrange, sizeof(wr), cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    SP_CUDA(cudaGetLastError());
    g->wmin_h = wr[0];
    g->wmax_h = wr[1];
    g->max_outdeg = (int64_t)h[0];
    g->max_indeg = g->directed ? (int64_t)h[1] : (int64_t)h[0];
    g->nnz_rows = (int64_t)h[2];
    return SP_OK;
}

// Forward build from device edge arrays.
template <class IdxT>
int build_forward_t(sp_graph *g, Call &c, const int32_t *u, const int32_t *v,
                    const int32_t *w, int64_t ne) {
    int64_t n = g->n, m = g->m;
    int b = bits_for(n);
    int64_t *excl = nullptr;
    if (!g->directed) {
        SP_TRY(c.alloc(&excl, ne + 1));
        k_nonloop<<<gridN(ne, c.device), 256, 0, c.stream>>>(u, v, ne, excl);
        SP_TRY(cub_call(c, [&](void *t, size_t &sz) {
            return cub::DeviceScan::ExclusiveSum(t, sz, excl, excl, ne, c.stream);
        }));
    }
    uint64_t *key, *keys;
    IdxT *vi, *perm;
    int32_t *sw;
    SP_TRY(c.alloc(&key, m));
    SP_TRY(c.alloc(&keys, m));
    SP_TRY(c.alloc(&vi, m));
    SP_TRY(c.alloc(&perm, m));
    SP_TRY(c.alloc(&sw, m));
    if (ne)
        k_fill_slots<IdxT><<<gridN(ne, c.device), 256, 0, c.stream>>>(u, v, w, ne, excl, g->directed,
                                                                      b, key, vi, sw);
    if (m)
        SP_TRY(cub_call(c, [&](void *t, size_t &sz) {
            return cub::DeviceRadixSort::SortPairs(t, sz, key, keys, vi, perm, m, 0, 2 * b, c.stream);
        }));
    SP_TRY(dalloc(&g->off, n + 1));
    SP_TRY(dalloc(&g->adj, m));
    SP_TRY(dalloc(&g->w, m));
    SP_TRY(dalloc(&g->weff, m));
    int64_t *runstart;
    SP_TRY(c.alloc(&runstart, m));
    k_offsets<<<gridN(m + 1, c.device), 256, 0, c.stream>>>(keys, m, n, b, g->off);
    if (m) {
        k_forward<IdxT><<<gridN(m, c.device), 256, 0, c.stream>>>(keys, perm, sw, m, b, g->adj, g->w,
                                                                  runstart);
        SP_TRY(cub_call(c, [&](void *t, size_t &sz) {
            return cub::DeviceScan::InclusiveScan(t, sz, runstart, runstart, MaxOp(), m, c.stream);
        }));
        k_weff<<<gridN(m, c.device), 256, 0, c.stream>>>(g->w, runstart, m, g->weff);
    }
    SP_CUDA(cudaGetLastError());
    return SP_OK;
}

int build_from_device_edges(sp_graph *g, Call &c, const int32_t *u, const int32_t *v,
                            const int32_t *w, int64_t ne, int64_t n_hint) {
    // vertex count and id validation (graph.py:110,114)
    int *mm;
    SP_TRY(c.alloc(&mm, 2));
    int init[2] = {0x7fffffff, -1};
    SP_CUDA(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, c.stream));
    if (ne) k_id_range<<<gridN(ne, c.device), 256, 0, c.stream>>>(u, v, ne, mm, mm + 1);
    int h[2];
    SP_CUDA(cudaMemcpyAsync(h, mm, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    int64_t *nl = nullptr;
    SP_CUDA(cudaStreamSynchronize(c.stream));
    SP_CHECK(ne == 0 || h[0] >= 0, SP_ERR_ARG, "negative vertex id %d in edge list", h[0]);
    int64_t n = n_hint > (int64_t)h[1] + 1 ? n_hint : (int64_t)h[1] + 1;
    SP_CHECK(n < 0x7fffffffll, SP_ERR_UNSUPPORTED, "n = %lld exceeds int32 vertex ids", (long long)n);
    g->n = n;
    int64_t m = ne;
    if (!g->directed && ne) {
        // m = ne + #non-loop edges
        SP_TRY(c.alloc(&nl, ne));
        k_nonloop<<<gridN(ne, c.device), 256, 0, c.stream>>>(u, v, ne, nl);
        int64_t *tot;
        SP_TRY(c.alloc(&tot, 1));
        SP_TRY(cub_call(c, [&](void *t, size_t &sz) {
            return cub::DeviceReduce::Sum(t, sz, nl, tot, ne, c.stream);
        }));
        int64_t ht = 0;
        SP_CUDA(cudaMemcpyAsync(&ht, tot, sizeof(ht), cudaMemcpyDeviceToHost, c.stream));
        SP_CUDA(cudaStreamSynchronize(c.stream));
        m += ht;
    }
    g->m = m;
    if (m < (int64_t)0xFFFFFFFFll)
        SP_TRY(build_forward_t<uint32_t>(g, c, u, v, w, ne));
    else
        SP_TRY(build_forward_t<uint64_t>(g, c, u, v, w, ne));
    return finish_graph(g, c);
}

int new_graph(int directed, int device, sp_graph **out) {
    sp_graph *g = new (std::nothrow) sp_graph();
    SP_CHECK(g, SP_ERR_OOM, "host allocation failed");
    g->directed = directed ? 1 : 0;
    g->device = device;
    *out = g;
    return SP_OK;
}

// Dedupe sorted 64-bit keys in place; drop the ~0 self-loop sentinel.
int unique_keys(Call &c, uint64_t *key, int64_t ne, uint64_t **uniq, int64_t *nu) {
    uint64_t *keys, *outk;
    SP_TRY(c.alloc(&keys, ne));
    SP_TRY(c.alloc(&outk, ne));
    SP_TRY(cub_call(c, [&](void *t, size_t &sz) {
        return cub::DeviceRadixSort::SortKeys(t, sz, key, keys, ne, 0, 64, c.stream);
    }));
    int64_t *cnt;
    SP_TRY(c.alloc(&cnt, 1));
    SP_TRY(cub_call(c, [&](void *t, size_t &sz) {
        return cub::DeviceSelect::Unique(t, sz, keys, outk, cnt, ne, c.stream);
    }));
    int64_t h = 0;
    SP_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    SP_CUDA(cudaStreamSynchronize(c.stream));
    if (h > 0) {
        uint64_t last = 0;
        SP_CUDA(cudaMemcpy(&last, outk + h - 1, sizeof(last), cudaMemcpyDeviceToHost));
        if (last == ~0ull) h--;
    }
    *uniq = outk;
    *nu = h;
    return SP_OK;
}

}  // namespace

namespace sp {

void prep_mark(sp_graph *g, int kind, int end, cudaStream_t s) {
    if (kind < 0 || kind >= kPrepKinds) return;
    cudaEvent_t &e = g->prep_ev[kind][end ? 1 : 0];
    if (!e && cudaEventCreate(&e) != cudaSuccess) {
        cudaGetLastError();
        e = nullptr;
        return;
    }
    cudaEventRecord(e, s);
}

// w_eff on first use (graphs adopted from a CSR defer it; see from_csr).
int ensure_weff(sp_graph *g, Call &c) {
    std::lock_guard<std::mutex> lk(g_lazy_mu);
    if (g->weff || g->m == 0) return SP_OK;
    int32_t *weff = nullptr;
    prep_mark(g, kPrepWeff, 0, c.stream);
    SP_TRY(dalloc(&weff, g->m));
    k_weff_csr<<<gridN(g->n * 32, c.device), 256, 0, c.stream>>>(g->off, g->adj, g->w, g->n, weff);
    prep_mark(g, kPrepWeff, 1, c.stream);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
    if (e != cudaSuccess) {
        resident_free(weff);
        SP_CUDA(e);
    }
    g->weff = weff;
    return SP_OK;
}

__global__ void k_rweff(const int32_t *__restrict__ weff, const int64_t *__restrict__ reid,
                        int64_t m, int32_t *rw) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
         k += (int64_t)gridDim.x * blockDim.x)
        rw[k] = weff[reid[k]];
}

__global__ void k_ell_fill(const int64_t *__restrict__ off, const int32_t *__restrict__ adj,
                           const int32_t *__restrict__ weff, int64_t n, int d, int2 *ell) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * d;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / d, k = i - v * d;
        const int64_t e = off[v] + k;
        ell[i] = e < off[v + 1] ? make_int2(adj[e], weff[e]) : make_int2(-1, 0);
    }
}

template <int S>
__global__ void k_ell2_fill(const int2 *__restrict__ ell, int d, int64_t n, int hops, int2 *ell2) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        int2 out[S];
        int cnt = 0;
        auto put = [&](int32_t y, int64_t w) {
            if (y < 0 || y == (int32_t)v || w > 0x7fffffffll) return;
            for (int k = 0; k < cnt; k++)
                if (out[k].x == y) {
                    if (w < out[k].y) out[k].y = (int)w;
                    return;
                }
            if (cnt < S) out[cnt++] = make_int2(y, (int)w);
        };
        for (int i = 0; i < d; i++) {
            const int2 e = ell[v * d + i];
            put(e.x, e.y);
        }
        // one more hop from every entry so far, `hops - 1` times (the 1-hop
        // entries come first, so they are never crowded out)
        int lo = 0;
        for (int h = 1; h < hops; h++) {
            const int hi = cnt;
            for (int k = lo; k < hi; k++) {
                const int32_t x = out[k].x;
                const int64_t wx = out[k].y;
                for (int j = 0; j < d; j++) {
                    const int2 f = ell[(int64_t)x * d + j];
                    if (f.x >= 0) put(f.x, wx + (int64_t)f.y);
                }
            }
            lo = hi;
        }
        for (int k = 0; k < S; k++) ell2[v * S + k] = k < cnt ? out[k] : make_int2(-1, 0);
    }
}

int ensure_ell2(sp_graph *g, Call &c, int hops) {
    std::lock_guard<std::mutex> lk(g_lazy_mu);
    if (g->ell2 || !g->ell || g->ell_d > 4 || g->n == 0) return SP_OK;
    const int S = hops >= 3 ? kEll3 : kEll2;
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
        cudaGetLastError();
        return SP_OK;
    }
    if ((double)g->n * S * sizeof(int2) > 0.25 * (double)fr) return SP_OK;  // optional
    int2 *e2 = nullptr;
    if (dalloc(&e2, g->n * S) != SP_OK) {
        cudaGetLastError();
        return SP_OK;
    }
    prep_mark(g, kPrepEll2, 0, c.stream);
    if (S == kEll3)
        k_ell2_fill<kEll3><<<gridN(g->n, c.device), 256, 0, c.stream>>>(g->ell, g->ell_d, g->n, 3, e2);
    else
        k_ell2_fill<kEll2><<<gridN(g->n, c.device), 256, 0, c.stream>>>(g->ell, g->ell_d, g->n, 2, e2);
    prep_mark(g, kPrepEll2, 1, c.stream);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
    if (e != cudaSuccess) {
        resident_free(e2);
        SP_CUDA(e);
    }
    g->ell2 = e2;
    g->ell2_slots = S;
    return SP_OK;
}

int ensure_ell(sp_graph *g, Call &c, int d_max) {
    std::lock_guard<std::mutex> lk(g_lazy_mu);
    if (g->ell || g->max_outdeg > d_max || g->n == 0) return SP_OK;
    int d = 2;  // rows are read as 16-byte pairs of slots
    while (d < g->max_outdeg) d <<= 1;
    // an optional copy: skipped (CSR rows) when it would not fit comfortably
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
        cudaGetLastError();
        return SP_OK;
    }
    if ((double)g->n * d * sizeof(int2) > 0.25 * (double)fr) return SP_OK;
    int2 *ell = nullptr;
    prep_mark(g, kPrepEll, 0, c.stream);
    if (dalloc(&ell, g->n * d) != SP_OK) {
        cudaGetLastError();
        return SP_OK;
    }
    k_ell_fill<<<gridN(g->n * d, c.device), 256, 0, c.stream>>>(g->off, g->adj, g->weff, g->n, d,
                                                                 ell);
    prep_mark(g, kPrepEll, 1, c.stream);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
    if (e != cudaSuccess) {
        resident_free(ell);
        SP_CUDA(e);
    }
    g->ell = ell;
    g->ell_d = d;
    return SP_OK;
}

int ensure_rweff(sp_graph *g, Call &c) {
    SP_TRY(ensure_weff(g, c));
    std::lock_guard<std::mutex> lk(g_lazy_mu);
    if (g->rweff || g->m == 0) return SP_OK;
    if (!g->directed) {  // reverse CSR == forward CSR, mirrored slots share runs (F11)
        g->rweff = g->weff;
        return SP_OK;
    }
    prep_mark(g, kPrepRweff, 0, c.stream);
    if (!g->reid) SP_TRY(build_reverse(g, c, false, true));
    int32_t *rw = nullptr;
    SP_TRY(dalloc(&rw, g->m));
    k_rweff<<<gridN(g->m, c.device), 256, 0, c.stream>>>(g->weff, g->reid, g->m, rw);
    prep_mark(g, kPrepRweff, 1, c.stream);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
    if (e != cudaSuccess) {
        resident_free(rw);
        SP_CUDA(e);
    }
    g->rweff = rw;
    return SP_OK;
}

}  // namespace sp

extern "C" {

int sp_graph_prep_ms(const sp_graph *g, int kind, double *ms) {
    SP_CHECK(g && ms && kind >= 0 && kind < kPrepKinds, SP_ERR_ARG,
             "sp_graph_prep_ms: bad arguments");
    *ms = -1.0;
    cudaEvent_t a = g->prep_ev[kind][0], b = g->prep_ev[kind][1];
    if (!a || !b) return SP_OK;  // not built (or built at creation, untimed)
    SP_CUDA(cudaSetDevice(g->device));
    SP_CUDA(cudaEventSynchronize(b));
    float f = 0.f;
    SP_CUDA(cudaEventElapsedTime(&f, a, b));
    *ms = f;
    return SP_OK;
}

int sp_graph_from_edges(const int32_t *u, const int32_t *v, const int32_t *w, int64_t nedges,
                        int64_t n, int directed, int mem, int device, sp_graph **out) {
    SP_CHECK(out && nedges >= 0 && (nedges == 0 || (u && v && w)), SP_ERR_ARG,
             "sp_graph_from_edges: bad arguments");
    *out = nullptr;
    Call c;
    SP_TRY(c.begin(device));
    const int32_t *du = u, *dv = v, *dw = w;
    if (mem == SP_MEM_HOST && nedges) {
        int32_t *a, *b2, *cc;
        SP_TRY(c.alloc(&a, nedges));
        SP_TRY(c.alloc(&b2, nedges));
        SP_TRY(c.alloc(&cc, nedges));
        SP_TRY(to_device(a, u, nedges * 4, mem, c.stream));
        SP_TRY(to_device(b2, v, nedges * 4, mem, c.stream));
        SP_TRY(to_device(cc, w, nedges * 4, mem, c.stream));
        du = a; dv = b2; dw = cc;
    }
    sp_graph *g;
    SP_TRY(new_graph(directed, device, &g));
    int rc = build_from_device_edges(g, c, du, dv, dw, nedges, n);
    if (rc == SP_OK) rc = c.finish(nullptr);
    if (rc != SP_OK) {
        free_graph(g);
        return rc;
    }
    *out = g;
    return SP_OK;
}

// SP_CUDA for a do { } while (0) build block: record rc and leave the block
#define SP_CUDA_BREAK(call)                                                  \
    {                                                                        \
        cudaError_t _e = (call);                                             \
        if (_e != cudaSuccess) {                                             \
            rc = ::sp::cuda_fail(_e, #call, __FILE__, __LINE__);             \
            break;                                                           \
        }                                                                    \
    }

int sp_graph_from_csr(const int64_t *offsets, const int32_t *adj, const int32_t *weights,
                      int64_t n, int64_t m, int directed, int mem, int device, sp_graph **out) {
    SP_CHECK(out && n >= 0 && m >= 0 && offsets, SP_ERR_ARG, "sp_graph_from_csr: bad arguments");
    SP_CHECK(n < 0x7fffffffll, SP_ERR_UNSUPPORTED, "n exceeds int32 vertex ids");
    *out = nullptr;
    Call c;
    SP_TRY(c.begin(device));
    sp_graph *g;
    SP_TRY(new_graph(directed, device, &g));
    g->n = n;
    g->m = m;
    int rc = SP_OK;
    do {
        if ((rc = dalloc(&g->off, n + 1))) break;
        if ((rc = dalloc(&g->adj, m))) break;
        if ((rc = dalloc(&g->w, m))) break;
        if ((rc = to_device(g->off, offsets, (n + 1) * 8, mem, c.stream))) break;
        // the offsets are trusted by every build kernel: checked first
        int *bad, *hbad;
        if ((rc = c.alloc(&bad, 1)) || (rc = c.host_as(&hbad))) break;
        SP_CUDA_BREAK(cudaMemsetAsync(bad, 0, sizeof(int), c.stream));
        k_check_off<<<gridN(n + 1, c.device), 256, 0, c.stream>>>(g->off, n, m, bad);
        SP_CUDA_BREAK(cudaMemcpyAsync(hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
        SP_CUDA_BREAK(cudaStreamSynchronize(c.stream));
        if (*hbad) {
            set_error("sp_graph_from_csr: offsets must start at 0, be non-decreasing and end "
                      "at m = %lld", (long long)m);
            rc = SP_ERR_ARG;
            break;
        }
        // large directed host CSR: the reverse CSR is built while the
        // adjacency is still crossing PCIe (ids checked in flight, k_start32)
        const bool pipelined = directed && mem == SP_MEM_HOST && m >= kUpMinSlots &&
                               m < (int64_t)0xFFFFFFFFll && !getenv("SP_UPLOAD_PLAIN");
        if (pipelined) {
            if ((rc = upload_adj_build_reverse(g, c, adj, bad))) break;
        } else {
            if ((rc = to_device(g->adj, adj, m * 4, mem, c.stream))) break;
            if (m) k_check_ids<<<gridN(m, c.device), 256, 0, c.stream>>>(g->adj, m, n, bad);
            SP_CUDA_BREAK(cudaMemcpyAsync(hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
            SP_CUDA_BREAK(cudaStreamSynchronize(c.stream));
        }
        if (!pipelined && *hbad) {
            set_error("sp_graph_from_csr: adjacency id outside [0, %lld)", (long long)n);
            rc = SP_ERR_ARG;
            break;
        }
        if (weights) {
            if ((rc = to_device(g->w, weights, m * 4, mem, c.stream))) break;
        } else if (m) {  // unweighted CSR: every slot has the default weight 1
            k_fill_w<<<gridN(m, c.device), 256, 0, c.stream>>>(g->w, m, 1);
        }
        // w_eff is built on first use (ensure_weff): PR/BC/TC never read it
        if ((rc = finish_graph(g, c, weights == nullptr))) break;
        if (pipelined) {  // finish_graph synchronised the stream
            SP_CUDA_BREAK(cudaMemcpyAsync(hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
            SP_CUDA_BREAK(cudaStreamSynchronize(c.stream));
            if (*hbad) {
                set_error("sp_graph_from_csr: adjacency id outside [0, %lld)", (long long)n);
                rc = SP_ERR_ARG;
                break;
            }
        }
        rc = c.finish(nullptr);
    } while (0);
    if (rc != SP_OK) {
        free_graph(g);
        return rc;
    }
    *out = g;
    return SP_OK;
}

int sp_graph_generate(int kind, int64_t p0, int64_t p1, int64_t seed, int undirected, int device,
                      sp_graph **out) {
    SP_CHECK(out, SP_ERR_ARG, "sp_graph_generate: out is NULL");
    *out = nullptr;
    Call c;
    SP_TRY(c.begin(device));
    uint64_t sk = splitmix64((uint64_t)seed);
    uint64_t wsk = splitmix64((uint64_t)seed ^ 0x5EEDull);
    int32_t *u, *v, *w;
    int64_t ne = 0, n = 0;
    if (kind == SP_GEN_GRID) {
        SP_CHECK(p0 > 0 && p1 > 0 && p0 * p1 < 0x7fffffffll, SP_ERR_ARG, "bad grid size");
        n = p0 * p1;
        ne = p0 * (p1 - 1) + (p0 - 1) * p1;
        SP_TRY(c.alloc(&u, ne));
        SP_TRY(c.alloc(&v, ne));
        SP_TRY(c.alloc(&w, ne));
        k_gen_grid<<<gridN(n, c.device), 256, 0, c.stream>>>(p0, p1, wsk, u, v, w);
        undirected = 1;
    } else {
        int64_t cand;
        uint64_t *key;
        if (kind == SP_GEN_RMAT) {
            SP_CHECK(p0 >= 1 && p0 <= 30 && p1 >= 1, SP_ERR_ARG, "bad RMAT scale/edge factor");
            n = (int64_t)1 << p0;
            cand = p1 << p0;
            SP_TRY(c.alloc(&key, cand));
            int ta = 37356, tb = 37356 + 12452, tc = 37356 + 12452 + 12452;
            k_gen_rmat<<<gridN(cand, c.device), 256, 0, c.stream>>>(cand, (int)p0, sk, ta, tb, tc,
                                                                   undirected, key);
        } else if (kind == SP_GEN_UNIFORM) {
            SP_CHECK(p0 >= 1 && p0 < 0x7fffffffll && p1 >= 0, SP_ERR_ARG, "bad uniform size");
            n = p0;
            cand = p1;
            SP_TRY(c.alloc(&key, cand));
            k_gen_uniform<<<gridN(cand, c.device), 256, 0, c.stream>>>(cand, (uint64_t)n, sk,
                                                                      undirected, key);
        } else {
            SP_CHECK(false, SP_ERR_ARG, "unknown generator kind %d", kind);
        }
        uint64_t *uk;
        SP_TRY(unique_keys(c, key, cand, &uk, &ne));
        SP_TRY(c.alloc(&u, ne));
        SP_TRY(c.alloc(&v, ne));
        SP_TRY(c.alloc(&w, ne));
        if (ne) k_keys_to_edges<<<gridN(ne, c.device), 256, 0, c.stream>>>(uk, ne, wsk, u, v, w);
    }
    SP_CUDA(cudaGetLastError());
    sp_graph *g;
    SP_TRY(new_graph(!undirected, device, &g));
    int rc = build_from_device_edges(g, c, u, v, w, ne, n);
    if (rc == SP_OK) rc = c.finish(nullptr);
    if (rc != SP_OK) {
        free_graph(g);
        return rc;
    }
    *out = g;
    return SP_OK;
}

int sp_graph_info(const sp_graph *g, int64_t *n, int64_t *m, int *directed) {
    SP_CHECK(g, SP_ERR_ARG, "null graph");
    if (n) *n = g->n;
    if (m) *m = g->m;
    if (directed) *directed = g->directed;
    return SP_OK;
}

int sp_graph_download(const sp_graph *cg, int which, void *dst) {
    SP_CHECK(cg && dst, SP_ERR_ARG, "sp_graph_download: bad arguments");
    sp_graph *g = const_cast<sp_graph *>(cg);
    SP_CUDA(cudaSetDevice(g->device));
    const void *src = nullptr;
    size_t bytes = 0;
    switch (which) {
        case SP_ARR_OFFSETS: src = g->off; bytes = (g->n + 1) * 8; break;
        case SP_ARR_ADJ: src = g->adj; bytes = g->m * 4; break;
        case SP_ARR_WEIGHTS: src = g->w; bytes = g->m * 4; break;
        case SP_ARR_REV_OFFSETS: src = g->roff; bytes = (g->n + 1) * 8; break;
        case SP_ARR_REV_ADJ: src = g->radj; bytes = g->m * 4; break;
        case SP_ARR_WEFF: {
            Call c;
            SP_TRY(c.begin(g->device));
            SP_TRY(ensure_weff(g, c));
            SP_TRY(c.finish(nullptr));
            src = g->weff;
            bytes = g->m * 4;
            break;
        }
        case SP_ARR_REV_EID: {
            std::lock_guard<std::mutex> lk(g_lazy_mu);
            if (!g->reid && g->m) {
                Call c;
                SP_TRY(c.begin(g->device));
                SP_TRY(build_reverse(g, c, false, true));
                SP_TRY(c.finish(nullptr));
            }
            src = g->reid;
            bytes = g->m * 8;
            break;
        }
        default: SP_CHECK(false, SP_ERR_ARG, "unknown array id %d", which);
    }
    if (bytes) SP_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    return SP_OK;
}

int sp_graph_weight_range(const sp_graph *g, int32_t *wmin, int32_t *wmax) {
    SP_CHECK(g, SP_ERR_ARG, "null graph");
    SP_CHECK(g->m > 0, SP_ERR_ARG, "weight range of a graph with no edges");
    SP_CUDA(cudaSetDevice(g->device));
    if (wmin) *wmin = g->wmin_h;  // read at creation (the graph is immutable)
    if (wmax) *wmax = g->wmax_h;
    return SP_OK;
}

void sp_graph_destroy(sp_graph *g) { free_graph(g); }

}  // extern "C"
