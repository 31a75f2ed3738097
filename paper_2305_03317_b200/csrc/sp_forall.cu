// sp_forall.cu -- generic forall / reduction over neighbour rows.
//
// The shape of corpus/programs/reduction.sp (reduction.sp:5-10) and of any
// program whose outer forall visits every vertex and whose inner forall
// reduces a node property over g.neighbors(v) (or g.nodesTo(v)):
//     forall (v in g.nodes()) forall (u in N(v)) acc_v += prop[u]
// with the per-vertex results and their total.  Integer sums are exact in
// any order, so the reduction needs no ordering (interp.py:347-359,
// 561-572).  The kernel is a template over the value type and the
// per-slot term, so other corpus-shaped reductions reuse it.
//
// Layout: one warp per row with lanes striding its slots (rows of any
// length), warp sum, lane 0 writes the row result; the total is a block
// reduction + one atomic per block.
#include <algorithm>

#include "sp_common.cuh"

using namespace sp;

namespace {

// term(u) for a slot pointing at u
struct PropTerm {
    const int64_t *prop;  // null: every vertex's property is 1 (attachNodeProperty(prop = 1))
    __device__ __forceinline__ int64_t operator()(int32_t u) const { return prop ? prop[u] : 1; }
};

template <class T, class Term>
__global__ void __launch_bounds__(256) k_neighbor_reduce(const int64_t *__restrict__ rowoff,
                                                         const int32_t *__restrict__ col,
                                                         int64_t n, Term term, T *per_vertex,
                                                         unsigned long long *total) {
    __shared__ T red[8];
    const unsigned lane = lane_id();
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    T acc_total = 0;
    for (int64_t v = warp; v < n; v += nwarps) {
        const int64_t r0 = rowoff[v], r1 = rowoff[v + 1];
        T s = 0;
        for (int64_t k = r0 + lane; k < r1; k += 32) s += term(__ldcs(col + k));
        s = warp_sum(s);
        if (lane == 0) {
            if (per_vertex) per_vertex[v] = s;
            acc_total += s;
        }
    }
    __syncwarp();
    if (lane == 0) red[threadIdx.x >> 5] = acc_total;
    __syncthreads();
    if (threadIdx.x == 0) {
        T t = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) t += red[i];
        if (t) atomicAdd(total, (unsigned long long)t);  // two's complement: exact
    }
}

}  // namespace

extern "C" int sp_neighbor_sum(sp_graph *g, const int64_t *prop, int mem, int reverse,
                               int64_t *per_vertex, int64_t *total, sp_stats *st) {
    SP_CHECK(g && total, SP_ERR_ARG, "sp_neighbor_sum: bad arguments");
    Call c;
    SP_TRY(c.begin(g->device));
    const int64_t n = g->n;
    const int64_t *dprop = nullptr;
    if (prop) {
        int64_t *p;
        SP_TRY(c.alloc(&p, std::max<int64_t>(1, n)));
        SP_TRY(to_device(p, prop, n * sizeof(int64_t), mem, c.stream));
        dprop = p;
    }
    int64_t *pv = nullptr;
    if (per_vertex) SP_TRY(c.alloc(&pv, std::max<int64_t>(1, n)));
    unsigned long long *tot;
    SP_TRY(c.alloc(&tot, 1));
    SP_CUDA(cudaMemsetAsync(tot, 0, sizeof(unsigned long long), c.stream));
    if (n) {
        const int64_t *rowoff = reverse ? g->roff : g->off;
        const int32_t *col = reverse ? g->radj : g->adj;
        k_neighbor_reduce<int64_t, PropTerm><<<grid_for(n * 32, 256, c.device, 8), 256, 0,
                                               c.stream>>>(rowoff, col, n, PropTerm{dprop}, pv,
                                                           tot);
        c.launches++;
        SP_CUDA(cudaGetLastError());
    }
    int64_t *h;
    SP_TRY(c.host_as(&h));
    SP_CUDA(cudaMemcpyAsync(h, tot, 8, cudaMemcpyDeviceToHost, c.stream));
    if (per_vertex && n) SP_TRY(from_device(per_vertex, pv, n * 8, mem, c.stream));
    SP_TRY(c.finish(st));
    *total = h[0];
    if (st) {
        st->iterations = 1;
        st->edges_visited = g->m;
        st->vertices_visited = n;
        st->main_kernel_ms = st->device_ms;
        st->main_kernel_launches = c.launches;
        st->model_bytes = 8 * (n + 1) + 4 * g->m + (prop ? 8 * g->m : 0);
    }
    return SP_OK;
}
