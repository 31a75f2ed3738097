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
#include <cstring>

#include "sp_common.cuh"

using namespace sp;

namespace {

// term(u) for a slot pointing at u
struct PropTerm {
    const int64_t *prop;  // null: every slot's term is `c` (a constant property / literal)
    int64_t c;
    __device__ __forceinline__ int64_t operator()(int32_t u) const { return prop ? prop[u] : c; }
};
struct ConstTerm {
    double c;
    __device__ __forceinline__ double operator()(int32_t) const { return c; }
};

// Reduction operators (exact in any order: integer sums, min, max).
struct OpSum {
    template <class T> __device__ __forceinline__ static T id() { return T(0); }
    template <class T> __device__ __forceinline__ static T f(T a, T b) { return a + b; }
};
struct OpMin {
    template <class T> __device__ __forceinline__ static T id() { return T(INFINITY); }
    template <class T> __device__ __forceinline__ static T f(T a, T b) { return fmin(a, b); }
};
struct OpMax {
    template <class T> __device__ __forceinline__ static T id() { return T(-INFINITY); }
    template <class T> __device__ __forceinline__ static T f(T a, T b) { return fmax(a, b); }
};

template <class Op, class T>
__device__ __forceinline__ T warp_reduce(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = Op::f(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ void total_combine(OpSum, int64_t *tot, int64_t t) {
    if (t) atomicAdd(reinterpret_cast<unsigned long long *>(tot), (unsigned long long)t);
}
__device__ __forceinline__ void total_combine(OpMin, double *tot, double t) {
    // doubles in [-inf, inf]: order-preserving integer image of the bits
    const long long b = __double_as_longlong(t);
    atomicMin(reinterpret_cast<long long *>(tot), b >= 0 ? b : b ^ 0x7fffffffffffffffll);
}
__device__ __forceinline__ void total_combine(OpMax, double *tot, double t) {
    const long long b = __double_as_longlong(t);
    atomicMax(reinterpret_cast<long long *>(tot), b >= 0 ? b : b ^ 0x7fffffffffffffffll);
}

// forall v: forall u in row(v): acc_v = Op(acc_v, term(u)); per_vertex[v]
// = the row's reduction (Op's identity for an empty row), *total = Op over
// all rows.  One warp per row, lanes striding its slots.
template <class Op, class T, class Term>
__global__ void __launch_bounds__(256) k_neighbor_reduce(const int64_t *__restrict__ rowoff,
                                                         const int32_t *__restrict__ col,
                                                         int64_t n, Term term, T *per_vertex,
                                                         T *total) {
    __shared__ T red[8];
    const unsigned lane = lane_id();
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    T acc_total = Op::template id<T>();
    for (int64_t v = warp; v < n; v += nwarps) {
        const int64_t r0 = rowoff[v], r1 = rowoff[v + 1];
        T s = Op::template id<T>();
        for (int64_t k = r0 + lane; k < r1; k += 32) s = Op::f(s, term(__ldcs(col + k)));
        s = warp_reduce<Op>(s);
        if (lane == 0) {
            if (per_vertex) per_vertex[v] = s;
            acc_total = Op::f(acc_total, s);
        }
    }
    __syncwarp();
    if (lane == 0) red[threadIdx.x >> 5] = acc_total;
    __syncthreads();
    if (threadIdx.x == 0) {
        T t = Op::template id<T>();
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) t = Op::f(t, red[i]);
        total_combine(Op{}, total, t);
    }
}

__global__ void k_total_init_f64(double *tot, int op) {
    const double v = op == 1 ? INFINITY : -INFINITY;
    const long long b = __double_as_longlong(v);
    *reinterpret_cast<long long *>(tot) = b >= 0 ? b : b ^ 0x7fffffffffffffffll;
}
__global__ void k_total_fini_f64(double *tot) {
    const long long b = *reinterpret_cast<long long *>(tot);
    *tot = __longlong_as_double(b >= 0 ? b : b ^ 0x7fffffffffffffffll);
}

}  // namespace

extern "C" int sp_neighbor_sum(sp_graph *g, const int64_t *prop, int mem, int reverse,
                               int64_t *per_vertex, int64_t *total, sp_stats *st) {
    return sp_neighbor_reduce(g, SP_REDUCE_SUM_I64, reverse, 1, 0.0, prop, mem, per_vertex, total,
                              st);
}

extern "C" int sp_neighbor_reduce(sp_graph *g, int op, int reverse, int64_t iterm, double dterm,
                                  const int64_t *prop, int mem, void *per_vertex, void *total,
                                  sp_stats *st) {
    SP_CHECK(g && total && op >= SP_REDUCE_SUM_I64 && op <= SP_REDUCE_MAX_F64 &&
                 (prop == nullptr || op == SP_REDUCE_SUM_I64),
             SP_ERR_ARG, "sp_neighbor_reduce: bad arguments");
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
    void *pv = nullptr;
    if (per_vertex) SP_TRY(c.alloc(reinterpret_cast<int64_t **>(&pv), std::max<int64_t>(1, n)));
    int64_t *tot;
    SP_TRY(c.alloc(&tot, 1));
    const int64_t *rowoff = reverse ? g->roff : g->off;
    const int32_t *col = reverse ? g->radj : g->adj;
    const int grid = grid_for(n * 32, 256, c.device, 8);
    if (op == SP_REDUCE_SUM_I64) {
        SP_CUDA(cudaMemsetAsync(tot, 0, 8, c.stream));
        if (n)
            k_neighbor_reduce<OpSum, int64_t, PropTerm><<<grid, 256, 0, c.stream>>>(
                rowoff, col, n, PropTerm{dprop, iterm}, static_cast<int64_t *>(pv), tot);
    } else {
        double *dt = reinterpret_cast<double *>(tot);
        k_total_init_f64<<<1, 1, 0, c.stream>>>(dt, op);
        if (n && op == SP_REDUCE_MIN_F64)
            k_neighbor_reduce<OpMin, double, ConstTerm><<<grid, 256, 0, c.stream>>>(
                rowoff, col, n, ConstTerm{dterm}, static_cast<double *>(pv), dt);
        else if (n)
            k_neighbor_reduce<OpMax, double, ConstTerm><<<grid, 256, 0, c.stream>>>(
                rowoff, col, n, ConstTerm{dterm}, static_cast<double *>(pv), dt);
        k_total_fini_f64<<<1, 1, 0, c.stream>>>(dt);
        c.launches += 2;
    }
    c.launches += n ? 1 : 0;
    SP_CUDA(cudaGetLastError());
    int64_t *h;
    SP_TRY(c.host_as(&h));
    SP_CUDA(cudaMemcpyAsync(h, tot, 8, cudaMemcpyDeviceToHost, c.stream));
    if (per_vertex && n) SP_TRY(from_device(per_vertex, pv, n * 8, mem, c.stream));
    SP_TRY(c.finish(st));
    memcpy(total, h, 8);
    if (st) {
        st->iterations = 1;
        st->edges_visited = g->m;
        st->vertices_visited = n;
        st->main_kernel_ms = st->device_ms;
        st->main_kernel_launches = c.launches;
        st->model_bytes = 8 * (n + 1) + 4 * g->m + (prop ? 8 * g->m : 0) + (per_vertex ? 8 * n : 0);
    }
    return SP_OK;
}
