/*
 * cpu_ref.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference interpreter (trident.interp.run,
 * /root/reference/pkg/src/trident/interp.py) executing the four corpus
 * programs, plus the CSR builder of trident/graph.py.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library; the product (paper_2305_03317_b200/) never does.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every function below
 * bit-for-bit against golden vectors produced by the Python reference
 * itself (tests/golden/make_golden.py): 14 corpus fixtures x {directed,
 * undirected} x {SSSP, PR, BC, TC, CSR arrays} plus seeded RMAT / uniform /
 * grid graphs.
 *
 * Floating point: compile with -O2 -ffp-contract=off (no FMA contraction),
 * so every double op rounds exactly like CPython's float arithmetic.
 *
 * Each entry point optionally uses OpenMP (nthreads > 1) in a way that keeps
 * the result bit-identical: per-vertex folds stay sequential, maxima and
 * integer sums are order-independent.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define CR_INT_MAX 2147483647LL
#define CR_INT_MIN (-2147483648LL)

/* ------------------------------------------------------------------------
 * Graph construction: trident/graph.py:101-116 (from_edges) and 68-98
 * (_build_csr).
 * ---------------------------------------------------------------------- */

/* Number of stored slots: one per edge, plus the mirror for undirected
 * non-loop edges (graph.py:112-113; self-loops stored once). */
int64_t cr_count_slots(int64_t ne, const int32_t *u, const int32_t *v,
                       int directed)
{
    int64_t s = ne;
    if (!directed)
        for (int64_t i = 0; i < ne; i++)
            s += (u[i] != v[i]);
    return s;
}

/* Stable counting sort of idx[0..m) by key[idx[i]] into out (keys in [0,n)). */
static void stable_count_sort(int64_t n, int64_t m, const int32_t *key,
                              const int64_t *idx, int64_t *out, int64_t *cnt)
{
    memset(cnt, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t i = 0; i < m; i++)
        cnt[key[idx[i]] + 1]++;
    for (int64_t k = 0; k < n; k++)
        cnt[k + 1] += cnt[k];
    for (int64_t i = 0; i < m; i++)
        out[cnt[key[idx[i]]]++] = idx[i];
}

/*
 * Build forward + reverse CSR.  Slot order = graph.py:107-113 append order;
 * forward = stable sort by (src, dst) (graph.py:70-81, sort key dst is
 * stable within the src bucket); reverse = (dst, src, eid) (graph.py:84-96).
 * Output arrays are caller-allocated with m = cr_count_slots(...) entries.
 */
int cr_build_csr(int64_t n, int64_t ne, const int32_t *u, const int32_t *v,
                 const int32_t *w, int directed, int64_t *off, int32_t *adj,
                 int32_t *wt, int64_t *roff, int32_t *radj, int64_t *reid)
{
    int64_t m = cr_count_slots(ne, u, v, directed);
    int32_t *ss = malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
    int32_t *sd = malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
    int32_t *sw = malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
    int64_t *a = calloc((size_t)(m ? m : 1), sizeof(int64_t));
    int64_t *b = malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
    int64_t *cnt = malloc(sizeof(int64_t) * (size_t)(n + 1));
    if (!ss || !sd || !sw || !a || !b || !cnt) {
        free(ss); free(sd); free(sw); free(a); free(b); free(cnt);
        return -1;
    }
    int64_t k = 0;
    for (int64_t i = 0; i < ne; i++) {
        ss[k] = u[i]; sd[k] = v[i]; sw[k] = w[i]; k++;
        if (!directed && u[i] != v[i]) {
            ss[k] = v[i]; sd[k] = u[i]; sw[k] = w[i]; k++;
        }
    }
    for (int64_t i = 0; i < m; i++)
        a[i] = i;
    /* LSD: stable by dst, then stable by src == stable by (src, dst). */
    stable_count_sort(n, m, sd, a, b, cnt);
    stable_count_sort(n, m, ss, b, a, cnt);
    memset(off, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t e = 0; e < m; e++) {
        adj[e] = sd[a[e]];
        wt[e] = sw[a[e]];
        off[ss[a[e]] + 1]++;
    }
    for (int64_t x = 0; x < n; x++)
        off[x + 1] += off[x];
    /* Reverse: forward slots are already in (src, eid) order; a stable sort
     * by dst yields (dst, src, eid) -- graph.py:92. */
    for (int64_t e = 0; e < m; e++)
        b[e] = e;
    stable_count_sort(n, m, adj, b, reid, cnt);
    memset(roff, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t x = 0; x < n; x++)
        for (int64_t e = off[x]; e < off[x + 1]; e++)
            roff[adj[e] + 1]++;
    for (int64_t x = 0; x < n; x++)
        roff[x + 1] += roff[x];
    for (int64_t kk = 0; kk < m; kk++) {
        /* src of forward slot reid[kk]: binary search in off */
        int64_t e = reid[kk], lo = 0, hi = n - 1;
        while (lo < hi) {
            int64_t mid = (lo + hi + 1) / 2;
            if (off[mid] <= e) lo = mid; else hi = mid - 1;
        }
        radj[kk] = (int32_t)lo;
    }
    free(ss); free(sd); free(sw); free(a); free(b); free(cnt);
    return 0;
}

/* Effective SSSP weight: get_edge(v, nbr) resolves to the FIRST slot v->nbr
 * (graph.py:56-62 bisect_left; interp.py:545-551), so every slot of a run of
 * equal destinations relaxes with the weight of the run's first slot. */
void cr_weff(int64_t n, const int64_t *off, const int32_t *adj,
             const int32_t *w, int32_t *weff)
{
    for (int64_t x = 0; x < n; x++)
        for (int64_t e = off[x]; e < off[x + 1]; e++)
            weff[e] = (e > off[x] && adj[e] == adj[e - 1]) ? weff[e - 1] : w[e];
}

/* ------------------------------------------------------------------------
 * SSSP: corpus/programs/sssp.sp:1-20 under interp.py semantics.
 * Vertices ascending (interp.py:217-218), neighbours in CSR order
 * (390-394), strict-< Min with companion (197-209, 575-576), in-place
 * (Gauss-Seidel) dist reads, staged modified/modified_nxt, convergence
 * = !any(modified) after the body (401-421), cap -> NonConvergence.
 * Returns 0 ok, 1 cap reached, 2 int32 underflow of a distance.
 * ---------------------------------------------------------------------- */
int cr_sssp(int64_t n, const int64_t *off, const int32_t *adj,
            const int32_t *weff, int32_t src, int64_t cap, int32_t *dist,
            int64_t *iters_out)
{
    uint8_t *mod = calloc((size_t)(n ? n : 1), 1);
    uint8_t *nxt = calloc((size_t)(n ? n : 1), 1);
    for (int64_t x = 0; x < n; x++)
        dist[x] = (int32_t)CR_INT_MAX;
    dist[src] = 0;
    mod[src] = 1;
    int64_t iters = 0;
    int rc = 0;
    for (;;) {
        for (int64_t x = 0; x < n; x++) {
            if (!mod[x])
                continue;
            for (int64_t e = off[x]; e < off[x + 1]; e++) {
                int32_t y = adj[e];
                int64_t cand = (int64_t)dist[x] + (int64_t)weff[e];
                if (cand < (int64_t)dist[y]) {
                    if (cand < CR_INT_MIN) { rc = 2; goto done; }
                    dist[y] = (int32_t)cand;
                    nxt[y] = 1;
                }
            }
        }
        int any = 0;
        for (int64_t x = 0; x < n; x++) {
            mod[x] = nxt[x];
            nxt[x] = 0;
            any |= mod[x];
        }
        iters++;
        if (!any)
            break;
        if (iters >= cap) { rc = 1; break; }
    }
done:
    *iters_out = iters;
    free(mod);
    free(nxt);
    return rc;
}

/* ------------------------------------------------------------------------
 * SSSP distances by Dijkstra: trident/oracles.py:23-40 (oracle_dijkstra,
 * the reference's own independent validator) over the w_eff slot weights
 * sssp.sp relaxes with (get_edge's first-slot weight).  For
 * non-negative weights the shortest distances are the unique relaxation
 * fixpoint, so this equals cr_sssp's dist without its ~10^4 sequential
 * sweeps on a large-diameter graph (cfg5a).  Binary heap of (dist, vertex)
 * with lazy deletion, like heapq.  Returns 0, or 3 for a negative weight.
 * ---------------------------------------------------------------------- */
typedef struct { int64_t d; int32_t v; } cr_hent;

static void heap_push(cr_hent **h, int64_t *len, int64_t *cap, int64_t d, int32_t v)
{
    if (*len == *cap) {
        *cap = *cap ? 2 * *cap : 1024;
        *h = realloc(*h, (size_t)*cap * sizeof(cr_hent));
    }
    int64_t i = (*len)++;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if ((*h)[p].d < d || ((*h)[p].d == d && (*h)[p].v <= v)) break;
        (*h)[i] = (*h)[p];
        i = p;
    }
    (*h)[i].d = d;
    (*h)[i].v = v;
}

static cr_hent heap_pop(cr_hent *h, int64_t *len)
{
    cr_hent top = h[0], last = h[--*len];
    int64_t i = 0;
    for (;;) {
        int64_t c = 2 * i + 1;
        if (c >= *len) break;
        if (c + 1 < *len && (h[c + 1].d < h[c].d || (h[c + 1].d == h[c].d && h[c + 1].v < h[c].v)))
            c++;
        if (last.d < h[c].d || (last.d == h[c].d && last.v <= h[c].v)) break;
        h[i] = h[c];
        i = c;
    }
    if (*len) h[i] = last;
    return top;
}

int cr_sssp_dijkstra(int64_t n, const int64_t *off, const int32_t *adj,
                     const int32_t *weff, int32_t src, int32_t *dist)
{
    for (int64_t e = 0; n && e < off[n]; e++)
        if (weff[e] < 0) return 3;
    uint8_t *done = calloc((size_t)(n ? n : 1), 1);
    cr_hent *h = NULL;
    int64_t len = 0, cap = 0;
    for (int64_t x = 0; x < n; x++)
        dist[x] = (int32_t)CR_INT_MAX;
    dist[src] = 0;
    heap_push(&h, &len, &cap, 0, src);
    while (len) {
        cr_hent t = heap_pop(h, &len);
        if (done[t.v]) continue;
        done[t.v] = 1;
        for (int64_t e = off[t.v]; e < off[t.v + 1]; e++) {
            int32_t y = adj[e];
            int64_t nd = t.d + (int64_t)weff[e];
            if (nd < (int64_t)dist[y]) {  /* candidates >= INT_MAX never win (F12) */
                dist[y] = (int32_t)nd;
                heap_push(&h, &len, &cap, nd, y);
            }
        }
    }
    free(h);
    free(done);
    return 0;
}

/* ------------------------------------------------------------------------
 * PageRank: corpus/programs/pr.sp:1-30.  Per vertex a left fold over the
 * reverse-CSR row (interp.py:395-398) of u.rank / count_outNbrs(u)
 * (interp.py:543-544), newRank = (1-d)/n + d*sum, diff = max |newRank-rank|,
 * Jacobi swap, iter++, stop when diff < eps || iter >= maxIter (checked
 * after the body, interp.py:405-416).  Returns 0 ok, 1 cap reached.
 * rank[] holds the final ranks (== rank_nxt at exit).
 * ---------------------------------------------------------------------- */
int cr_pagerank(int64_t n, const int64_t *off, const int64_t *roff,
                const int32_t *radj, double damping, double eps,
                int64_t max_iter, int64_t cap, double *rank,
                int64_t *iter_out, double *diff_out, int64_t *iters_out,
                int nthreads)
{
    double *nxt = malloc(sizeof(double) * (size_t)(n ? n : 1));
    double nd = (double)n;
    for (int64_t x = 0; x < n; x++)
        rank[x] = 1.0 / nd;
    int64_t iter = 0, iters = 0;
    double diff = 0.0;
    int rc = 0;
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    for (;;) {
        diff = 0.0;
        double dmax = 0.0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(max : dmax) if (nthreads > 1)
        for (int64_t x = 0; x < n; x++) {
            double sum = 0.0;
            for (int64_t k = roff[x]; k < roff[x + 1]; k++) {
                int32_t y = radj[k];
                sum = sum + rank[y] / (double)(off[y + 1] - off[y]);
            }
            double nr = (1.0 - damping) / nd + damping * sum;
            double d = nr - rank[x];
            if (d < 0.0)
                d = 0.0 - d;
            if (d > dmax)
                dmax = d;
            nxt[x] = nr;
        }
        if (dmax > diff)
            diff = dmax;
        memcpy(rank, nxt, sizeof(double) * (size_t)n);
        iter = iter + 1;
        iters++;
        if (diff < eps || iter >= max_iter)
            break;
        if (iters >= cap) { rc = 1; break; }
    }
    *iter_out = iter;
    *diff_out = diff;
    *iters_out = iters;
    free(nxt);
    return rc;
}

/* ------------------------------------------------------------------------
 * Betweenness centrality: corpus/programs/bc.sp:1-22.  Sources in list
 * order (duplicates re-run, interp.py:384-385); BFS levels over forward
 * adjacency (445-461); ascending levels: sigma_v += sigma_w over reverse-CSR
 * parents at level-1 (467-469; for the root that is level -1, i.e. the
 * unreached in-neighbours whose sigma is 0.0); descending levels:
 * delta_v += sigma_v / sigma_w * (1 + delta_w) over CSR children at
 * level+1 (463-465), then bc_v += delta_v / 2 if v != src.
 * sigma/delta hold the LAST source's arrays on exit (zeros if nsrc == 0).
 * ---------------------------------------------------------------------- */
void cr_bc(int64_t n, const int64_t *off, const int32_t *adj,
           const int64_t *roff, const int32_t *radj, const int32_t *srcs,
           int64_t nsrc, double *bc, double *sigma, double *delta,
           int nthreads)
{
    int32_t *level = malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    int32_t *queue = malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    int64_t *lstart = malloc(sizeof(int64_t) * (size_t)(n + 2));
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    for (int64_t x = 0; x < n; x++) {
        bc[x] = 0.0;
        sigma[x] = 0.0;
        delta[x] = 0.0;
    }
    for (int64_t si = 0; si < nsrc; si++) {
        int32_t s = srcs[si];
        for (int64_t x = 0; x < n; x++) {
            sigma[x] = 0.0;
            delta[x] = 0.0;
            level[x] = -1;
        }
        sigma[s] = 1.0;
        level[s] = 0;
        /* BFS; levels as contiguous queue segments (vertex order inside a
         * level is irrelevant: same-level vertices never interact). */
        int64_t head = 0, tail = 0, nlev = 0;
        queue[tail++] = s;
        lstart[0] = 0;
        while (head < tail) {
            int64_t lend = tail;
            nlev++;
            lstart[nlev] = lend;
            for (; head < lend; head++) {
                int32_t x = queue[head];
                for (int64_t e = off[x]; e < off[x + 1]; e++) {
                    int32_t y = adj[e];
                    if (level[y] == -1) {
                        level[y] = level[x] + 1;
                        queue[tail++] = y;
                    }
                }
            }
        }
        for (int64_t L = 0; L < nlev; L++) {
#pragma omp parallel for schedule(dynamic, 256) if (nthreads > 1)
            for (int64_t q = lstart[L]; q < lstart[L + 1]; q++) {
                int32_t x = queue[q];
                double sg = sigma[x];
                for (int64_t k = roff[x]; k < roff[x + 1]; k++) {
                    int32_t y = radj[k];
                    if (level[y] == (int32_t)L - 1)
                        sg = sg + sigma[y];
                }
                sigma[x] = sg;
            }
        }
        for (int64_t L = nlev - 1; L >= 0; L--) {
#pragma omp parallel for schedule(dynamic, 256) if (nthreads > 1)
            for (int64_t q = lstart[L]; q < lstart[L + 1]; q++) {
                int32_t x = queue[q];
                double dl = delta[x];
                for (int64_t e = off[x]; e < off[x + 1]; e++) {
                    int32_t y = adj[e];
                    if (level[y] == (int32_t)L + 1)
                        dl = dl + sigma[x] / sigma[y] * (1.0 + delta[y]);
                }
                delta[x] = dl;
                if (x != s)
                    bc[x] = bc[x] + dl / 2.0;
            }
        }
    }
    free(level);
    free(queue);
    free(lstart);
}

/* ------------------------------------------------------------------------
 * Triangle counting: corpus/programs/tc.sp:1-14 counted with multiplicity
 * (SURVEY F3): sum over v, over slots u<v of N(v), over slots w>v of N(v),
 * of the multiplicity of w in N(u).  Rows are sorted, so for each (v,u) the
 * inner double loop is a multiset intersection of N(v)_{>v} and N(u)_{>v};
 * it walks the shorter side and binary-searches the longer.
 * ---------------------------------------------------------------------- */
static int64_t lower_bound32(const int32_t *a, int64_t lo, int64_t hi, int32_t x)
{
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

static uint64_t mset_dot(const int32_t *adj, int64_t a0, int64_t a1,
                         int64_t b0, int64_t b1)
{
    if (a1 - a0 > b1 - b0) {
        int64_t t0 = a0, t1 = a1;
        a0 = b0; a1 = b1; b0 = t0; b1 = t1;
    }
    uint64_t c = 0;
    int64_t i = a0;
    while (i < a1) {
        int32_t x = adj[i];
        int64_t j = i + 1;
        while (j < a1 && adj[j] == x)
            j++;
        int64_t lb = lower_bound32(adj, b0, b1, x);
        int64_t ub = lb;
        while (ub < b1 && adj[ub] == x)
            ub++;
        c += (uint64_t)(j - i) * (uint64_t)(ub - lb);
        b0 = lb;
        i = j;
    }
    return c;
}

uint64_t cr_tc(int64_t n, const int64_t *off, const int32_t *adj, int nthreads)
{
    uint64_t total = 0;
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : total) if (nthreads > 1)
    for (int64_t x = 0; x < n; x++) {
        int64_t r0 = off[x], r1 = off[x + 1];
        int64_t ahi0 = lower_bound32(adj, r0, r1, (int32_t)x + 1); /* first > x */
        if (ahi0 >= r1)
            continue;
        for (int64_t k = r0; k < r1 && adj[k] < x; k++) {
            int32_t y = adj[k];
            int64_t b0 = lower_bound32(adj, off[y], off[y + 1], (int32_t)x + 1);
            total += mset_dot(adj, ahi0, r1, b0, off[y + 1]);
        }
    }
    return total;
}

int cr_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
