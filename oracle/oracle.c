/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * A plain-C restatement of the reference CPU path, function by function:
 *   build_graph           /root/reference/proj/src/graph.cpp:93-172
 *   orient_edges          /root/reference/proj/src/graph.cpp:180-193
 *   three_graphlets_hash  /root/reference/proj/src/kernels.cpp:27-50   (Alg. 1)
 *   three_graphlets_bsearch kernels.cpp:52-65                          (Alg. 2)
 *   derive_s_v            kernels.cpp:67-83
 *   clique_res / cycle_res kernels.cpp:85-113                          (Algs. 3-4)
 *   clique_hash           kernels.cpp:115-127                          (Alg. 5)
 *   cycle_hash            kernels.cpp:129-141                          (Alg. 6)
 *   process_edge_hash     kernels.cpp:143-156
 *   accumulate_unrestricted counts.cpp:6-27
 *   merge                 counts.cpp:29-45
 *   global_from_unrestricted counts.cpp:86-111
 *   micro_counts          counts.cpp:122-136
 *   classify_three/four, brute_force_global  oracle.cpp:8-66
 * The edge-centric hash pipeline is what the reference runs per edge; it is
 * deliberately kept as is (no algorithmic shortcuts) so the checker stays an
 * independent implementation of the reference semantics.
 */
#include "oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- sorting */

static void radix_sort_u64(uint64_t *a, uint64_t n) {
    if (n < 2) return;
    uint64_t *tmp = (uint64_t *)malloc(n * sizeof(uint64_t));
    uint64_t *src = a, *dst = tmp;
    for (int pass = 0; pass < 8; ++pass) {
        uint64_t cnt[256] = {0};
        int shift = pass * 8;
        for (uint64_t i = 0; i < n; ++i) cnt[(src[i] >> shift) & 0xff]++;
        if (cnt[(src[0] >> shift) & 0xff] == n) continue; /* digit constant */
        uint64_t sum = 0;
        for (int d = 0; d < 256; ++d) { uint64_t c = cnt[d]; cnt[d] = sum; sum += c; }
        for (uint64_t i = 0; i < n; ++i) dst[cnt[(src[i] >> shift) & 0xff]++] = src[i];
        uint64_t *t = src; src = dst; dst = t;
    }
    if (src != a) memcpy(a, src, n * sizeof(uint64_t));
    free(tmp);
}

static uint64_t unique_u64(uint64_t *a, uint64_t n) {
    if (n == 0) return 0;
    uint64_t w = 1;
    for (uint64_t i = 1; i < n; ++i)
        if (a[i] != a[w - 1]) a[w++] = a[i];
    return w;
}

static uint32_t lower_bound_u64(const uint64_t *a, uint64_t n, uint64_t x) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return (uint32_t)lo;
}

/* ------------------------------------------------------------ build_graph */

static const uint32_t *g_sort_deg; /* comparator context (build is single-threaded) */
static int cmp_deg_desc(const void *pa, const void *pb) {
    uint32_t a = *(const uint32_t *)pa, b = *(const uint32_t *)pb;
    if (g_sort_deg[a] != g_sort_deg[b]) return g_sort_deg[a] > g_sort_deg[b] ? -1 : 1;
    return a < b ? -1 : (a > b);
}

/* graph.cpp:93-172: label universe incl. self-loop endpoints, loop removal,
 * undirected dedup, relabel by (degree asc, label asc), id-sorted rows plus
 * a degree-descending iteration view. */
int or_build_graph(const uint64_t *ea, const uint64_t *eb, uint64_t count, or_graph *g) {
    memset(g, 0, sizeof(*g));
    uint64_t *labels = (uint64_t *)malloc((2 * count + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < count; ++i) { labels[2 * i] = ea[i]; labels[2 * i + 1] = eb[i]; }
    radix_sort_u64(labels, 2 * count);
    uint64_t n = unique_u64(labels, 2 * count);
    if (n >= 0xffffffffull) { free(labels); return -1; }

    uint64_t *keys = (uint64_t *)malloc((count + 1) * sizeof(uint64_t));
    uint64_t k = 0;
    for (uint64_t i = 0; i < count; ++i) {
        if (ea[i] == eb[i]) continue;
        uint64_t x = lower_bound_u64(labels, n, ea[i]);
        uint64_t y = lower_bound_u64(labels, n, eb[i]);
        if (x > y) { uint64_t t = x; x = y; y = t; }
        keys[k++] = (x << 32) | y;
    }
    radix_sort_u64(keys, k);
    uint64_t m = unique_u64(keys, k);

    uint32_t *deg = (uint32_t *)calloc(n + 1, sizeof(uint32_t));
    for (uint64_t i = 0; i < m; ++i) { deg[keys[i] >> 32]++; deg[keys[i] & 0xffffffffu]++; }

    /* relabel: ascending degree, ties by ascending original label (== compact id) */
    uint64_t *ord = (uint64_t *)malloc((n + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) ord[i] = ((uint64_t)deg[i] << 32) | i;
    radix_sort_u64(ord, n);
    uint32_t *new_id = (uint32_t *)malloc((n + 1) * sizeof(uint32_t));
    g->degree = (uint32_t *)malloc((n + 1) * sizeof(uint32_t));
    g->inverse_map = (uint64_t *)malloc((n + 1) * sizeof(uint64_t));
    for (uint64_t r = 0; r < n; ++r) {
        uint32_t old = (uint32_t)(ord[r] & 0xffffffffu);
        new_id[old] = (uint32_t)r;
        g->degree[r] = deg[old];
        g->inverse_map[r] = labels[old];
    }
    g->n = n;
    g->m = m;
    g->dmax = 0;
    for (uint64_t v = 0; v < n; ++v) if (g->degree[v] > g->dmax) g->dmax = g->degree[v];

    g->offsets = (uint64_t *)malloc((n + 1) * sizeof(uint64_t));
    g->offsets[0] = 0;
    for (uint64_t v = 0; v < n; ++v) g->offsets[v + 1] = g->offsets[v] + g->degree[v];

    /* directed pairs sorted by (src, dst) give id-sorted rows directly */
    uint64_t *dir = (uint64_t *)malloc((2 * m + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < m; ++i) {
        uint64_t a = new_id[keys[i] >> 32], b = new_id[keys[i] & 0xffffffffu];
        dir[2 * i] = (a << 32) | b;
        dir[2 * i + 1] = (b << 32) | a;
    }
    radix_sort_u64(dir, 2 * m);
    g->adj_id = (uint32_t *)malloc((2 * m + 1) * sizeof(uint32_t));
    g->adj_deg = (uint32_t *)malloc((2 * m + 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < 2 * m; ++i) g->adj_id[i] = (uint32_t)(dir[i] & 0xffffffffu);
    memcpy(g->adj_deg, g->adj_id, 2 * m * sizeof(uint32_t));
    g_sort_deg = g->degree;
    for (uint64_t v = 0; v < n; ++v)
        qsort(g->adj_deg + g->offsets[v], g->degree[v], sizeof(uint32_t), cmp_deg_desc);

    free(dir); free(new_id); free(ord); free(deg); free(keys); free(labels);
    return 0;
}

void or_free_graph(or_graph *g) {
    free(g->offsets); free(g->adj_id); free(g->adj_deg); free(g->degree); free(g->inverse_map);
    memset(g, 0, sizeof(*g));
}

/* graph.cpp:180-193: ascending (v,u) with u < v. */
void or_orient_edges(const or_graph *g, uint32_t *v_out, uint32_t *u_out) {
    uint64_t k = 0;
    for (uint64_t v = 0; v < g->n; ++v)
        for (uint64_t j = g->offsets[v]; j < g->offsets[v + 1]; ++j) {
            uint32_t u = g->adj_id[j];
            if (u >= v) break;
            v_out[k] = (uint32_t)v; u_out[k] = u; ++k;
        }
}

static int has_edge(const or_graph *g, uint32_t a, uint32_t b) {
    if (g->degree[a] > g->degree[b]) { uint32_t t = a; a = b; b = t; }
    const uint32_t *row = g->adj_id + g->offsets[a];
    uint64_t lo = 0, hi = g->degree[a];
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (row[mid] < b) lo = mid + 1; else if (row[mid] > b) hi = mid; else return 1;
    }
    return 0;
}

/* -------------------------------------------------- per-edge hash pipeline */

typedef struct {
    uint64_t *psi;             /* StampTable: n marks (kernels.hpp:14-23) */
    uint32_t *tri, *su, *sv;   /* NeighborhoodSets (kernels.hpp:28-46) */
} scratch_t;

static void scratch_init(scratch_t *s, const or_graph *g) {
    s->psi = (uint64_t *)calloc(g->n + 1, sizeof(uint64_t));
    s->tri = (uint32_t *)malloc((g->dmax + 1) * sizeof(uint32_t));
    s->su = (uint32_t *)malloc((g->dmax + 1) * sizeof(uint32_t));
    s->sv = (uint32_t *)malloc((g->dmax + 1) * sizeof(uint32_t));
}
static void scratch_free(scratch_t *s) { free(s->psi); free(s->tri); free(s->su); free(s->sv); }

/* rec = {t, s_u, s_v, x7, x10}; process_edge_hash (kernels.cpp:143-156). */
static void process_edge_hash(const or_graph *g, scratch_t *s, uint32_t v, uint32_t u,
                              uint64_t k, uint64_t rec[5]) {
    const uint64_t l1 = 3 * k + 1, l2 = 3 * k + 2, l3 = 3 * k + 3;
    uint64_t *psi = s->psi;
    /* Alg. 1 (kernels.cpp:27-50) */
    const uint32_t *nv = g->adj_deg + g->offsets[v];
    uint32_t dv = g->degree[v];
    for (uint32_t i = 0; i < dv; ++i) if (nv[i] != u) psi[nv[i]] = l1;
    const uint32_t *nu = g->adj_deg + g->offsets[u];
    uint32_t du = g->degree[u];
    uint32_t nt = 0, nsu = 0, nsv = 0;
    for (uint32_t i = 0; i < du; ++i) {
        uint32_t w = nu[i];
        if (w == v) continue;
        if (psi[w] == l1) { psi[w] = l3; s->tri[nt++] = w; }
        else { psi[w] = l2; s->su[nsu++] = w; }
    }
    /* derive_s_v (kernels.cpp:67-83): merge N(v) against T in degree order */
    uint32_t ti = 0;
    for (uint32_t i = 0; i < dv; ++i) {
        uint32_t w = nv[i];
        if (w == u) continue;
        if (ti < nt && s->tri[ti] == w) { ++ti; continue; }
        s->sv[nsv++] = w;
    }
    /* Alg. 5 clique_hash (kernels.cpp:115-127) */
    uint64_t cliques = 0;
    for (uint32_t i = 0; i < nt; ++i) {
        uint32_t w = s->tri[i];
        const uint32_t *nw = g->adj_deg + g->offsets[w];
        for (uint32_t j = 0; j < g->degree[w]; ++j) if (psi[nw[j]] == l3) ++cliques;
        psi[w] = 0;
    }
    /* Alg. 6 cycle_hash (kernels.cpp:129-141): S_v members still carry l1 */
    uint64_t cycles = 0;
    for (uint32_t i = 0; i < nsu; ++i) {
        uint32_t w = s->su[i];
        const uint32_t *nw = g->adj_deg + g->offsets[w];
        for (uint32_t j = 0; j < g->degree[w]; ++j) if (psi[nw[j]] == l1) ++cycles;
        psi[w] = 0;
    }
    rec[0] = nt; rec[1] = nsu; rec[2] = nsv; rec[3] = cliques; rec[4] = cycles;
}

/* Algs. 2-4, binary-search pipeline (kernels.cpp:52-65, 85-113, 158-171). */
void or_process_edge_bsearch(const or_graph *g, uint32_t v, uint32_t u, uint64_t rec[5]) {
    uint32_t *tri = (uint32_t *)malloc((g->dmax + 1) * sizeof(uint32_t));
    uint32_t *su = (uint32_t *)malloc((g->dmax + 1) * sizeof(uint32_t));
    uint32_t *sv = (uint32_t *)malloc((g->dmax + 1) * sizeof(uint32_t));
    uint32_t nt = 0, nsu = 0, nsv = 0;
    const uint32_t *nu = g->adj_deg + g->offsets[u];
    for (uint32_t i = 0; i < g->degree[u]; ++i) {
        uint32_t w = nu[i];
        if (w == v) continue;
        if (has_edge(g, w, v)) tri[nt++] = w; else su[nsu++] = w;
    }
    const uint32_t *nv = g->adj_deg + g->offsets[v];
    uint32_t ti = 0;
    for (uint32_t i = 0; i < g->degree[v]; ++i) {
        uint32_t w = nv[i];
        if (w == u) continue;
        if (ti < nt && tri[ti] == w) { ++ti; continue; }
        sv[nsv++] = w;
    }
    uint64_t x7 = 0, x10 = 0;
    for (uint32_t i = 0; i < nt; ++i)
        for (uint32_t j = i + 1; j < nt; ++j) x7 += has_edge(g, tri[j], tri[i]);
    for (uint32_t i = 0; i < nsu; ++i)
        for (uint32_t j = 0; j < nsv; ++j) x10 += has_edge(g, su[i], sv[j]);
    rec[0] = nt; rec[1] = nsu; rec[2] = nsv; rec[3] = x7; rec[4] = x10;
    free(tri); free(su); free(sv);
}

void or_process_edge_hash_one(const or_graph *g, uint32_t v, uint32_t u, uint64_t eid, uint64_t rec[5]) {
    scratch_t s;
    scratch_init(&s, g);
    process_edge_hash(g, &s, v, u, eid, rec);
    scratch_free(&s);
}

/* Hash pipeline for a list of edge ids, one shared scratch.  out: k x 5. */
void or_edges_hash(const or_graph *g, const uint64_t *ids, uint64_t k, uint64_t *out) {
    uint32_t *ev = (uint32_t *)malloc((g->m + 1) * sizeof(uint32_t));
    uint32_t *eu = (uint32_t *)malloc((g->m + 1) * sizeof(uint32_t));
    or_orient_edges(g, ev, eu);
    scratch_t s;
    scratch_init(&s, g);
    for (uint64_t i = 0; i < k; ++i) process_edge_hash(g, &s, ev[ids[i]], eu[ids[i]], ids[i], out + 5 * i);
    scratch_free(&s);
    free(ev); free(eu);
}

/* ------------------------------------------------------------ count algebra */

typedef struct { u128 c[17]; int overflow; } unres_t;

static void add128(unres_t *a, int i, u128 x) {
    u128 s = a->c[i] + x;
    if (s < a->c[i]) a->overflow = 1;
    a->c[i] = s;
}
static u128 ch2(uint64_t x) { return x < 2 ? 0 : (u128)x * (x - 1) / 2; }
static u128 ch3(uint64_t x) { return x < 3 ? 0 : (u128)x * (x - 1) / 2 * (x - 2) / 3; }
static u128 ch4(uint64_t x) { return x < 4 ? 0 : (u128)x * (x - 1) / 2 * (x - 2) / 3 * (x - 3) / 4; }

/* counts.cpp:6-27 */
static void accumulate(unres_t *acc, const uint64_t rec[5], uint64_t n, uint64_t m) {
    uint64_t t = rec[0], su = rec[1], sv = rec[2];
    uint64_t de = n - (su + sv + t) - 2;
    add128(acc, 3, t);
    add128(acc, 4, su + sv);
    add128(acc, 5, de);
    add128(acc, 7, rec[3]);
    add128(acc, 8, ch2(t));
    add128(acc, 9, (u128)t * (su + sv));
    add128(acc, 10, rec[4]);
    add128(acc, 11, ch2(sv) + ch2(su));
    add128(acc, 12, (u128)sv * su);
    add128(acc, 13, (u128)t * de);
    add128(acc, 14, (u128)(m - (t + su + 1) - (t + sv + 1) + 1));
    add128(acc, 15, (u128)(sv + su) * de);
    add128(acc, 16, ch2(de));
}

static int div_exact(u128 num, unsigned den, u128 *out) {
    if (num % den) return -1;
    *out = num / den;
    return 0;
}
static int sub_exact(u128 a, u128 b, u128 *out) {
    if (a < b) return -1;
    *out = a - b;
    return 0;
}

/* counts.cpp:86-111 */
static int global_from(const u128 *c, uint64_t n, uint64_t m, u128 *X) {
    u128 t;
    memset(X, 0, 18 * sizeof(u128));
    X[1] = m;
    if (sub_exact(ch2(n), m, &X[2])) return -1;
    if (div_exact(c[3], 3, &X[3])) return -1;
    if (div_exact(c[4], 2, &X[4])) return -1;
    X[5] = c[5];
    if (sub_exact(ch3(n), X[3] + X[4] + X[5], &X[6])) return -1;
    if (div_exact(c[7], 6, &X[7])) return -1;
    if (sub_exact(c[8], c[7], &X[8])) return -1;
    if (sub_exact(c[9], 4 * X[8], &t) || div_exact(t, 2, &X[9])) return -1;
    if (div_exact(c[10], 4, &X[10])) return -1;
    if (sub_exact(c[11], X[9], &t) || div_exact(t, 3, &X[11])) return -1;
    if (sub_exact(c[12], c[10], &X[12])) return -1;
    if (sub_exact(c[13], X[9], &t) || div_exact(t, 3, &X[13])) return -1;
    if (sub_exact(c[14], 6 * X[7] + 4 * X[8] + 2 * X[9] + 4 * X[10] + 2 * X[12], &t) ||
        div_exact(t, 2, &X[14])) return -1;
    if (sub_exact(c[15], 2 * X[12], &t) || div_exact(t, 2, &X[15])) return -1;
    if (sub_exact(c[16], 2 * X[14], &X[16])) return -1;
    u128 conn = 0;
    for (int i = 7; i <= 16; ++i) conn += X[i];
    if (sub_exact(ch4(n), conn, &X[17])) return -1;
    return 0;
}

static void store128(uint64_t *dst, const u128 *src, int count) {
    for (int i = 0; i < count; ++i) {
        dst[2 * i] = (uint64_t)src[i];
        dst[2 * i + 1] = (uint64_t)(src[i] >> 64);
    }
}

int or_global_from_unrestricted(const uint64_t C[34], uint64_t n, uint64_t m, uint64_t X[36]) {
    u128 c[17], x[18];
    for (int i = 0; i < 17; ++i) c[i] = ((u128)C[2 * i + 1] << 64) | C[2 * i];
    if (global_from(c, n, m, x)) return -1;
    store128(X, x, 18);
    return 0;
}

/* ------------------------------------------------------------ threaded run */

typedef struct {
    const or_graph *g;
    const uint32_t *ev, *eu;
    const uint64_t *ids; /* optional sample */
    uint64_t total;
    volatile uint64_t *next;
    pthread_mutex_t *mu;
    unres_t acc;
    or_micro *micro;
    uint64_t checksum;
} worker_t;

static void *worker_main(void *arg) {
    worker_t *w = (worker_t *)arg;
    scratch_t s;
    scratch_init(&s, w->g);
    const uint64_t n = w->g->n, m = w->g->m;
    const uint64_t chunk = 64;
    for (;;) {
        uint64_t begin = __atomic_fetch_add(w->next, chunk, __ATOMIC_RELAXED);
        if (begin >= w->total) break;
        uint64_t end = begin + chunk < w->total ? begin + chunk : w->total;
        for (uint64_t i = begin; i < end; ++i) {
            uint64_t k = w->ids ? w->ids[i] : i;
            uint64_t rec[5];
            process_edge_hash(w->g, &s, w->ev[k], w->eu[k], k, rec);
            accumulate(&w->acc, rec, n, m);
            w->checksum += rec[0] + rec[3] + rec[4];
            if (w->micro) {
                /* counts.cpp:113-136 */
                or_micro *r = &w->micro[k];
                uint64_t de = n - (rec[1] + rec[2] + rec[0]) - 2;
                r->edge_id = k; r->x3 = rec[0]; r->x4 = rec[1] + rec[2]; r->x5 = de;
                r->x7 = rec[3]; r->x10 = rec[4]; r->t = rec[0]; r->s_u = rec[1];
                r->s_v = rec[2]; r->d_e = de;
            }
        }
    }
    scratch_free(&s);
    return NULL;
}

static int run_workers(const or_graph *g, int nthreads, const uint64_t *ids, uint64_t total,
                       or_micro *micro, unres_t *out, uint64_t *checksum) {
    if (nthreads < 1) nthreads = 1;
    uint32_t *ev = (uint32_t *)malloc((g->m + 1) * sizeof(uint32_t));
    uint32_t *eu = (uint32_t *)malloc((g->m + 1) * sizeof(uint32_t));
    or_orient_edges(g, ev, eu);
    volatile uint64_t next = 0;
    worker_t *ws = (worker_t *)calloc(nthreads, sizeof(worker_t));
    pthread_t *th = (pthread_t *)calloc(nthreads, sizeof(pthread_t));
    for (int i = 0; i < nthreads; ++i) {
        ws[i].g = g; ws[i].ev = ev; ws[i].eu = eu; ws[i].ids = ids; ws[i].total = total;
        ws[i].next = &next; ws[i].micro = micro;
        pthread_create(&th[i], NULL, worker_main, &ws[i]);
    }
    memset(out, 0, sizeof(*out));
    uint64_t cs = 0;
    for (int i = 0; i < nthreads; ++i) {
        pthread_join(th[i], NULL);
        for (int j = 0; j < 17; ++j) add128(out, j, ws[i].acc.c[j]); /* merge, counts.cpp:29-45 */
        out->overflow |= ws[i].acc.overflow;
        cs += ws[i].checksum;
    }
    if (checksum) *checksum = cs;
    free(ws); free(th); free(ev); free(eu);
    return out->overflow ? -1 : 0;
}

int or_count(const or_graph *g, int nthreads, uint64_t X[36], or_micro *micro) {
    unres_t acc;
    if (run_workers(g, nthreads, NULL, g->m, micro, &acc, NULL)) return -1;
    u128 x[18];
    if (global_from(acc.c, g->n, g->m, x)) return -1;
    store128(X, x, 18);
    return 0;
}

double or_time_sample(const or_graph *g, int nthreads, const uint64_t *edge_ids, uint64_t k,
                      uint64_t *checksum) {
    struct timespec a, b;
    unres_t acc;
    clock_gettime(CLOCK_MONOTONIC, &a);
    run_workers(g, nthreads, edge_ids, k, NULL, &acc, checksum);
    clock_gettime(CLOCK_MONOTONIC, &b);
    return (double)(b.tv_sec - a.tv_sec) + 1e-9 * (double)(b.tv_nsec - a.tv_nsec);
}

/* ------------------------------------------------------------ brute force */

/* oracle.cpp:8-16 */
static int classify_three(const or_graph *g, uint32_t a, uint32_t b, uint32_t c) {
    int e = has_edge(g, a, b) + has_edge(g, a, c) + has_edge(g, b, c);
    return e == 3 ? 3 : e == 2 ? 4 : e == 1 ? 5 : 6;
}

/* oracle.cpp:18-46: (edge count, sorted degree sequence) -> class */
static int classify_four(const or_graph *g, const uint32_t q[4]) {
    int deg[4] = {0, 0, 0, 0}, edges = 0;
    for (int i = 0; i < 4; ++i)
        for (int j = i + 1; j < 4; ++j)
            if (has_edge(g, q[i], q[j])) { ++edges; ++deg[i]; ++deg[j]; }
    for (int i = 1; i < 4; ++i) /* insertion sort */
        for (int j = i; j > 0 && deg[j - 1] > deg[j]; --j) { int t = deg[j]; deg[j] = deg[j - 1]; deg[j - 1] = t; }
    switch (edges) {
    case 0: return 17;
    case 1: return 16;
    case 2: return (deg[0] == 1 && deg[3] == 1) ? 14 : 15;
    case 3:
        if (deg[0] == 0) return 13;
        if (deg[3] == 3) return 11;
        return 12;
    case 4: return deg[0] == 2 ? 10 : 9;
    case 5: return 8;
    default: return 7;
    }
}

int or_brute_force_global(const or_graph *g, uint32_t cap, uint64_t X[36]) {
    if (g->n > cap) return -1;
    uint32_t n = (uint32_t)g->n;
    u128 x[18];
    memset(x, 0, sizeof(x));
    for (uint32_t a = 0; a < n; ++a)
        for (uint32_t b = a + 1; b < n; ++b) {
            x[has_edge(g, a, b) ? 1 : 2] += 1;
            for (uint32_t c = b + 1; c < n; ++c) {
                x[classify_three(g, a, b, c)] += 1;
                for (uint32_t d = c + 1; d < n; ++d) {
                    uint32_t q[4] = {a, b, c, d};
                    x[classify_four(g, q)] += 1;
                }
            }
        }
    store128(X, x, 18);
    return 0;
}

/* ------------------------------------------------------------ generators */
/* Ports of the product's deterministic synthetic generators
 * (paper_1608_05138_b200/csrc/common.cuh mix64/hash2/rmat_edge and
 * csrc/host.cpp make_rmat_params/generate_ba), so that bench.py's reference
 * arm and the fixture scripts build the same graphs WITHOUT loading the
 * product library.  tests/test_oracle.py pins them equal to the product's. */

static uint64_t g_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t g_hash2(uint64_t seed, uint64_t ctr) { return g_mix64(seed ^ g_mix64(ctr)); }
static uint32_t g_threshold(double x) {
    double v = x * 4294967296.0;
    if (v >= 4294967295.0) return 0xffffffffu;
    return (uint32_t)v;
}

typedef struct {
    uint32_t scale, ta, tb, tc;
    uint64_t seed, count;
    uint64_t *out;
    int part, parts;
} rmat_job;

static void *rmat_worker(void *p) {
    rmat_job *j = (rmat_job *)p;
    uint64_t lo = j->count * (uint64_t)j->part / (uint64_t)j->parts;
    uint64_t hi = j->count * (uint64_t)(j->part + 1) / (uint64_t)j->parts;
    for (uint64_t i = lo; i < hi; ++i) {
        uint64_t r = 0, c = 0;
        for (uint32_t l = 0; l < j->scale; ++l) {
            uint32_t x = (uint32_t)(g_hash2(j->seed, i * 64 + l) >> 32);
            r <<= 1;
            c <<= 1;
            if (x < j->ta) {
            } else if (x < j->tb) {
                c |= 1;
            } else if (x < j->tc) {
                r |= 1;
            } else {
                r |= 1;
                c |= 1;
            }
        }
        j->out[2 * i] = r;
        j->out[2 * i + 1] = c;
    }
    return NULL;
}

int or_generate_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c, uint64_t seed,
                     int nthreads, uint64_t *out) {
    if (scale == 0 || scale > 40 || a < 0 || b < 0 || c < 0 || a + b + c > 1.0) return -1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    rmat_job jobs[256];
    uint64_t count = (uint64_t)edge_factor << scale;
    for (int t = 0; t < nthreads; ++t) {
        rmat_job j = {scale, g_threshold(a), g_threshold(a + b), g_threshold(a + b + c), seed, count, out, t, nthreads};
        jobs[t] = j;
        pthread_create(&th[t], NULL, rmat_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    return 0;
}

static uint64_t g_bounded(uint64_t h, uint64_t n) { return (uint64_t)(((u128)h * n) >> 64); }

/* Barabasi-Albert: vertices 0..k form a clique, every later vertex attaches k
 * distinct targets drawn from the endpoint list.  *out is malloc'd (2*count
 * labels), freed with or_free_pairs. */
int or_generate_ba(uint64_t n, uint32_t k, uint64_t seed, uint64_t **out, uint64_t *count) {
    *out = NULL;
    *count = 0;
    if (k == 0) return -1;
    if (n == 0) return 0;
    uint64_t n0 = n < (uint64_t)k + 1 ? n : (uint64_t)k + 1;
    uint64_t cap = n0 * (n0 - 1) / 2 + (n - n0) * (uint64_t)k;
    uint64_t *pairs = (uint64_t *)malloc((2 * cap + 2) * sizeof(uint64_t));
    uint64_t *ends = (uint64_t *)malloc((2 * cap + 2) * sizeof(uint64_t));
    uint64_t *picked = (uint64_t *)malloc((uint64_t)k * sizeof(uint64_t));
    if (!pairs || !ends || !picked) {
        free(pairs);
        free(ends);
        free(picked);
        return -1;
    }
    uint64_t np = 0, ne = 0, ctr = 0;
    for (uint64_t x = 0; x < n0; ++x)
        for (uint64_t y = x + 1; y < n0; ++y) {
            pairs[2 * np] = y;
            pairs[2 * np + 1] = x;
            ++np;
            ends[ne++] = x;
            ends[ne++] = y;
        }
    for (uint64_t v = n0; v < n; ++v) {
        uint32_t np_ = 0;
        while (np_ < k) {
            uint64_t w = ends[g_bounded(g_hash2(seed, ctr++), ne)];
            int dup = 0;
            for (uint32_t q = 0; q < np_; ++q) dup |= picked[q] == w;
            if (!dup) picked[np_++] = w;
        }
        for (uint32_t q = 0; q < k; ++q) {
            pairs[2 * np] = v;
            pairs[2 * np + 1] = picked[q];
            ++np;
            ends[ne++] = v;
            ends[ne++] = picked[q];
        }
    }
    free(ends);
    free(picked);
    *out = pairs;
    *count = np;
    return 0;
}

void or_free_pairs(uint64_t *p) { free(p); }
