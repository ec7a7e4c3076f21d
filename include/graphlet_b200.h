/*
 * graphlet_b200.h -- C-ABI of the B200-native edge-centric k<=4 graphlet
 * counter (arxiv 1608.05138).  Plain pointers and sizes only; no torch or CUDA
 * types cross this boundary (streams are passed as void*).
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/proj/include/graphlet/ headers); see INTEGRATION.md for the
 * binding a maintainer of the reference would add.
 *
 * Error behaviour mirrors the reference's exception classes: every function
 * returns GL_OK (0) or a negative code, and gl_last_error() holds the message
 * (thread-local).  parse errors additionally report the 1-based line number
 * through gl_last_error_line(), like graphlet::parse_error::line().
 */
#ifndef GRAPHLET_B200_H
#define GRAPHLET_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes (reference exception class in parentheses) ---- */
#define GL_OK 0
#define GL_ERR_INVALID -1     /* std::invalid_argument (incl. >= 2^32-1 vertices or edges, graph.cpp:103-104) */
#define GL_ERR_PARSE -2       /* graphlet::parse_error           (graph.hpp:23-33)  */
#define GL_ERR_IO -3          /* std::runtime_error "cannot open" (graph.cpp:87-91) */
#define GL_ERR_CUDA -4        /* device failure / no CUDA device / ext. missing      */
#define GL_ERR_CONSISTENCY -5 /* graphlet::count_consistency_error (counts.hpp:13-16)*/
#define GL_ERR_OVERFLOW -6    /* graphlet::count_overflow_error (128-bit sums, 16-bit H-member ids) */
#define GL_ERR_OOM -7         /* device allocation failed                           */
#define GL_ERR_STATE -8       /* call sequence violated (e.g. finish before begin)  */

const char *gl_last_error(void);
uint64_t gl_last_error_line(void);
const char *gl_version(void);

/* 128-bit unsigned count, little-endian limbs (count_t, common.hpp:17). */
typedef struct {
    uint64_t lo, hi;
} gl_u128;

/* Global counts X_0..X_17, X[0] unused (GraphletVector, counts.hpp:55-61). */
typedef struct {
    gl_u128 x[18];
} gl_graphlet_vector;

/* Unrestricted sums C_0..C_16, indices 3..5 and 7..16 used
 * (UnrestrictedCounts, counts.hpp:41-47). */
typedef struct {
    gl_u128 c[17];
} gl_unrestricted;

/* Per-edge micro record, field-for-field the reference MicroRecord
 * (counts.hpp:82-89) widened to 64-bit edge ids. */
typedef struct {
    uint64_t edge_id, x3, x4, x5, x7, x10, t, s_u, s_v, d_e;
} gl_micro_record;

/* ------------------------------------------------------------------ input */

/* Parse a text edge list held in memory (load_edge_list, graph.hpp:38;
 * graph.cpp:47-85): '#'/'%' comments, a %%MatrixMarket banner skips the next
 * dimension line, two unsigned integer tokens per data line.  On success
 * *pairs is a malloc'd array of 2*count labels (a0,b0,a1,b1,...) to be freed
 * with gl_free(); an empty input yields count 0. */
int gl_load_edge_list(const char *text, size_t len, uint64_t **pairs, uint64_t *count);
/* load_edge_list_file (graph.hpp:39; graph.cpp:87-91). */
int gl_load_edge_list_file(const char *path, uint64_t **pairs, uint64_t *count);
/* load_edge_list (graph.cpp:47-85) executed on `device`: the text is copied to
 * HBM and cut, checked and parsed there, one thread per line (same rules and
 * the same parse_error line numbers and messages as gl_load_edge_list).
 * Pairs returned like gl_load_edge_list (free with gl_free). */
int gl_parse_edge_list_device(const char *text, size_t len, int device, uint64_t **pairs, uint64_t *count);
void gl_free(void *p);
/* Device memory freed by gl_graph_free is cached per device for the next
 * graph (no reference counterpart: the reference is host-only); this returns
 * the cache to the driver. */
int gl_trim_device_cache(void);

/* Deterministic synthetic generators (SPEC cli "built-in deterministic
 * generator"); host output, 2*count labels.  RMAT uses Graph500 quadrant
 * probabilities given as a,b,c (d = 1-a-b-c) and a counter-based hash, so
 * gl_generate_rmat_device() produces the identical list directly in HBM. */
int gl_generate_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                     uint64_t seed, uint64_t **pairs, uint64_t *count);
int gl_generate_rmat_device(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                            uint64_t seed, int device, uint64_t *d_pairs /* 2*count */,
                            uint64_t count);
/* Erdos-Renyi G(n, m): exactly m distinct non-loop edges. */
int gl_generate_gnm(uint64_t n, uint64_t m, uint64_t seed, uint64_t **pairs, uint64_t *count);
/* Barabasi-Albert: n vertices, each new vertex attaches `attach` edges. */
int gl_generate_ba(uint64_t n, uint32_t attach, uint64_t seed, uint64_t **pairs, uint64_t *count);

/* ------------------------------------------------------------------ graph */

typedef struct gl_graph gl_graph; /* device-resident preprocessed graph */

/* build_graph (graph.hpp:96; graph.cpp:93-172) executed on `device`:
 * label compaction, self-loop and duplicate removal, P1 relabel by
 * (degree asc, label asc), id-sorted CSR rows, oriented edge ids identical to
 * orient_edges (graph.cpp:180-193).  `pairs` is a HOST array of 2*count labels. */
int gl_graph_build(const uint64_t *pairs, uint64_t count, int device, gl_graph **out);
/* Same, `d_pairs` already in device memory on `device` (not modified). */
int gl_graph_build_device(const uint64_t *d_pairs, uint64_t count, int device, gl_graph **out);
/* gl_parse_edge_list_device + build_graph without the pairs leaving the device:
 * edge-list text -> device-resident graph. */
int gl_graph_build_text(const char *text, size_t len, int device, gl_graph **out);
void gl_graph_free(gl_graph *g);

uint64_t gl_graph_num_vertices(const gl_graph *g); /* Graph::num_vertices */
uint64_t gl_graph_num_edges(const gl_graph *g);    /* Graph::num_edges    */
uint32_t gl_graph_max_degree(const gl_graph *g);   /* Graph::max_degree   */
/* Host copies: degree[n] (Graph::degree), label[n] (Graph::original_label),
 * offsets[n+1] and adjacency[2m] (Graph::neighbors_by_id rows). */
int gl_graph_degrees(const gl_graph *g, uint32_t *degree);
int gl_graph_labels(const gl_graph *g, uint64_t *label);
int gl_graph_csr(const gl_graph *g, uint64_t *offsets, uint32_t *adjacency);
/* orient_edges (graph.hpp:107): internal ids of (v = high, u = low) per edge id. */
int gl_orient_edges(const gl_graph *g, uint32_t *v, uint32_t *u);

/* ------------------------------------------------------------- counting */

/* Count all 2/3/4-vertex graphlets, macro and micro, on the graph's device.
 * Replaces the reference's per-edge loop process_edge_hash/_bsearch
 * (kernels.hpp:99-102) + accumulate_unrestricted + merge
 * (counts.hpp:49-51) + global_from_unrestricted (counts.hpp:69-70).
 * `unres` may be NULL.  Per-edge results stay resident on the device for
 * gl_micro_* below. */
int gl_count(gl_graph *g, gl_graphlet_vector *X, gl_unrestricted *unres);

/* Sharded form for one process per GPU.  The
 * graph is replicated; every rank calls, in order:
 *  1. gl_count_begin: this rank's cost-balanced share (rank of world) of the
 *     clique/triangle pass and of the cycle pass.  Leaves per-edge int64
 *     partial rows {x7, C4 - S} in `d_partials` (device memory of
 *     2*gl_partials_len(g, world) int64, zeroed by the callee) and partial
 *     per-edge triangle counts (gl_triangle_counts_device).
 *  2. caller sums the uint32 triangle counts across ranks in place
 *     (all-reduce; skip when world == 1).
 *  3. gl_count_mid: this rank's share of the triangle sums S (needs all of t).
 *  4. caller sums d_partials across ranks so that rank r holds the summed
 *     rows of its edge shard [edge_begin, edge_end) (reduce-scatter).
 *  5. gl_count_finish(d_shard = rows of edge_begin..edge_end): per-edge
 *     epilogue for that shard, micro records on device, unrestricted
 *     partial sums in *unres.
 *  6. caller sums unres across ranks (e.g. as 32-bit limbs in int64) and
 *     calls gl_global_from_unrestricted.
 * Steps 1-5 are asynchronous on `stream` (NULL: the graph's own stream); the
 * caller's collectives belong on the same stream or must wait for it.
 * gl_count_begin may be called again before gl_count_mid (it first drains the
 * previous call's cycle pass). */
uint64_t gl_partials_len(const gl_graph *g, int world);
int gl_count_begin(gl_graph *g, int rank, int world, int64_t *d_partials, void *stream);
int gl_triangle_counts_device(gl_graph *g, uint32_t **d_t, uint64_t *count);
int gl_count_mid(gl_graph *g, int64_t *d_partials, void *stream);
int gl_count_finish(gl_graph *g, const int64_t *d_shard, uint64_t edge_begin,
                    uint64_t edge_end, gl_unrestricted *unres, void *stream);

/* global_from_unrestricted (counts.cpp:86-111), host-side 128-bit algebra.
 * GL_ERR_CONSISTENCY on an inexact division or a negative intermediate. */
int gl_global_from_unrestricted(const gl_unrestricted *c, uint64_t n, uint64_t m,
                                gl_graphlet_vector *X);

/* micro_counts (counts.hpp:90; counts.cpp:122-136) for edge ids
 * [first, first+count) of the last gl_count / gl_count_finish shard. */
int gl_micro_records(const gl_graph *g, uint64_t first, uint64_t count, gl_micro_record *out);
/* gl_count plus the compact per-edge output of every edge id (t, x7, x10, as
 * gl_edge_counts; any pointer may be NULL): t and x7 are final after the
 * clique/triangle pass, so their device-to-host copies overlap the cycle pass
 * (pinned host buffers make that copy truly asynchronous). */
int gl_count_edges(gl_graph *g, gl_graphlet_vector *X, gl_unrestricted *unres, uint32_t *t, uint64_t *x7,
                   uint64_t *x10);
/* EdgeMotifRecord (counts.hpp:20-35) of process_edge_hash (kernels.cpp:143-156)
 * for edge ids [first, first+count) of the last count's shard: t, s_u, s_v,
 * x7, x10 and the reference's deterministic operation counter, which for the
 * hash pipeline is closed-form: work_units = deg(u) + deg(v) + sum of deg(w)
 * over w in N(u) (three_graphlets_hash reads N(v) and N(u), derive_s_v
 * N(v), clique_hash / cycle_hash N(w) for w in T u S_u = N(u) \ {v}). */
typedef struct {
    uint32_t edge_id, t, s_u, s_v;
    uint64_t x7, x10, work_units;
} gl_edge_motif_record;
int gl_edge_motif_records(const gl_graph *g, uint64_t first, uint64_t count, gl_edge_motif_record *out);
/* Compact per-edge output (SoA, host): t, x7, x10 for edge ids
 * [first, first+count); any pointer may be NULL.  The other MicroRecord
 * fields are closed-form in (t, deg(u), deg(v), n) -- counts.cpp:113-136. */
int gl_edge_counts(const gl_graph *g, uint64_t first, uint64_t count, uint32_t *t, uint64_t *x7,
                   uint64_t *x10);
/* Device pointers of the resident per-edge arrays (t: uint32[m], x7 and x10:
 * uint64[m]); valid until the next count call or gl_graph_free. */
int gl_edge_counts_device(const gl_graph *g, const uint32_t **t, const uint64_t **x7,
                          const uint64_t **x10);

/* 1: the cycle pass runs on its own stream concurrently with the clique /
 * triangle pass; 0 (default; concurrency measured slower on B200: both
 * passes fill every SM and share L2) runs them one after the other on the
 * caller's stream. Process-wide. */
int gl_set_overlap(int on);

/* Kernel timing of the last count call (CUDA events on the launching stream),
 * milliseconds: [0] clique+triangle pass, [1] triangle sums, [2] cycles,
 * [3] epilogue+macro reduction, [4] total.  Launch count in *launches. */
int gl_last_timings(const gl_graph *g, float ms[5], uint32_t *launches);
/* Algorithmic work counters of the last count call:
 * algorithmic bytes per phase, same order as gl_last_timings [0..3]. */
int gl_last_work(const gl_graph *g, uint64_t work[4]);
/* Work items of the cycle pass's windowed (heavy) tops in the last
 * gl_count_begin, all ranks: 4 x u32 per item = (top a, c_lo, c_hi, wedge
 * estimate); item i covers the wedges a-b-c with c in [c_lo, c_hi).  A top
 * above the piece cap is split into several such c-range pieces, the unit of
 * fine-grained task splitting (reference cycle_res_range + split_threshold,
 * include/graphlet/kernels.hpp:68-80).  Writes min(*count_total, cap) items;
 * out may be NULL to query the count. */
int gl_cycle_pieces(const gl_graph *g, uint32_t *out, uint64_t cap, uint64_t *count_total);

#ifdef __cplusplus
}
#endif
#endif /* GRAPHLET_B200_H */
