/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's CPU graphlet path
 * (/root/reference/proj, arxiv 1608.05138 "Hybrid CPU-GPU Framework for
 * Network Motifs").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the
 * checker / CPU baseline.  The product path (libgraphlet_b200.so) never links
 * or calls it.
 *
 * Pinned against: the SPEC known-answer examples (tests/test_oracle.py), the
 * brute-force census restated from oracle.cpp, and golden vectors produced by
 * the reference's own sources compiled here (oracle/_ref, tests/golden/).
 */
#ifndef GRAPHLET_ORACLE_H
#define GRAPHLET_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint64_t n, m;
    uint32_t dmax;
    uint64_t *offsets;     /* n+1 */
    uint32_t *adj_id;      /* 2m, ascending id per row          (graph.cpp:161-168) */
    uint32_t *adj_deg;     /* 2m, degree-descending per row     (graph.cpp:170-171) */
    uint32_t *degree;      /* n */
    uint64_t *inverse_map; /* n: internal id -> original label  */
} or_graph;

/* One row per oriented edge, identical in meaning to the reference's
 * MicroRecord (counts.hpp:82-89) with x3=t, x4=s_u+s_v, x5=d_e. */
typedef struct {
    uint64_t edge_id, x3, x4, x5, x7, x10, t, s_u, s_v, d_e;
} or_micro;

/* 128-bit values travel as (lo, hi) pairs. X[2*i], X[2*i+1] = X_i. */
int  or_build_graph(const uint64_t *a, const uint64_t *b, uint64_t count, or_graph *g);
void or_free_graph(or_graph *g);

/* Oriented edge list (graph.cpp:180-193): v (high id), u (low id) per edge. */
void or_orient_edges(const or_graph *g, uint32_t *v_out, uint32_t *u_out);

/* Full pipeline: process_edge_hash for every edge, accumulate_unrestricted,
 * merge across threads, global_from_unrestricted.  micro may be NULL.
 * Returns 0 on success, -1 on count-consistency error. */
int or_count(const or_graph *g, int nthreads, uint64_t X[36], or_micro *micro);

/* Per-edge binary-search pipeline (Algs. 2-4) for one edge; for the
 * variant-equivalence tests. rec = {t, s_u, s_v, x7, x10}. */
void or_process_edge_bsearch(const or_graph *g, uint32_t v, uint32_t u, uint64_t rec[5]);
void or_process_edge_hash_one(const or_graph *g, uint32_t v, uint32_t u, uint64_t eid, uint64_t rec[5]);

/* Hash pipeline for the listed edge ids; out = k x {t, s_u, s_v, x7, x10}. */
void or_edges_hash(const or_graph *g, const uint64_t *ids, uint64_t k, uint64_t *out);

/* Process only the listed edge ids (hash pipeline) with nthreads workers and
 * return elapsed seconds; checksum = sum of (t + x7 + x10) over the sample. */
double or_time_sample(const or_graph *g, int nthreads, const uint64_t *edge_ids,
                      uint64_t k, uint64_t *checksum);

/* Exhaustive census (oracle.cpp:48-66); -1 if n > cap. */
int or_brute_force_global(const or_graph *g, uint32_t cap, uint64_t X[36]);

/* Unrestricted sums -> X_1..X_17 (counts.cpp:86-111); C[2*i..] for i in 0..16
 * holds C_i (indices 3..16 used).  Returns -1 on inexact/negative. */
int or_global_from_unrestricted(const uint64_t C[34], uint64_t n, uint64_t m, uint64_t X[36]);

/* Ports of the product's synthetic generators (csrc/common.cuh rmat_edge,
 * csrc/host.cpp generate_ba): identical pairs, no product library needed.
 * or_generate_rmat writes 2*(edge_factor << scale) labels into out. */
int or_generate_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c, uint64_t seed,
                     int nthreads, uint64_t *out);
int or_generate_ba(uint64_t n, uint32_t k, uint64_t seed, uint64_t **out, uint64_t *count);
void or_free_pairs(uint64_t *p);

#ifdef __cplusplus
}
#endif
#endif
