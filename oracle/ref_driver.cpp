// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the reference's OWN sources
// (/root/reference/proj/src/{graph,kernels,counts,oracle}.cpp, compiled in
// place by oracle/Makefile into oracle/_ref/libgraphlet_ref.so).  Nothing of
// the reference is copied here: this file only drives its public C++ API
// (graph.hpp, kernels.hpp, counts.hpp, oracle.hpp) so that tests can pin the
// C oracle and the CUDA path against the real thing, and bench.py can time the
// reference CPU path (`--impl reference`, cpu_baseline kind "reference").
//
// The reference snapshot has no scheduler.cpp (its CMakeLists lists one, the
// file is absent), so the multi-threaded driver below is the plain
// "split the oriented edge list across workers, merge the partials" schedule
// described in SPEC.md (scheduler module, cpu-only config): every worker runs
// the reference's process_edge_hash (kernels.cpp:143-156) with its own
// StampTable and NeighborhoodSets, accumulates with accumulate_unrestricted and
// the partials are combined with merge().

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "graphlet/counts.hpp"
#include "graphlet/graph.hpp"
#include "graphlet/kernels.hpp"
#include "graphlet/oracle.hpp"

using namespace graphlet;

namespace {

struct RefGraph {
    Graph g;
    std::vector<OrientedEdge> edges;
};

void store(std::uint64_t* dst, count_t v) {
    dst[0] = (std::uint64_t)v;
    dst[1] = (std::uint64_t)(v >> 64);
}

thread_local std::string g_err;

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_build(const std::uint64_t* a, const std::uint64_t* b, std::uint64_t count) {
    try {
        RawEdges raw;
        raw.pairs.reserve(count);
        for (std::uint64_t i = 0; i < count; ++i) raw.pairs.emplace_back(a[i], b[i]);
        auto* rg = new RefGraph;
        rg->g = build_graph(raw);
        rg->edges = orient_edges(rg->g);
        return rg;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_free(void* h) { delete static_cast<RefGraph*>(h); }
std::uint64_t ref_n(void* h) { return static_cast<RefGraph*>(h)->g.num_vertices(); }
std::uint64_t ref_m(void* h) { return static_cast<RefGraph*>(h)->g.num_edges(); }
std::uint32_t ref_dmax(void* h) { return static_cast<RefGraph*>(h)->g.max_degree(); }

// internal ids of the oriented edges and original labels of their endpoints
void ref_orient(void* h, std::uint32_t* v, std::uint32_t* u, std::uint64_t* v_label,
                std::uint64_t* u_label) {
    auto* rg = static_cast<RefGraph*>(h);
    for (std::size_t k = 0; k < rg->edges.size(); ++k) {
        const auto& e = rg->edges[k];
        if (v) v[k] = e.v;
        if (u) u[k] = e.u;
        if (v_label) v_label[k] = rg->g.original_label(e.v);
        if (u_label) u_label[k] = rg->g.original_label(e.u);
    }
}

void ref_degrees(void* h, std::uint32_t* deg) {
    auto* rg = static_cast<RefGraph*>(h);
    for (std::uint64_t v = 0; v < rg->g.num_vertices(); ++v) deg[v] = rg->g.degree((vid_t)v);
}

// Parse an edge list with the reference parser. Returns number of pairs, or
// -1 with *err_line set on parse_error.
std::int64_t ref_parse(const char* text, std::uint64_t len, std::uint64_t* out, std::uint64_t cap,
                       std::uint64_t* err_line) {
    try {
        std::istringstream in(std::string(text, len));
        RawEdges raw = load_edge_list(in);
        for (std::size_t i = 0; i < raw.pairs.size() && i < cap; ++i) {
            out[2 * i] = raw.pairs[i].first;
            out[2 * i + 1] = raw.pairs[i].second;
        }
        return (std::int64_t)raw.pairs.size();
    } catch (const parse_error& e) {
        g_err = e.what();
        if (err_line) *err_line = e.line();
        return -1;
    }
}

// Per-edge records for every oriented edge with the chosen pipeline
// (0 = hash, Algs. 1/5/6; 1 = binary search, Algs. 2/3/4).
// out: m x 6 = {t, s_u, s_v, x7, x10, work_units}.
void ref_edge_records(void* h, int variant, std::uint64_t* out) {
    auto* rg = static_cast<RefGraph*>(h);
    StampTable psi(rg->g.num_vertices());
    NeighborhoodSets sets;
    sets.reserve(rg->g.max_degree());
    for (std::size_t k = 0; k < rg->edges.size(); ++k) {
        EdgeMotifRecord r = variant == 0 ? process_edge_hash(rg->g, psi, rg->edges[k], sets)
                                         : process_edge_bsearch(rg->g, rg->edges[k], sets);
        std::uint64_t* o = out + 6 * k;
        o[0] = r.t; o[1] = r.s_u; o[2] = r.s_v; o[3] = r.x7; o[4] = r.x10; o[5] = r.work_units;
    }
}

// Full run: X (36 = 18 x (lo,hi)), optional micro table m x 10 in MicroRecord
// field order {edge_id, x3, x4, x5, x7, x10, t, s_u, s_v, d_e}.
int ref_count(void* h, int nthreads, std::uint64_t* X, std::uint64_t* micro) {
    auto* rg = static_cast<RefGraph*>(h);
    try {
        const std::uint64_t n = rg->g.num_vertices(), m = rg->g.num_edges();
        if (nthreads < 1) nthreads = 1;
        std::vector<UnrestrictedCounts> part(nthreads);
        std::atomic<std::uint64_t> next{0};
        std::vector<std::thread> th;
        std::vector<std::string> errs(nthreads);
        for (int w = 0; w < nthreads; ++w)
            th.emplace_back([&, w] {
                try {
                    StampTable psi(n);
                    NeighborhoodSets sets;
                    sets.reserve(rg->g.max_degree());
                    for (;;) {
                        std::uint64_t b = next.fetch_add(64);
                        if (b >= m) break;
                        std::uint64_t e = std::min<std::uint64_t>(b + 64, m);
                        for (std::uint64_t k = b; k < e; ++k) {
                            EdgeMotifRecord r = process_edge_hash(rg->g, psi, rg->edges[k], sets);
                            accumulate_unrestricted(part[w], r, n, m);
                            if (micro) {
                                MicroRecord mr = micro_counts(r, n);
                                std::uint64_t* o = micro + 10 * k;
                                o[0] = mr.edge_id; o[1] = mr.x3; o[2] = mr.x4; o[3] = mr.x5;
                                o[4] = mr.x7; o[5] = mr.x10; o[6] = mr.t; o[7] = mr.s_u;
                                o[8] = mr.s_v; o[9] = mr.d_e;
                            }
                        }
                    }
                } catch (const std::exception& ex) {
                    errs[w] = ex.what();
                }
            });
        for (auto& t : th) t.join();
        for (auto& e : errs)
            if (!e.empty()) { g_err = e; return -1; }
        UnrestrictedCounts acc;
        for (auto& p : part) acc = merge(acc, p);
        GraphletVector gv = global_from_unrestricted(acc, n, m);
        for (int i = 0; i < 18; ++i) store(X + 2 * i, gv.X(i));
        return 0;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return -1;
    }
}

// Time the reference hash pipeline over a sample of edge ids with nthreads
// workers; checksum = sum of (t + x7 + x10).
double ref_time_sample(void* h, int nthreads, const std::uint64_t* ids, std::uint64_t k,
                       std::uint64_t* checksum) {
    auto* rg = static_cast<RefGraph*>(h);
    const std::uint64_t n = rg->g.num_vertices(), m = rg->g.num_edges();
    if (nthreads < 1) nthreads = 1;
    std::vector<UnrestrictedCounts> part(nthreads);
    std::vector<std::uint64_t> sums(nthreads, 0);
    std::atomic<std::uint64_t> next{0};
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int w = 0; w < nthreads; ++w)
        th.emplace_back([&, w] {
            StampTable psi(n);
            NeighborhoodSets sets;
            sets.reserve(rg->g.max_degree());
            for (;;) {
                std::uint64_t b = next.fetch_add(16);
                if (b >= k) break;
                std::uint64_t e = std::min<std::uint64_t>(b + 16, k);
                for (std::uint64_t i = b; i < e; ++i) {
                    EdgeMotifRecord r = process_edge_hash(rg->g, psi, rg->edges[ids[i]], sets);
                    accumulate_unrestricted(part[w], r, n, m);
                    sums[w] += r.t + r.x7 + r.x10;
                }
            }
        });
    for (auto& t : th) t.join();
    auto t1 = std::chrono::steady_clock::now();
    std::uint64_t cs = 0;
    for (auto s : sums) cs += s;
    if (checksum) *checksum = cs;
    return std::chrono::duration<double>(t1 - t0).count();
}

// The reference's per-edge pipeline (process_edge_hash, kernels.cpp:143-156)
// for the listed oriented edge ids, nthreads workers; out = k rows of
// {v label, u label, t, s_u, s_v, x7, x10} (labels = original vertex labels,
// so a fixture also pins which edge an id names).
int ref_edges(void* h, int nthreads, const std::uint64_t* ids, std::uint64_t k, std::uint64_t* out) {
    auto* rg = static_cast<RefGraph*>(h);
    try {
        const std::uint64_t n = rg->g.num_vertices(), m = rg->g.num_edges();
        for (std::uint64_t i = 0; i < k; ++i)
            if (ids[i] >= m) throw std::out_of_range("edge id out of range");
        if (nthreads < 1) nthreads = 1;
        std::atomic<std::uint64_t> next{0};
        std::vector<std::thread> th;
        for (int w = 0; w < nthreads; ++w)
            th.emplace_back([&] {
                StampTable psi(n);
                NeighborhoodSets sets;
                sets.reserve(rg->g.max_degree());
                for (;;) {
                    const std::uint64_t i = next.fetch_add(1);
                    if (i >= k) break;
                    const OrientedEdge& e = rg->edges[ids[i]];
                    EdgeMotifRecord r = process_edge_hash(rg->g, psi, e, sets);
                    std::uint64_t* o = out + 7 * i;
                    o[0] = rg->g.original_label(e.v);
                    o[1] = rg->g.original_label(e.u);
                    o[2] = r.t; o[3] = r.s_u; o[4] = r.s_v; o[5] = r.x7; o[6] = r.x10;
                }
            });
        for (auto& t : th) t.join();
        return 0;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return -1;
    }
}

int ref_brute(void* h, std::uint32_t cap, std::uint64_t* X) {
    auto* rg = static_cast<RefGraph*>(h);
    try {
        CensusVector c = brute_force_global(rg->g, cap);
        for (int i = 0; i < 18; ++i) store(X + 2 * i, c.X(i));
        return 0;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return -1;
    }
}

// brute_force_edge (oracle.cpp:69-91) for every oriented edge:
// out m x 6 = {x3, x7, x10, t, s_u, s_v}
void ref_brute_edges(void* h, std::uint64_t* out) {
    auto* rg = static_cast<RefGraph*>(h);
    for (std::size_t k = 0; k < rg->edges.size(); ++k) {
        EdgeBruteCounts b = brute_force_edge(rg->g, rg->edges[k]);
        std::uint64_t* o = out + 6 * k;
        o[0] = b.x3; o[1] = b.x7; o[2] = b.x10; o[3] = b.t; o[4] = b.s_u; o[5] = b.s_v;
    }
}

} // extern "C"
