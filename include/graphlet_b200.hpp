// graphlet_b200.hpp -- header-only C++ mirror of the reference's counting-path
// API (/root/reference/proj/include/graphlet/{common,graph,counts}.hpp) over the
// C-ABI in graphlet_b200.h.  Same type names, field order and exception
// classes, in namespace graphlet::b200 so that it can sit beside the reference
// library in one program (INTEGRATION.md shows the switch-over).
//
//   reference                               here
//   RawEdges, parse_error                   RawEdges, parse_error          (graph.hpp:18-33)
//   load_edge_list(istream&) / _file        load_edge_list / _file         (graph.hpp:38-39)
//   Graph + build_graph(RawEdges)           Graph (device-resident), build_graph(raw, device)
//   OrientedEdge + orient_edges(g)          OrientedEdge, orient_edges(g)  (graph.hpp:100-107)
//   GraphletVector, UnrestrictedCounts      same                           (counts.hpp:41-61)
//   per-edge loop + accumulate/merge +      count(g) -> Counts{global, unrestricted}
//     global_from_unrestricted
//   MicroRecord + micro_counts              MicroRecord, micro_records(g)  (counts.hpp:82-90)
//   EdgeMotifRecord + process_edge_hash     EdgeMotifRecord, edge_motif_records(g), process_edge_hash(g, e)
//                                           (counts.hpp:20-35, kernels.hpp:99-102; work_units = the
//                                           hash pipeline's operation counter, closed form)
//   LocalThree + local_three_counts         same                           (counts.hpp:73-78)
//   Graph::degree / neighbors (degree-      same, on a host copy of the CSR loaded on first use
//     descending view) / neighbors_by_id /  (graph.hpp:56-79)
//     has_edge / original_label /
//     internal_id / degree_order_less
//   graphlet_name(i)                        graphlet_name(i)               (counts.hpp:64)
//   count_consistency_error,                same; CUDA failures -> cuda_error
//     count_overflow_error
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <istream>
#include <memory>
#include <span>
#include <unordered_map>
#include <iterator>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "graphlet_b200.h"

namespace graphlet {
namespace b200 {

using vid_t = std::uint32_t;
using eid_t = std::uint64_t; // widened: edge ids of the device path are 64-bit
using count_t = unsigned __int128;

// ------------------------------------------------------------------ errors

class parse_error : public std::runtime_error {
public:
    parse_error(std::size_t line, const std::string& what) : std::runtime_error(what), line_(line) {}
    std::size_t line() const { return line_; }

private:
    std::size_t line_;
};
class count_consistency_error : public std::logic_error {
public:
    using std::logic_error::logic_error;
};
class count_overflow_error : public std::overflow_error {
public:
    using std::overflow_error::overflow_error;
};
class cuda_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == GL_OK) return;
    const std::string msg = gl_last_error();
    switch (rc) {
    case GL_ERR_PARSE: throw parse_error((std::size_t)gl_last_error_line(), msg);
    case GL_ERR_CONSISTENCY: throw count_consistency_error(msg);
    case GL_ERR_OVERFLOW: throw count_overflow_error(msg);
    case GL_ERR_INVALID: throw std::invalid_argument(msg);
    case GL_ERR_IO: throw std::runtime_error(msg);
    case GL_ERR_STATE: throw std::logic_error(msg);
    default: throw cuda_error(msg);
    }
}

// ------------------------------------------------------------------ input

struct RawEdges {
    std::vector<std::pair<std::uint64_t, std::uint64_t>> pairs;
};

namespace detail {
inline RawEdges from_flat(std::uint64_t* flat, std::uint64_t count) {
    RawEdges r;
    r.pairs.reserve(count);
    for (std::uint64_t i = 0; i < count; ++i) r.pairs.emplace_back(flat[2 * i], flat[2 * i + 1]);
    gl_free(flat);
    return r;
}
inline std::vector<std::uint64_t> to_flat(const RawEdges& raw) {
    std::vector<std::uint64_t> flat;
    flat.reserve(raw.pairs.size() * 2);
    for (const auto& p : raw.pairs) {
        flat.push_back(p.first);
        flat.push_back(p.second);
    }
    return flat;
}
} // namespace detail

// graph.cpp:47-85 (same comment / MatrixMarket / token rules, parse_error line numbers)
inline RawEdges load_edge_list(std::istream& in) {
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    std::uint64_t* flat = nullptr;
    std::uint64_t count = 0;
    check(gl_load_edge_list(text.data(), text.size(), &flat, &count));
    return detail::from_flat(flat, count);
}
inline RawEdges load_edge_list_file(const std::string& path) {
    std::uint64_t* flat = nullptr;
    std::uint64_t count = 0;
    check(gl_load_edge_list_file(path.c_str(), &flat, &count));
    return detail::from_flat(flat, count);
}

// ------------------------------------------------------------------ counts

struct GraphletVector {
    count_t x[18] = {};
    count_t& X(int i) { return x[i]; }
    count_t X(int i) const { return x[i]; }
    bool operator==(const GraphletVector& o) const {
        for (int i = 0; i < 18; ++i)
            if (x[i] != o.x[i]) return false;
        return true;
    }
};
struct UnrestrictedCounts {
    count_t c3 = 0, c4 = 0, c5 = 0;
    count_t c7 = 0, c8 = 0, c9 = 0, c10 = 0, c11 = 0, c12 = 0;
    count_t c13 = 0, c14 = 0, c15 = 0, c16 = 0;
};
struct MicroRecord {
    eid_t edge_id = 0;
    std::uint64_t x3 = 0, x4 = 0, x5 = 0;
    std::uint64_t x7 = 0, x10 = 0;
    std::uint64_t t = 0, s_u = 0, s_v = 0, d_e = 0;
};
struct OrientedEdge {
    vid_t v = 0; // high-degree endpoint
    vid_t u = 0; // low-degree endpoint
    eid_t id = 0;
};
struct EdgeMotifRecord {
    eid_t edge_id = 0;
    std::uint32_t t = 0;
    std::uint32_t s_u = 0;
    std::uint32_t s_v = 0;
    std::uint64_t x7 = 0;
    std::uint64_t x10 = 0;
    std::uint64_t work_units = 0;

    std::uint32_t x3() const { return t; }
    std::uint64_t disconnected(std::uint64_t n) const { return n - ((std::uint64_t)s_u + s_v + t) - 2; }
};
struct LocalThree {
    std::uint64_t x3 = 0, x4 = 0, x5 = 0;
};
// counts.cpp:113-120
inline LocalThree local_three_counts(const EdgeMotifRecord& rec, std::uint64_t n) {
    if (n < 2) throw std::invalid_argument("local counts need at least two vertices");
    return LocalThree{rec.t, (std::uint64_t)rec.s_u + rec.s_v, rec.disconnected(n)};
}

namespace detail {
inline count_t u128(const gl_u128& v) { return ((count_t)v.hi << 64) | v.lo; }
inline gl_u128 g128(count_t v) { return gl_u128{(std::uint64_t)v, (std::uint64_t)(v >> 64)}; }
inline UnrestrictedCounts unres(const gl_unrestricted& c) {
    UnrestrictedCounts r;
    r.c3 = u128(c.c[3]), r.c4 = u128(c.c[4]), r.c5 = u128(c.c[5]);
    r.c7 = u128(c.c[7]), r.c8 = u128(c.c[8]), r.c9 = u128(c.c[9]), r.c10 = u128(c.c[10]);
    r.c11 = u128(c.c[11]), r.c12 = u128(c.c[12]), r.c13 = u128(c.c[13]), r.c14 = u128(c.c[14]);
    r.c15 = u128(c.c[15]), r.c16 = u128(c.c[16]);
    return r;
}
} // namespace detail

// counts.cpp:86-111 (exact divisions, nonnegative intermediates, else count_consistency_error)
inline GraphletVector global_from_unrestricted(const UnrestrictedCounts& u, std::uint64_t n, std::uint64_t m) {
    gl_unrestricted c{};
    const count_t v[17] = {0, 0, 0, u.c3, u.c4, u.c5, 0, u.c7, u.c8, u.c9, u.c10, u.c11, u.c12, u.c13, u.c14, u.c15,
                           u.c16};
    for (int i = 0; i < 17; ++i) c.c[i] = detail::g128(v[i]);
    gl_graphlet_vector X;
    check(gl_global_from_unrestricted(&c, n, m, &X));
    GraphletVector r;
    for (int i = 0; i < 18; ++i) r.x[i] = detail::u128(X.x[i]);
    return r;
}

// counts.cpp:47-68
inline const char* graphlet_name(int i) {
    static const char* names[18] = {"?",          "edge",           "2-node-independent", "triangle",
                                    "2-star",     "3-node-1-edge",  "3-node-independent", "4-clique",
                                    "chordal-cycle", "tailed-triangle", "4-cycle",       "3-star",
                                    "4-path",     "4-node-1-triangle", "4-node-2-edge",   "4-node-2-star",
                                    "4-node-1-edge", "4-node-independent"};
    return i >= 1 && i <= 17 ? names[i] : "?";
}

inline std::string to_decimal(count_t v) {
    if (v == 0) return "0";
    std::string s;
    while (v) {
        s.insert(s.begin(), char('0' + (int)(v % 10)));
        v /= 10;
    }
    return s;
}

// ------------------------------------------------------------------ graph

// Device-resident preprocessed graph (graph.hpp:41-93 semantics: P1 relabel by
// (degree, label), id-sorted rows, orient_edges ids).  Move-only RAII handle.
class Graph {
public:
    Graph() = default;
    explicit Graph(gl_graph* h) : h_(h) {}
    Graph(Graph&& o) noexcept : h_(o.h_), host_(std::move(o.host_)) { o.h_ = nullptr; }
    Graph& operator=(Graph&& o) noexcept {
        std::swap(h_, o.h_);
        std::swap(host_, o.host_);
        return *this;
    }
    Graph(const Graph&) = delete;
    Graph& operator=(const Graph&) = delete;
    ~Graph() {
        if (h_) gl_graph_free(h_);
    }

    std::uint64_t num_vertices() const { return gl_graph_num_vertices(h_); }
    std::uint64_t num_edges() const { return gl_graph_num_edges(h_); }
    std::uint32_t max_degree() const { return gl_graph_max_degree(h_); }
    std::vector<std::uint32_t> degrees() const {
        std::vector<std::uint32_t> d(num_vertices());
        check(gl_graph_degrees(h_, d.data()));
        return d;
    }
    std::vector<std::uint64_t> original_labels() const {
        std::vector<std::uint64_t> l(num_vertices());
        check(gl_graph_labels(h_, l.data()));
        return l;
    }
    gl_graph* handle() const { return h_; }

    // graph.hpp:56-79 accessors, served from a host copy of the CSR (loaded on
    // first use; the device graph is immutable)
    std::uint32_t degree(vid_t v) const { return host().deg.at(v); }
    std::span<const vid_t> neighbors_by_id(vid_t v) const {
        const Host& h = host();
        return {h.adj.data() + h.off.at(v), h.adj.data() + h.off.at(v + 1)};
    }
    // degree descending, ties by ascending id (the reference's P2 view)
    std::span<const vid_t> neighbors(vid_t v) const {
        const Host& h = host();
        return {h.adj_deg.data() + h.off.at(v), h.adj_deg.data() + h.off.at(v + 1)};
    }
    bool has_edge(vid_t a, vid_t b) const {
        const auto r = neighbors_by_id(a);
        return std::binary_search(r.begin(), r.end(), b);
    }
    std::uint64_t original_label(vid_t v) const { return host().label.at(v); }
    // throws std::out_of_range for an unknown label, like relabel_map_.at
    vid_t internal_id(std::uint64_t label) const { return host().relabel.at(label); }
    bool degree_order_less(vid_t a, vid_t b) const {
        const Host& h = host();
        return h.deg[a] != h.deg[b] ? h.deg[a] > h.deg[b] : a < b;
    }

private:
    struct Host {
        std::vector<std::uint64_t> off, label;
        std::vector<vid_t> adj, adj_deg;
        std::vector<std::uint32_t> deg;
        std::unordered_map<std::uint64_t, vid_t> relabel;
    };
    const Host& host() const {
        if (!host_) {
            auto h = std::make_shared<Host>();
            const std::uint64_t n = num_vertices();
            h->off.resize(n + 1);
            h->deg.resize(n);
            h->label.resize(n);
            check(gl_graph_degrees(h_, h->deg.data()));
            check(gl_graph_labels(h_, h->label.data()));
            h->adj.resize(2 * num_edges());
            check(gl_graph_csr(h_, h->off.data(), h->adj.data()));
            h->adj_deg = h->adj;
            for (std::uint64_t v = 0; v < n; ++v)
                std::sort(h->adj_deg.begin() + h->off[v], h->adj_deg.begin() + h->off[v + 1],
                          [&](vid_t a, vid_t b) { return h->deg[a] != h->deg[b] ? h->deg[a] > h->deg[b] : a < b; });
            h->relabel.reserve(n);
            for (std::uint64_t v = 0; v < n; ++v) h->relabel.emplace(h->label[v], (vid_t)v);
            host_ = std::move(h);
        }
        return *host_;
    }
    gl_graph* h_ = nullptr;
    mutable std::shared_ptr<Host> host_;
};

// graph.cpp:93-172, executed on `device`
inline Graph build_graph(const RawEdges& raw, int device = 0) {
    const std::vector<std::uint64_t> flat = detail::to_flat(raw);
    gl_graph* h = nullptr;
    check(gl_graph_build(flat.data(), raw.pairs.size(), device, &h));
    return Graph(h);
}

// graph.cpp:180-193 (ascending (v,u), dense ids)
inline std::vector<OrientedEdge> orient_edges(const Graph& g) {
    const std::uint64_t m = g.num_edges();
    std::vector<std::uint32_t> v(m), u(m);
    check(gl_orient_edges(g.handle(), v.data(), u.data()));
    std::vector<OrientedEdge> out(m);
    for (std::uint64_t i = 0; i < m; ++i) out[i] = OrientedEdge{v[i], u[i], i};
    return out;
}

struct Counts {
    GraphletVector global;            // X1..X17
    UnrestrictedCounts unrestricted;  // C3..C16
};

// every edge's process_edge_* + accumulate_unrestricted + merge +
// global_from_unrestricted, on the graph's device
inline Counts count(Graph& g) {
    gl_graphlet_vector X;
    gl_unrestricted C;
    check(gl_count(g.handle(), &X, &C));
    Counts r;
    for (int i = 0; i < 18; ++i) r.global.x[i] = detail::u128(X.x[i]);
    r.unrestricted = detail::unres(C);
    return r;
}

// micro_counts for every edge id (counts.cpp:122-136), after count(g)
inline std::vector<MicroRecord> micro_records(const Graph& g, std::uint64_t first = 0,
                                              std::uint64_t n = ~0ull) {
    const std::uint64_t m = g.num_edges();
    if (n == ~0ull) n = first < m ? m - first : 0;
    std::vector<gl_micro_record> raw(n);
    if (n) check(gl_micro_records(g.handle(), first, n, raw.data()));
    std::vector<MicroRecord> out(n);
    for (std::uint64_t i = 0; i < n; ++i) {
        const gl_micro_record& r = raw[i];
        out[i] = MicroRecord{r.edge_id, r.x3, r.x4, r.x5, r.x7, r.x10, r.t, r.s_u, r.s_v, r.d_e};
    }
    return out;
}

// EdgeMotifRecord of every edge id in [first, first+n) (after count(g)):
// process_edge_hash's record, kernels.cpp:143-156, work_units included
inline std::vector<EdgeMotifRecord> edge_motif_records(const Graph& g, std::uint64_t first = 0,
                                                       std::uint64_t n = ~0ull) {
    const std::uint64_t m = g.num_edges();
    if (n == ~0ull) n = first < m ? m - first : 0;
    std::vector<gl_edge_motif_record> raw(n);
    if (n) check(gl_edge_motif_records(g.handle(), first, n, raw.data()));
    std::vector<EdgeMotifRecord> out(n);
    for (std::uint64_t i = 0; i < n; ++i) {
        const gl_edge_motif_record& r = raw[i];
        out[i] = EdgeMotifRecord{r.edge_id, r.t, r.s_u, r.s_v, r.x7, r.x10, r.work_units};
    }
    return out;
}
// kernels.cpp:143-156 for one oriented edge (after count(g))
inline EdgeMotifRecord process_edge_hash(const Graph& g, const OrientedEdge& e) {
    return edge_motif_records(g, e.id, 1).at(0);
}

} // namespace b200
} // namespace graphlet
