// Device checks of the C++ mirror (include/graphlet_b200.hpp) against the
// reference's semantics: graph.hpp:56-79 accessors (degree-descending P2 view,
// has_edge, internal_id / original_label, degree_order_less) and
// process_edge_hash records (kernels.cpp:143-156) incl. work_units, on a
// diamond + pendant.  Built and run by tests/test_gpu_api.py; prints "ok".
#include <cassert>
#include <cstdio>
#include <sstream>
#include <stdexcept>

#include "graphlet_b200.hpp"

namespace gb = graphlet::b200;

int main() {
    // labels 10,20,30,40 form a diamond (chord 20-30), 50 hangs off 40.
    // P1 relabel by (degree, label): 50->0, 10->1, 20->2, 30->3, 40->4
    std::istringstream in("10 20\n10 30\n20 30\n20 40\n30 40\n40 50\n");
    gb::Graph g = gb::build_graph(gb::load_edge_list(in));
    assert(g.num_vertices() == 5 && g.num_edges() == 6);
    assert(g.internal_id(50) == 0 && g.internal_id(10) == 1 && g.internal_id(40) == 4);
    assert(g.original_label(3) == 30 && g.degree(4) == 3 && g.degree(0) == 1);
    bool unknown = false;
    try {
        g.internal_id(99);
    } catch (const std::out_of_range&) {
        unknown = true;
    }
    assert(unknown);
    const auto byid = g.neighbors_by_id(4);
    assert(byid.size() == 3 && byid[0] == 0 && byid[1] == 2 && byid[2] == 3);
    const auto p2 = g.neighbors(4); // degree descending, ties by ascending id
    assert(p2.size() == 3 && p2[0] == 2 && p2[1] == 3 && p2[2] == 0);
    assert(g.has_edge(2, 3) && g.has_edge(3, 2) && !g.has_edge(1, 4));
    assert(g.degree_order_less(2, 0) && g.degree_order_less(2, 3) && !g.degree_order_less(3, 2));
    gb::count(g);
    const auto edges = gb::orient_edges(g);
    const auto recs = gb::edge_motif_records(g);
    assert(recs.size() == edges.size());
    for (const auto& e : edges) {
        const gb::EdgeMotifRecord& r = recs[e.id];
        std::uint64_t nbr = 0;
        for (auto w : g.neighbors_by_id(e.u)) nbr += g.degree(w);
        assert(r.edge_id == e.id && r.s_u == g.degree(e.u) - r.t - 1 && r.s_v == g.degree(e.v) - r.t - 1);
        assert(r.work_units == g.degree(e.u) + g.degree(e.v) + nbr);
        if (e.v == 3 && e.u == 2) { // chord 20-30: T = {10, 40}, no edge inside T, S_u = S_v = {}
            const gb::EdgeMotifRecord one = gb::process_edge_hash(g, e);
            assert(one.t == 2 && one.x7 == 0 && one.x10 == 0 && one.s_u == 0 && one.s_v == 0);
            assert(one.work_units == 14); // 3 + 3 (N(v), N(u)) + 3 (derive_s_v) + 2 + 3 (N(w), w in T)
            const gb::LocalThree l = gb::local_three_counts(one, g.num_vertices());
            assert(l.x3 == 2 && l.x4 == 0 && l.x5 == 1);
        }
    }
    std::printf("ok\n");
    return 0;
}
