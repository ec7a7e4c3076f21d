// Host-only checks of the C++ mirror (include/graphlet_b200.hpp): parser and
// error mapping, count algebra, names.  Built and run by tests/test_host.py
// (no device calls); prints "ok" on success.
#include <cassert>
#include <cstdio>
#include <sstream>

#include "graphlet_b200.hpp"

namespace gb = graphlet::b200;

int main() {
    std::istringstream in("%%MatrixMarket matrix coordinate\n3 3 2\n# c\n1 2\n2 3\n");
    gb::RawEdges r = gb::load_edge_list(in);
    assert(r.pairs.size() == 2 && r.pairs[0].first == 1 && r.pairs[1].second == 3);
    std::istringstream bad("1 2\n3 x\n");
    bool threw = false;
    try {
        gb::load_edge_list(bad);
    } catch (const gb::parse_error& e) {
        threw = e.line() == 2;
    }
    assert(threw);
    // path P3 (n = 3, m = 2): C3 = 0 (no triangle), C4 = 2 (one 2-star seen from both edges)
    gb::UnrestrictedCounts u;
    u.c4 = 2;
    u.c5 = 0;
    gb::GraphletVector X = gb::global_from_unrestricted(u, 3, 2);
    assert(X.X(1) == 2 && X.X(2) == 1 && X.X(4) == 1 && X.X(3) == 0);
    bool inconsistent = false;
    try {
        gb::UnrestrictedCounts v;
        v.c3 = 1; // a triangle counted once instead of three times
        gb::global_from_unrestricted(v, 3, 3);
    } catch (const gb::count_consistency_error&) {
        inconsistent = true;
    }
    assert(inconsistent);
    assert(std::string(gb::graphlet_name(10)) == "4-cycle" && std::string(gb::graphlet_name(0)) == "?");
    assert(gb::to_decimal((gb::count_t)1 << 100) == "1267650600228229401496703205376");
    // counts.cpp:113-120
    gb::EdgeMotifRecord rec{0, 2, 3, 1, 1, 0, 0};
    const gb::LocalThree l3 = gb::local_three_counts(rec, 10);
    assert(l3.x3 == 2 && l3.x4 == 4 && l3.x5 == 2);
    bool small = false;
    try {
        gb::local_three_counts(rec, 1);
    } catch (const std::invalid_argument&) {
        small = true;
    }
    assert(small);
    std::printf("ok\n");
    return 0;
}
