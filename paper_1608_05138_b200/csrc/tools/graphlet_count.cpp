// graphlet_count -- command-line driver of the B200 counting path, written
// against the C++ mirror of the reference API (include/graphlet_b200.hpp).
// Mirrors the reference CLI's count command (SPEC "cli" cmd_count) for the
// path this repo builds: the result document lists graph metadata and X1..X17
// as exact decimal strings (JSON default, or CSV), --micro writes one row per
// oriented edge with the reference MicroRecord fields.
//
//   graphlet_count count <edge-list> [--device N] [--format json|csv]
//                  [--output PATH] [--micro PATH]
//   exit codes: 0 ok, 1 IO / device failure, 2 usage or parse error
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "graphlet_b200.hpp"

namespace gb = graphlet::b200;

static int usage() {
    std::fprintf(stderr,
                 "usage: graphlet_count count <edge-list> [--device N] [--format json|csv] "
                 "[--output PATH] [--micro PATH]\n");
    return 2;
}

int main(int argc, char** argv) {
    if (argc < 3 || std::strcmp(argv[1], "count") != 0) return usage();
    std::string path = argv[2], format = "json", output, micro;
    int device = 0;
    for (int i = 3; i < argc; ++i) {
        const std::string a = argv[i];
        if (i + 1 >= argc) return usage();
        if (a == "--device")
            device = std::atoi(argv[++i]);
        else if (a == "--format")
            format = argv[++i];
        else if (a == "--output")
            output = argv[++i];
        else if (a == "--micro")
            micro = argv[++i];
        else
            return usage();
    }
    if (format != "json" && format != "csv") return usage();
    try {
        const gb::RawEdges raw = gb::load_edge_list_file(path);
        gb::Graph g = gb::build_graph(raw, device);
        const gb::Counts c = gb::count(g);
        std::ostringstream doc;
        if (format == "json") {
            doc << "{\"n\": " << g.num_vertices() << ", \"m\": " << g.num_edges()
                << ", \"d_max\": " << g.max_degree() << ", \"counts\": {";
            for (int i = 1; i <= 17; ++i)
                doc << (i > 1 ? ", " : "") << "\"X" << i << "\": \"" << gb::to_decimal(c.global.X(i)) << "\"";
            doc << "}}\n";
        } else {
            doc << "class,name,count\n";
            for (int i = 1; i <= 17; ++i)
                doc << "X" << i << "," << gb::graphlet_name(i) << "," << gb::to_decimal(c.global.X(i)) << "\n";
        }
        if (output.empty()) {
            std::cout << doc.str();
        } else {
            std::ofstream f(output);
            if (!f) throw std::runtime_error("cannot open " + output);
            f << doc.str();
        }
        if (!micro.empty()) {
            std::ofstream f(micro);
            if (!f) throw std::runtime_error("cannot open " + micro);
            f << "edge_id,x3,x4,x5,x7,x10,t,s_u,s_v,d_e\n";
            for (const gb::MicroRecord& r : gb::micro_records(g))
                f << r.edge_id << "," << r.x3 << "," << r.x4 << "," << r.x5 << "," << r.x7 << "," << r.x10 << ","
                  << r.t << "," << r.s_u << "," << r.s_v << "," << r.d_e << "\n";
        }
    } catch (const gb::parse_error& e) {
        std::fprintf(stderr, "parse error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
