// capi_parity.cpp -- C++ host-side parity driver: uses the header-only mirror
// (include/tmotif_b200.hpp) the way a reference caller would, on the Fig.-1
// toy graph and a seeded random graph, and prints the census so the gpu test
// can compare it with the oracle.  Mirrors test_executor.cpp:135-163.
#include <cstdio>
#include <string>
#include <vector>

#include "tmotif_b200.hpp"

using namespace tmotif::b200;

int main(int argc, char** argv) {
    if (argc > 3 && std::string(argv[1]) == "parse") {  // "parse <delta> <file>": the GPU reader
        try {
            std::FILE* f = std::fopen(argv[3], "rb");
            if (!f) return 4;
            std::string text;
            char buf[65536];
            std::size_t got;
            while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) text.append(buf, got);
            std::fclose(f);
            EdgeList el = parse_edge_list(text);
            GraphContext ctx(el);
            RunConfig cfg;
            cfg.delta = std::stoll(argv[2]);
            MotifCensus a = run_parallel(ctx, cfg);
            std::printf("NODES %zu EDGES %zu DROPPED %zu FIRST %s\n", el.node_count(), el.edge_count(),
                        el.dropped_self_loops(), el.node_count() ? el.node_ids()[0].c_str() : "-");
            for (int k = 0; k < 36; ++k) std::printf("%s %llu\n", signature(k).c_str(),
                                                     (unsigned long long)a.count_at(k));
        } catch (const ParseError& e) {
            std::printf("PARSE_ERROR %zu %s\n", e.line(), e.what());
            return 5;
        }
        return 0;
    }
    std::size_t n = 0;
    std::vector<NodeId> src, dst;
    std::vector<Timestamp> t;
    Timestamp delta = 10;
    if (argc > 1) {  // "n delta" then edges on stdin
        n = std::stoul(argv[1]);
        delta = std::stoll(argv[2]);
        unsigned long long a, b;
        long long tt;
        while (std::scanf("%llu %llu %lld", &a, &b, &tt) == 3) {
            src.push_back((NodeId)a);
            dst.push_back((NodeId)b);
            t.push_back(tt);
        }
    } else {  // toy graph (a..e by first appearance: e d a c b)
        const int E[12][3] = {{0, 1, 1},  {2, 3, 4},  {0, 3, 6},  {2, 3, 8},
                              {1, 2, 9},  {1, 3, 10}, {2, 4, 11}, {1, 0, 14},
                              {2, 3, 15}, {3, 1, 17}, {0, 1, 18}, {1, 0, 21}};
        n = 5;
        for (auto& e : E) {
            src.push_back(e[0]);
            dst.push_back(e[1]);
            t.push_back(e[2]);
        }
    }
    try {
        GraphContext ctx(src, dst, t, n);
        RunConfig cfg;
        cfg.delta = delta;
        MotifCensus a = run_parallel(ctx, cfg);
        cfg.triangle_mode = TriangleMode::removal;
        MotifCensus b = run_parallel(ctx, cfg);
        if (!a.same_counts(b)) {
            std::printf("MODE_MISMATCH\n");
            return 2;
        }
        cfg.workers = 4;  // removal + workers > 1 must be a ConfigError (executor.cpp:155)
        try {
            run_parallel(ctx, cfg);
            std::printf("NO_CONFIG_ERROR\n");
            return 3;
        } catch (const ConfigError&) {
        }
        for (int k = 0; k < 36; ++k) std::printf("%s %llu\n", signature(k).c_str(),
                                                 (unsigned long long)a.count_at(k));
    } catch (const std::exception& e) {
        std::printf("ERROR %s\n", e.what());
        return 1;
    }
    return 0;
}
