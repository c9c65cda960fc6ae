// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference sources
// (/root/reference/proj/src/{graph,indexes,motifs,star_engine,triangle_engine,
// oracle,executor}.cpp), compiled in place by oracle/Makefile into
// oracle/_ref/libtmotif_ref.so.  Used to (a) pin the C restatement in
// oracle/tmotif_oracle.c, (b) generate tests/golden fixtures, and (c) time the
// reference's own std::thread HARE path as bench.py's CPU baseline / reference
// arm.  Nothing here is on the product path.
#include <chrono>
#include <sstream>
#include <cstring>
#include <string>
#include <vector>

#include "tmotif/executor.hpp"
#include "tmotif/graph.hpp"
#include "tmotif/indexes.hpp"
#include "tmotif/oracle.hpp"
#include "tmotif/star_engine.hpp"
#include "tmotif/triangle_engine.hpp"

using namespace tmotif;

namespace {

TemporalGraph make_graph(uint64_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                         const int64_t* t) {
    std::vector<std::string> ids(n);
    for (uint64_t u = 0; u < n; ++u) ids[u] = std::to_string(u);
    std::vector<TemporalGraph::RawEdge> edges(m);
    for (uint64_t i = 0; i < m; ++i) edges[i] = {src[i], dst[i], t[i]};
    return TemporalGraph::build(std::move(ids), edges);
}

void copy_cells(std::span<const std::uint64_t> cells, uint64_t* out) {
    if (out) std::memcpy(out, cells.data(), cells.size() * sizeof(uint64_t));
}

int classify_error() {
    try {
        throw;
    } catch (const CounterOverflowError&) {
        return 3;
    } catch (const ConfigError&) {
        return 4;
    } catch (const ConsistencyError&) {
        return 5;
    } catch (...) {
        return 1;
    }
}

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
        .count();
}

}  // namespace

extern "C" {

// parse_edge_list (graph.cpp:73) over a text buffer.  Edges are returned in
// ingestion order (edge i at index ordinal); ids joined by '\n'.  Outputs:
// counts[0..3) = n, m, dropped; the arrays must hold one entry per line and
// `ids` len + 1 bytes.  Returns 0, or 2 with err_line / err_msg (<= 511
// chars) for a ParseError.
int ref_parse_edge_list(const char* text, uint64_t len, int drop_self_loops, uint64_t* counts,
                        uint32_t* src, uint32_t* dst, int64_t* t, char* ids, uint64_t* ids_len,
                        uint64_t* err_line, char* err_msg) {
    try {
        std::istringstream in(std::string(text, len));
        ParseOptions opt;
        opt.drop_self_loops = drop_self_loops != 0;
        TemporalGraph g = parse_edge_list(in, opt);
        counts[0] = g.node_count();
        counts[1] = g.edge_count();
        counts[2] = g.dropped_self_loops();
        for (const TemporalEdge& e : g.edges()) {
            src[e.ordinal] = e.src;
            dst[e.ordinal] = e.dst;
            t[e.ordinal] = e.t;
        }
        std::string joined;
        for (std::size_t u = 0; u < g.node_count(); ++u) {
            if (u) joined += '\n';
            joined += g.node_id(static_cast<NodeId>(u));
        }
        std::memcpy(ids, joined.data(), joined.size());
        *ids_len = joined.size();
        return 0;
    } catch (const ParseError& e) {
        *err_line = e.line();
        std::strncpy(err_msg, e.what(), 511);
        err_msg[511] = 0;
        return 2;
    }
}

struct ref_ctx {
    GraphContext ctx;
};

ref_ctx* ref_build(uint64_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                   const int64_t* t) {
    try {
        return new ref_ctx{GraphContext::build(make_graph(n, m, src, dst, t))};
    } catch (...) {
        return nullptr;
    }
}

void ref_free(ref_ctx* c) { delete c; }

// Raw counters of the sequential composition (star_engine.cpp:129,
// triangle_engine.cpp:64).
int ref_counters(const ref_ctx* c, int64_t delta, int removal, uint64_t* star, uint64_t* pair,
                 uint64_t* tri) {
    try {
        CenterStarResult sp = count_star_pair(c->ctx.sequences, delta);
        TriCounter tr = count_triangles(c->ctx.sequences, c->ctx.pairs, delta,
                                        removal ? TriangleMode::removal : TriangleMode::count_all);
        copy_cells(sp.star.cells(), star);
        copy_cells(sp.pair.cells(), pair);
        copy_cells(tr.cells(), tri);
        return 0;
    } catch (...) {
        return classify_error();
    }
}

int ref_star_pair_at_center(const ref_ctx* c, uint32_t u, int64_t delta, uint64_t begin,
                            uint64_t end, uint64_t* star, uint64_t* pair) {
    try {
        CenterStarResult r = count_star_pair_at_center(c->ctx.sequences, u, delta, {begin, end});
        copy_cells(r.star.cells(), star);
        copy_cells(r.pair.cells(), pair);
        return 0;
    } catch (...) {
        return classify_error();
    }
}

int ref_triangles_at_center(const ref_ctx* c, uint32_t u, int64_t delta, uint64_t begin,
                            uint64_t end, const uint8_t* live, uint64_t* tri) {
    try {
        std::vector<std::uint8_t> mask;
        if (live) mask.assign(live, live + c->ctx.graph.node_count());
        TriCounter r = count_triangles_at_center(c->ctx.sequences, c->ctx.pairs, u, delta,
                                                 {begin, end}, live ? &mask : nullptr);
        copy_cells(r.cells(), tri);
        return 0;
    } catch (...) {
        return classify_error();
    }
}

// run_parallel (executor.cpp:149).  thr < 0: auto; thr == INT64_MAX: no sharding.
int ref_run_parallel(const ref_ctx* c, int64_t delta, unsigned workers, int64_t thr, int removal,
                     int motif_mask, uint64_t shard_target, uint64_t* census) {
    try {
        RunConfig cfg;
        cfg.delta = delta;
        cfg.workers = workers;
        if (thr >= 0) cfg.degree_threshold = static_cast<std::size_t>(thr);
        if (thr == INT64_MAX) cfg.degree_threshold = static_cast<std::size_t>(-1);
        cfg.triangle_mode = removal ? TriangleMode::removal : TriangleMode::count_all;
        cfg.motifs = {(motif_mask & 1) != 0, (motif_mask & 2) != 0, (motif_mask & 4) != 0};
        if (shard_target) cfg.shard_target = shard_target;
        MotifCensus mc = run_parallel(c->ctx, cfg);
        for (std::size_t k = 0; k < 36; ++k) census[k] = mc.count_at(k);
        return 0;
    } catch (...) {
        return classify_error();
    }
}

int ref_oracle_census(const ref_ctx* c, int64_t delta, uint64_t* census) {
    try {
        MotifCensus mc = oracle_census(c->ctx.graph, delta);
        for (std::size_t k = 0; k < 36; ++k) census[k] = mc.count_at(k);
        return 0;
    } catch (...) {
        return classify_error();
    }
}

uint64_t ref_auto_degree_threshold(const ref_ctx* c) {
    return auto_degree_threshold(c->ctx.graph);
}

int ref_signature(int idx, char* out) {
    auto all = all_signatures();
    if (idx < 0 || idx >= static_cast<int>(all.size())) return 1;
    std::string s = all[idx].to_string();
    std::memcpy(out, s.c_str(), 9);
    return 0;
}

// Full reference pipeline from raw ingestion-order arrays: TemporalGraph::build
// + GraphContext::build + run_parallel.  Reports build / count wall times.
int ref_pipeline(uint64_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                 const int64_t* t, int64_t delta, unsigned workers, uint64_t* census,
                 double* ms_build, double* ms_count) {
    try {
        std::vector<std::string> ids(n);
        for (uint64_t u = 0; u < n; ++u) ids[u] = std::to_string(u);
        std::vector<TemporalGraph::RawEdge> edges(m);
        for (uint64_t i = 0; i < m; ++i) edges[i] = {src[i], dst[i], t[i]};
        auto t0 = std::chrono::steady_clock::now();
        GraphContext ctx = GraphContext::build(TemporalGraph::build(std::move(ids), edges));
        if (ms_build) *ms_build = ms_since(t0);
        t0 = std::chrono::steady_clock::now();
        RunConfig cfg;
        cfg.delta = delta;
        cfg.workers = workers;
        MotifCensus mc = run_parallel(ctx, cfg);
        if (ms_count) *ms_count = ms_since(t0);
        for (std::size_t k = 0; k < 36; ++k) census[k] = mc.count_at(k);
        return 0;
    } catch (...) {
        return classify_error();
    }
}

// generate_random_graph (graph.cpp:140) in ingestion (ordinal) order.
int ref_generate_random_graph(uint64_t nodes, uint64_t m, int64_t t_max, uint64_t seed,
                              uint32_t* src, uint32_t* dst, int64_t* t) {
    try {
        TemporalGraph g = generate_random_graph(nodes, m, t_max, seed);
        for (const TemporalEdge& e : g.edges()) {
            src[e.ordinal] = e.src;
            dst[e.ordinal] = e.dst;
            t[e.ordinal] = e.t;
        }
        return 0;
    } catch (...) {
        return 1;
    }
}

}  // extern "C"
