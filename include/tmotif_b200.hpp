// tmotif_b200.hpp -- header-only C++ mirror of the reference's counting API
// (namespace tmotif, /root/reference/proj/include/tmotif) over the C-ABI in
// tmotif_b200.h.  A reference caller swaps
//     #include "tmotif/executor.hpp"   ->   #include "tmotif_b200.hpp"
//     tmotif::run_parallel(ctx, cfg)   ->   tmotif::b200::run_parallel(ctx, cfg)
// and keeps its RunConfig fields, counter layouts, census order and the
// exception types (ConfigError, CounterOverflowError, ConsistencyError).
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "tmotif_b200.h"

namespace tmotif::b200 {

using NodeId = std::uint32_t;
using Timestamp = std::int64_t;

enum class Direction : std::uint8_t { outward = 0, inward = 1 };           // types.hpp:15
enum class TriangleMode : std::uint8_t { count_all = 0, removal = 1 };     // motifs.hpp:35-38

struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CounterOverflowError : std::runtime_error {
    CounterOverflowError() : std::runtime_error("motif counter overflow") {}
};
struct ConsistencyError : std::logic_error { using std::logic_error::logic_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };
// types.hpp:35-44: "line N: what", line() = N
struct ParseError : std::runtime_error {
    ParseError(std::size_t line, const std::string& what_full) : std::runtime_error(what_full), line_(line) {}
    std::size_t line() const { return line_; }

private:
    std::size_t line_;
};

inline void check(int rc) {
    switch (rc) {
        case TM_OK: return;
        case TM_ERR_PARSE: throw ParseError(tm_parse_error_line(), tm_last_error());
        case TM_ERR_INVALID: throw std::invalid_argument(tm_last_error());
        case TM_ERR_OVERFLOW: throw CounterOverflowError();
        case TM_ERR_CONFIG: throw ConfigError(tm_last_error());
        case TM_ERR_CONSISTENCY: throw ConsistencyError(tm_last_error());
        default: throw DeviceError(tm_last_error());
    }
}

// Counter arrays with the reference's cell layout (motifs.hpp:72-135).
struct StarCounter { std::array<std::uint64_t, 24> cells{}; };
struct PairCounter { std::array<std::uint64_t, 8> cells{}; };
struct TriCounter { std::array<std::uint64_t, 24> cells{}; };
struct CenterStarResult { StarCounter star; PairCounter pair; };

// MotifCensus over the 36 signatures in lexicographic order (motifs.hpp:168).
struct MotifCensus {
    std::array<std::uint64_t, 36> counts{};
    Timestamp delta = 0;
    std::uint64_t count_at(std::size_t k) const { return counts[k]; }
    std::uint64_t total() const {
        std::uint64_t s = 0;
        for (auto c : counts) s += c;
        return s;
    }
    bool same_counts(const MotifCensus& o) const { return counts == o.counts; }
};

inline std::string signature(int idx) {
    char buf[9];
    check(tm_signature(idx, buf));
    return buf;
}

struct MotifFilter { bool star = true, pair = true, triangle = true; };

// RunConfig (executor.hpp:36-46).
struct RunConfig {
    Timestamp delta = 0;
    unsigned workers = 1;
    std::optional<std::size_t> degree_threshold;
    TriangleMode triangle_mode = TriangleMode::count_all;
    MotifFilter motifs;
    std::size_t shard_target = 4096;
    std::size_t light_batch = 64;
};

// parse_edge_list / load_edge_list (graph.hpp:60-70) on the GPU: the parsed
// edges stay in device memory (ingestion order) for GraphContext below.
struct ParseOptions { bool drop_self_loops = true; };
class EdgeList {
public:
    explicit EdgeList(const std::string& text, const ParseOptions& o = {}) {
        check(tm_parse_edge_list(text.data(), text.size(), 0, o.drop_self_loops ? 1 : 0, nullptr, &el_));
        check(tm_edge_list_info(el_, &n_, &m_, &dropped_, &id_bytes_));
    }
    ~EdgeList() { tm_edge_list_free(el_); }
    EdgeList(const EdgeList&) = delete;
    EdgeList& operator=(const EdgeList&) = delete;
    std::size_t node_count() const { return n_; }
    std::size_t edge_count() const { return m_; }
    std::size_t dropped_self_loops() const { return dropped_; }
    // node_id(u) for every u (graph.hpp:46), in id order
    std::vector<std::string> node_ids() const {
        std::string all(id_bytes_, '\0');
        check(tm_edge_list_copy(el_, nullptr, nullptr, nullptr, all.data()));
        std::vector<std::string> out;
        std::size_t b = 0;
        for (std::size_t u = 0; u < n_; ++u) {
            const std::size_t e = all.find('\n', b);
            out.push_back(all.substr(b, e == std::string::npos ? std::string::npos : e - b));
            b = e + 1;
        }
        return out;
    }
    const tm_edge_list* handle() const { return el_; }

private:
    tm_edge_list* el_ = nullptr;
    std::uint64_t n_ = 0, m_ = 0, dropped_ = 0, id_bytes_ = 0;
};
inline EdgeList parse_edge_list(const std::string& text, const ParseOptions& o = {}) { return EdgeList(text, o); }

// Device-resident GraphContext (indexes.hpp:95-105): built from edges in
// ingestion order; the (t, ordinal) sort and all indexes are built on the GPU.
class GraphContext {
public:
    explicit GraphContext(const EdgeList& el) {
        const std::uint32_t *s, *d;
        const std::int64_t* t;
        check(tm_edge_list_device_arrays(el.handle(), &s, &d, &t));
        check(tm_graph_build(s, d, t, el.edge_count(), el.node_count(), 1, nullptr, &g_));
    }
    GraphContext(const std::vector<NodeId>& src, const std::vector<NodeId>& dst,
                 const std::vector<Timestamp>& t, std::size_t node_count) {
        check(tm_graph_build(src.data(), dst.data(), t.data(), src.size(), node_count, 0, nullptr,
                             &g_));
    }
    ~GraphContext() { tm_graph_free(g_); }
    GraphContext(const GraphContext&) = delete;
    GraphContext& operator=(const GraphContext&) = delete;
    tm_graph* handle() const { return g_; }
    std::size_t node_count() const { return tm_graph_node_count(g_); }
    std::size_t edge_count() const { return tm_graph_edge_count(g_); }

private:
    tm_graph* g_ = nullptr;
};

inline CenterStarResult count_star_pair(const GraphContext& ctx, Timestamp delta) {
    CenterStarResult r;
    check(tm_count_star_pair(ctx.handle(), delta, r.star.cells.data(), r.pair.cells.data()));
    return r;
}

inline CenterStarResult count_star_pair_at_center(const GraphContext& ctx, NodeId u, Timestamp delta,
                                                  std::size_t begin, std::size_t end) {
    CenterStarResult r;
    const std::uint64_t b = begin, e = end;
    check(tm_count_star_pair_items(ctx.handle(), delta, 1, &u, &b, &e, r.star.cells.data(),
                                   r.pair.cells.data()));
    return r;
}

inline TriCounter count_triangles(const GraphContext& ctx, Timestamp delta, TriangleMode mode) {
    TriCounter r;
    check(tm_count_triangles(ctx.handle(), delta, static_cast<int>(mode), r.cells.data()));
    return r;
}

inline TriCounter count_triangles_at_center(const GraphContext& ctx, NodeId u, Timestamp delta,
                                            std::size_t begin, std::size_t end,
                                            const std::vector<std::uint8_t>* live = nullptr) {
    TriCounter r;
    const std::uint64_t b = begin, e = end;
    check(tm_count_triangles_items(ctx.handle(), delta, 1, &u, &b, &e, live ? live->data() : nullptr,
                                   r.cells.data()));
    return r;
}

inline MotifCensus merge_census(const StarCounter& s, const PairCounter& p, const TriCounter& t,
                                TriangleMode mode) {
    MotifCensus c;
    check(tm_merge_census(s.cells.data(), p.cells.data(), t.cells.data(), static_cast<int>(mode),
                          c.counts.data()));
    return c;
}

inline std::size_t auto_degree_threshold(const GraphContext& ctx) {
    std::uint64_t v = 0;
    check(tm_auto_degree_threshold(ctx.handle(), &v));
    return v;
}

inline tm_run_config to_c(const RunConfig& c, std::uint32_t cb = 0, std::uint32_t ce = 0) {
    tm_run_config r{};
    r.delta = c.delta;
    r.workers = c.workers;
    r.degree_threshold = c.degree_threshold ? static_cast<std::int64_t>(*c.degree_threshold) : -1;
    r.triangle_mode = static_cast<std::int32_t>(c.triangle_mode);
    r.motifs = (c.motifs.star ? TM_MOTIF_STAR : 0u) | (c.motifs.pair ? TM_MOTIF_PAIR : 0u) |
               (c.motifs.triangle ? TM_MOTIF_TRIANGLE : 0u);
    r.shard_target = c.shard_target;
    r.center_begin = cb;
    r.center_end = ce;
    r.has_first_edge_t_end = 0;
    r.first_edge_t_end = 0;
    return r;
}

// run_parallel (executor.cpp:149-215).
inline MotifCensus run_parallel(const GraphContext& ctx, const RunConfig& config,
                                tm_phase_timings* timings = nullptr) {
    if (!config.motifs.star && !config.motifs.pair && !config.motifs.triangle)
        throw std::invalid_argument("empty motif filter");
    const tm_run_config c = to_c(config);
    MotifCensus out;
    check(tm_run_parallel(ctx.handle(), &c, nullptr, out.counts.data(), timings));
    out.delta = config.delta;
    return out;
}

}  // namespace tmotif::b200
