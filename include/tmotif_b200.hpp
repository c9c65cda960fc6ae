// tmotif_b200.hpp -- header-only C++ mirror of the reference's counting API
// (namespace tmotif, /root/reference/proj/include/tmotif) over the C-ABI in
// tmotif_b200.h.  A reference caller swaps
//     #include "tmotif/executor.hpp"   ->   #include "tmotif_b200.hpp"
//     tmotif::run_parallel(ctx, cfg)   ->   tmotif::b200::run_parallel(ctx, cfg)
// and keeps its RunConfig fields, counter layouts, census order and the
// exception types (ConfigError, CounterOverflowError, ConsistencyError).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <limits>
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
struct ClassificationError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
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

inline std::string signature(int idx) {
    char buf[9];
    check(tm_signature(idx, buf));
    return buf;
}

// signature_index (motifs.hpp:164): position of "sd|sd|sd" in all_signatures()
inline std::optional<std::size_t> signature_index(const std::string& sig) {
    for (int k = 0; k < 36; ++k)
        if (signature(k) == sig) return static_cast<std::size_t>(k);
    return std::nullopt;
}

// CensusMeta (motifs.hpp:172-177)
struct CensusMeta {
    std::string input;
    std::size_t edge_count = 0;
    std::string triangle_mode;
    unsigned workers = 0;
};

// MotifCensus over the 36 signatures in lexicographic order (motifs.hpp:179-201).
struct MotifCensus {
    std::array<std::uint64_t, 36> counts{};
    Timestamp delta = 0;
    CensusMeta meta;
    std::uint64_t count_at(std::size_t k) const { return counts[k]; }
    // count(sig) (motifs.cpp:221-225): ClassificationError for an unknown signature
    std::uint64_t count(const std::string& sig) const {
        const auto k = signature_index(sig);
        if (!k) throw ClassificationError("unknown signature: " + sig);
        return counts[*k];
    }
    // total() (motifs.cpp:239-243): checked sum
    std::uint64_t total() const {
        std::uint64_t s = 0;
        for (auto c : counts) {
            if (s > std::numeric_limits<std::uint64_t>::max() - c) throw CounterOverflowError();
            s += c;
        }
        return s;
    }
    bool same_counts(const MotifCensus& o) const { return counts == o.counts; }
};

struct MotifFilter {
    bool star = true, pair = true, triangle = true;
    bool any_star_pair() const { return star || pair; }
};

// PhaseTimings (executor.hpp:55-65); ingest_ms = host->device copy of the edges
struct PhaseTimings {
    double ingest_ms = 0, index_ms = 0, star_pair_ms = 0, triangle_ms = 0, merge_ms = 0;
    double total_ms() const { return ingest_ms + index_ms + star_pair_ms + triangle_ms + merge_ms; }
};

inline const char* triangle_mode_name(TriangleMode m) { return m == TriangleMode::count_all ? "countall" : "removal"; }

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

// TemporalGraph::degrees (graph.cpp:52-59)
inline std::vector<std::size_t> degrees(const GraphContext& ctx) {
    std::vector<std::uint64_t> d(ctx.node_count());
    if (!d.empty()) check(tm_graph_degrees(ctx.handle(), d.data()));
    return {d.begin(), d.end()};
}

// IndexRange / full_star_range / full_triangle_range (types.hpp:25-33,
// star_engine.hpp:36-38, triangle_engine.hpp:27-29)
struct IndexRange {
    std::size_t begin = 0, end = 0;
    std::size_t size() const { return end > begin ? end - begin : 0; }
    bool empty() const { return end <= begin; }
    bool operator==(const IndexRange& o) const { return begin == o.begin && end == o.end; }
};
inline IndexRange full_star_range(std::size_t s) { return {0, s >= 3 ? s - 2 : 0}; }
inline IndexRange full_triangle_range(std::size_t s) { return {0, s >= 2 ? s - 1 : 0}; }

// SchedulePlan / plan_schedule (executor.hpp:20-33, executor.cpp:23-52): the
// reference's CPU work plan, for callers that drive the per-center API
// (count_*_at_center) themselves.  The device passes do not need it: they
// parallelise over records / wedges, and route the long windows of every
// node, heavy or not, to the cooperative path.
struct SchedulePlan {
    struct HeavyNode {
        NodeId node;
        std::vector<IndexRange> shards;
    };
    std::vector<HeavyNode> heavy;
    std::vector<NodeId> light;
    std::size_t thr_d = 0;
    std::size_t shard_target = 0;
    bool run_star_pair = true;
    bool run_triangle = true;
};
inline SchedulePlan plan_schedule(const GraphContext& ctx, std::size_t thr_d, std::size_t shard_target,
                                  const MotifFilter& motifs) {
    if (shard_target < 1) throw ConfigError("shard_target must be >= 1");
    SchedulePlan plan;
    plan.thr_d = thr_d;
    plan.shard_target = shard_target;
    plan.run_star_pair = motifs.any_star_pair();
    plan.run_triangle = motifs.triangle;
    const auto deg = degrees(ctx);
    for (NodeId u = 0; u < deg.size(); ++u) {
        if (deg[u] > thr_d) {
            SchedulePlan::HeavyNode h{u, {}};
            const IndexRange full = full_star_range(deg[u]);
            for (std::size_t b = full.begin; b < full.end; b += shard_target)
                h.shards.push_back({b, std::min(b + shard_target, full.end)});
            plan.heavy.push_back(std::move(h));
        } else {
            plan.light.push_back(u);
        }
    }
    return plan;
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

// run_parallel (executor.cpp:149-215).  An empty motif filter yields the
// all-zero census, as in the reference.
inline MotifCensus run_parallel(const GraphContext& ctx, const RunConfig& config,
                                PhaseTimings* timings = nullptr) {
    const tm_run_config c = to_c(config);
    MotifCensus out;
    tm_phase_timings t{};
    check(tm_run_parallel(ctx.handle(), &c, nullptr, out.counts.data(), timings ? &t : nullptr));
    if (timings) {
        timings->star_pair_ms = t.star_pair_ms;
        timings->triangle_ms = t.triangle_ms;
        timings->merge_ms = t.merge_ms;
    }
    out.delta = config.delta;
    out.meta.edge_count = ctx.edge_count();
    out.meta.triangle_mode = triangle_mode_name(config.triangle_mode);
    out.meta.workers = config.workers;
    return out;
}

// The whole pipeline for one batch of ingestion-order HOST edges (the
// reference's TemporalGraph::build + GraphContext::build + run_parallel):
// copy-in (ingest_ms), index build (index_ms), both passes and the merge.
inline MotifCensus count_edges(const std::vector<NodeId>& src, const std::vector<NodeId>& dst,
                               const std::vector<Timestamp>& t, std::size_t node_count, const RunConfig& config,
                               PhaseTimings* timings = nullptr) {
    if (src.size() != dst.size() || src.size() != t.size()) throw std::invalid_argument("edge arrays differ in length");
    const tm_run_config c = to_c(config);
    MotifCensus out;
    tm_phase_timings tt{};
    check(tm_count_edges(src.data(), dst.data(), t.data(), src.size(), node_count, 0, nullptr, &c, nullptr,
                         out.counts.data(), timings ? &tt : nullptr));
    if (timings) {
        timings->ingest_ms = tt.ingest_ms;
        timings->index_ms = tt.index_ms;
        timings->star_pair_ms = tt.star_pair_ms;
        timings->triangle_ms = tt.triangle_ms;
        timings->merge_ms = tt.merge_ms;
    }
    out.delta = config.delta;
    out.meta.edge_count = src.size();
    out.meta.triangle_mode = triangle_mode_name(config.triangle_mode);
    out.meta.workers = config.workers;
    return out;
}

}  // namespace tmotif::b200
