/*
 * tmotif_b200.h -- C-ABI of the B200-native temporal motif counter.
 *
 * Drop-in boundary for the reference's counting path (arXiv 2204.09236
 * FAST-Star / FAST-Tri / HARE; reference tree /root/reference/proj).  Every
 * entry point takes plain pointers and sizes; no torch or CUDA C++ types
 * cross this line (streams are passed as opaque `void*` cudaStream_t).
 *
 * Counter layouts are the reference's, cell-for-cell:
 *   star[24]  index ((type*2 + d1)*2 + d2)*2 + d3   (motifs.hpp:78-83)
 *   pair[8]   index (d1*2 + d2)*2 + d3              (motifs.hpp:103-106)
 *   tri[24]   index ((type*2 + di)*2 + dj)*2 + dk   (motifs.hpp:127-131)
 *   census[36] in lexicographic signature order      (motifs.hpp:159-161)
 * with Direction outward = 0, inward = 1 (types.hpp:15).
 *
 * Error codes: 2 / 3 / 4 are the reference CLI's exit codes for the same
 * exception (exit_parse, exit_overflow, exit_config; tmotif_main.cpp:20-30,
 * 283-294).  The CLI folds std::invalid_argument and ConsistencyError (a
 * std::logic_error) into exit_usage = 1 through its std::exception catch; the
 * C-ABI keeps them apart (1 and 10) so a binding raises the precise type.
 * Codes 5-7 are the CLI's exit_too_large / exit_mismatch /
 * exit_nondeterministic (oracle, verify and bench subcommands, not on this
 * path) and are never returned; 8+ are this library's own.
 */
#ifndef TMOTIF_B200_H
#define TMOTIF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TM_OK 0
#define TM_ERR_INVALID 1     /* std::invalid_argument (graph.cpp:20,29,32)      */
#define TM_ERR_PARSE 2       /* ParseError (types.hpp:35), CLI exit_parse        */
#define TM_ERR_OVERFLOW 3    /* CounterOverflowError (types.hpp:50): any counter
                                cell, class sum or census cell above 2^64 - 1
                                (cells are summed exactly on the device)      */
#define TM_ERR_CONFIG 4      /* ConfigError (types.hpp:46, executor.cpp:151-156)  */
#define TM_ERR_CONSISTENCY 10 /* ConsistencyError (types.hpp:55, motifs.cpp:254)  */
#define TM_ERR_CUDA 8        /* no device / CUDA failure: the path never falls back */
#define TM_ERR_LIMIT 9       /* graph exceeds the 32-bit position layout         */

#define TM_TRI_COUNT_ALL 0 /* TriangleMode::count_all (motifs.hpp:36) */
#define TM_TRI_REMOVAL 1   /* TriangleMode::removal   (motifs.hpp:37) */

#define TM_MOTIF_STAR 1u
#define TM_MOTIF_PAIR 2u
#define TM_MOTIF_TRIANGLE 4u

typedef struct tm_graph tm_graph; /* device-resident GraphContext (indexes.hpp:95-105) */

typedef struct tm_counters {
    uint64_t star[24];
    uint64_t pair[8];
    uint64_t tri[24];
} tm_counters;

/* RunConfig (executor.hpp:36-46) plus a center partition for multi-GPU. */
typedef struct tm_run_config {
    int64_t delta;
    uint32_t workers;          /* kept for the removal-mode check only            */
    int64_t degree_threshold;  /* < 0: auto top-20 rule (executor.cpp:15)          */
    int32_t triangle_mode;     /* TM_TRI_COUNT_ALL | TM_TRI_REMOVAL                */
    uint32_t motifs;           /* TM_MOTIF_* bit set (MotifFilter); 0 = the empty
                                  filter: nothing runs, the census is all zero
                                  (executor.cpp:28-29)                             */
    uint64_t shard_target;     /* accepted for API parity; semantics-free           */
    uint32_t center_begin;     /* center partition [begin, end); end == 0: all      */
    uint32_t center_end;
    /* time-slice partition: when nonzero, count only the instances whose
     * earliest edge (in (t, ordinal) order) has t < first_edge_t_end.  A rank
     * that builds the edges with t in [lo, hi + delta) and counts with
     * first_edge_t_end = hi owns exactly the instances starting in [lo, hi). */
    int32_t has_first_edge_t_end;
    int64_t first_edge_t_end;
} tm_run_config;

/* PhaseTimings (executor.hpp:55-65); device-event times in ms.  ingest_ms is
 * the host->device copy of the edge arrays (0 for device pointers). */
typedef struct tm_phase_timings {
    double ingest_ms;
    double index_ms;
    double star_pair_ms;
    double triangle_ms;
    double merge_ms;
} tm_phase_timings;

/* ---- graph construction --------------------------------------------------
 * Replaces TemporalGraph::build (graph.cpp:13-44) + GraphContext::build
 * (indexes.hpp:99-103): edges arrive in ingestion order (ordinal = index),
 * self-loops / out-of-range endpoints are rejected with TM_ERR_INVALID.
 * `device_ptrs` != 0: src/dst/t are device pointers, else host pointers
 * (copied in with cudaMemcpyAsync).  `stream` may be NULL (library stream). */
int tm_graph_build(const uint32_t* src, const uint32_t* dst, const int64_t* t, uint64_t m,
                   uint64_t n, int device_ptrs, void* stream, tm_graph** out);
void tm_graph_free(tm_graph* g);
uint64_t tm_graph_node_count(const tm_graph* g);
uint64_t tm_graph_edge_count(const tm_graph* g);
void* tm_graph_stream(const tm_graph* g);

/* TemporalGraph::degrees (graph.cpp:52-59); out_host has n entries. */
int tm_graph_degrees(const tm_graph* g, uint64_t* out_host);
/* NodeSequenceIndex::sequence (indexes.hpp:28-30) copied to host; len = S_u. */
int tm_graph_sequence(const tm_graph* g, uint32_t u, int64_t* t, uint64_t* ordinal,
                      uint32_t* other, uint8_t* dir, uint64_t cap, uint64_t* len);
/* PairEdgeIndex::edges_in_window (indexes.cpp:75-85). */
int tm_pair_window(const tm_graph* g, uint32_t v, uint32_t w, int64_t lo, int64_t hi,
                   int64_t* t, uint64_t* ordinal, uint8_t* dir_rel_v, uint64_t cap,
                   uint64_t* len);
/* auto_degree_threshold (executor.cpp:15-21). */
int tm_auto_degree_threshold(const tm_graph* g, uint64_t* out);

/* ---- counting ----------------------------------------------------------- */
/* count_star_pair (star_engine.cpp:129-136). */
int tm_count_star_pair(tm_graph* g, int64_t delta, uint64_t* star24, uint64_t* pair8);
/* count_triangles (triangle_engine.cpp:64-84): mode TM_TRI_*. */
int tm_count_triangles(tm_graph* g, int64_t delta, int mode, uint64_t* tri24);
/* count_star_pair_at_center (star_engine.cpp:64) batched over work items
 * (node, [begin, end)) -- the HARE plan items (executor.cpp:31-52). */
int tm_count_star_pair_items(tm_graph* g, int64_t delta, uint64_t n_items, const uint32_t* nodes,
                             const uint64_t* begin, const uint64_t* end, uint64_t* star_out,
                             uint64_t* pair_out);
/* count_triangles_at_center (triangle_engine.cpp:20) batched; live: host
 * array of n bytes or NULL (removal-mode live mask). */
int tm_count_triangles_items(tm_graph* g, int64_t delta, uint64_t n_items, const uint32_t* nodes,
                             const uint64_t* begin, const uint64_t* end, const uint8_t* live,
                             uint64_t* tri_out);
/* run_parallel (executor.cpp:149-215).  With a center or time-slice partition
 * the raw counters are partial sums and census is left zeroed (merge after the
 * all-reduce); for the full graph census holds merge_census(raw). */
int tm_run_parallel(tm_graph* g, const tm_run_config* cfg, tm_counters* raw, uint64_t* census36,
                    tm_phase_timings* timings);
/* Whole pipeline for one step: build + run_parallel + free. */
int tm_count_edges(const uint32_t* src, const uint32_t* dst, const int64_t* t, uint64_t m,
                   uint64_t n, int device_ptrs, void* stream, const tm_run_config* cfg,
                   tm_counters* raw, uint64_t* census36, tm_phase_timings* timings);
/* Pipelined variant of tm_count_edges for callers that stream batches from
 * host memory (serving): enqueues the host->device copy of the edge arrays on
 * a copy stream, the census on `stream` once its copy has landed, and the
 * counter read-back, then returns a ticket without waiting, so the copy of
 * the next batch overlaps this batch's census.  Host arrays should be pinned
 * for the copy to be asynchronous.  At most two batches per host thread are
 * staged at a time (a third call first completes the oldest, whose result is
 * kept for its tm_count_edges_wait).  Results are those of tm_count_edges on
 * the same arrays; errors (invalid edges, ...) are reported by the wait. */
int tm_count_edges_async(const uint32_t* src, const uint32_t* dst, const int64_t* t, uint64_t m,
                         uint64_t n, void* stream, const tm_run_config* cfg, uint64_t* ticket);
/* Input bytes the most recently submitted tm_count_edges_async batch puts on
 * the host->device link: 16 per edge, or 10 per edge (+ 8 per 4096 edges) /
 * 12 per edge (+ 8 per 65536 edges) when the batch's timestamps travel packed
 * -- batches of >= 2^24 edges above the graph-replay size are rewritten by host
 * worker threads (TM_HOST_THREADS, default all cores up to 32) as per-block i64
 * bases + u16 offsets (u32 offsets from the first batch on that has a block of
 * 4096 edges spanning 2^16 or more, which itself takes a plain copy of t;
 * TM_H2D_PACK16=0 starts with u32) into pinned staging while src / dst are on
 * the wire, and expanded on the device (TM_H2D_PACK=0 copies t as it is).
 * Results are identical either way. */
int tm_async_h2d_bytes(uint64_t* bytes);
/* Blocks until the ticket's census is done and returns it (once per ticket). */
int tm_count_edges_wait(uint64_t ticket, tm_counters* raw, uint64_t* census36);
/* One rank's share of a time-sliced census (multi-GPU without a replicated
 * index build): the edges with t in [t_lo, t_hi + delta) are compacted on the
 * GPU (ingestion order kept), indexed, and counted for the instances whose
 * earliest edge has t in [t_lo, t_hi).  has_lo / has_hi = 0 leave the first /
 * last slice open.  Summing raw over slices that partition the time axis gives
 * the whole graph's counters exactly. */
int tm_count_edges_time_slice(const uint32_t* src, const uint32_t* dst, const int64_t* t, uint64_t m,
                              uint64_t n, int device_ptrs, void* stream, const tm_run_config* cfg,
                              int has_lo, int64_t t_lo, int has_hi, int64_t t_hi, tm_counters* raw,
                              tm_phase_timings* timings);
/* Degree-cost balanced center partition for rank `rank` of `world`. */
int tm_partition_centers(const tm_graph* g, uint32_t world, uint32_t rank, uint32_t* begin,
                         uint32_t* end);

/* ---- edge-list text (the reader in front of the path) -------------------
 * parse_edge_list (graph.cpp:73-116) on the GPU: whitespace-separated
 * "SRC DST T" lines, '#'-prefixed and blank lines skipped, CRLF accepted,
 * fields past the third ignored, node ids = arbitrary tokens mapped to dense
 * indices in order of first appearance among retained edges, self-loops
 * dropped and tallied (drop_self_loops = 1) or rejected.  Errors return
 * TM_ERR_PARSE with the reference's ParseError text ("line N: ...") in
 * tm_last_error and N in tm_parse_error_line.  The edge arrays stay on the
 * device in ingestion order, ready for tm_graph_build / tm_count_edges with
 * device_ptrs = 1 (TemporalGraph::build's (t, ordinal) sort happens there). */
typedef struct tm_edge_list tm_edge_list;
int tm_parse_edge_list(const char* text, uint64_t bytes, int device_text, int drop_self_loops, void* stream,
                       tm_edge_list** out);
/* node_count, edge_count, dropped_self_loops (graph.hpp:44-54) and the size
 * of the '\n'-joined node-id tokens in id order. */
int tm_edge_list_info(const tm_edge_list* el, uint64_t* nodes, uint64_t* edges, uint64_t* dropped_self_loops,
                      uint64_t* id_bytes);
int tm_edge_list_device_arrays(const tm_edge_list* el, const uint32_t** src, const uint32_t** dst,
                               const int64_t** t);
/* host copies; any NULL output is skipped.  ids: id_bytes bytes, tokens in
 * id order joined by '\n' (TemporalGraph::node_id, graph.hpp:46). */
int tm_edge_list_copy(const tm_edge_list* el, uint32_t* src, uint32_t* dst, int64_t* t, char* ids);
uint64_t tm_parse_error_line(void);
/* write_edge_list (graph.cpp:170-175) for graphs whose node ids are their
 * decimal indices (generate_random_graph's naming): "SRC DST T\n" per edge
 * in the order given (the reference writes graph.edges(), i.e. (t, ordinal)
 * order: pass time-ordered edges for byte-identical output).  With out == NULL only *bytes is set; otherwise out
 * (host, or device when device_out) receives *bytes bytes. */
int tm_write_edge_list(const uint32_t* src, const uint32_t* dst, const int64_t* t, uint64_t m, int device_ptrs,
                       void* stream, char* out, int device_out, uint64_t* bytes);
void tm_edge_list_free(tm_edge_list* el);

/* ---- taxonomy (host only) ----------------------------------------------- */
/* merge_census (motifs.cpp:233-281). */
int tm_merge_census(const uint64_t* star24, const uint64_t* pair8, const uint64_t* tri24,
                    int mode, uint64_t* census36);
/* all_signatures()[idx] (motifs.cpp:196) as "sd|sd|sd" + NUL. */
int tm_signature(int idx, char* out9);
/* signature index of a counter cell; kind 0 star, 1 pair, 2 tri. */
int tm_cell_signature(int kind, int cell);
/* label_for_signature (motifs.cpp:207). */
int tm_signature_label(int idx, char* out16);
/* generate_random_graph (graph.cpp:140-168), ingestion order. */
int tm_generate_random_graph(uint64_t nodes, uint64_t m, int64_t t_max, uint64_t seed,
                             uint32_t* src, uint32_t* dst, int64_t* t);

/* ---- diagnostics -------------------------------------------------------- */
/* Work counters of the graph's last counting run: [0] star first-edge
 * candidates, [1] star third-edge candidates, [2] short-window wedges,
 * [3] long-window first edges, [4] long-window wedges, [5..7] reserved. */
int tm_run_stats(const tm_graph* g, uint64_t* out8);
const char* tm_last_error(void);
/* Test hook (this host thread, eager runs): every raw star/pair accumulator
 * cell starts at `bias` instead of 0, so Pair = bias + count while Star is
 * unchanged -- exercises the exact 2^64 overflow detection.  0 = off. */
void tm_debug_acc_bias(uint64_t bias);
/* Number of this library's kernels launched since load. */
uint64_t tm_kernel_launches(void);
/* Per-kernel CUDA-event timing on the launching stream. */
void tm_kernel_timing_enable(int on);
void tm_kernel_timing_reset(void);
/* Aggregated device time of kernels whose name matches `name` exactly. */
int tm_kernel_timing_get(const char* name, double* total_ms, uint64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* TMOTIF_B200_H */
