// tm_capi.cu -- extern "C" boundary (include/tmotif_b200.h) and host logic:
// run_parallel orchestration (executor.cpp:149-215), census merge
// (motifs.cpp:233-281), signature taxonomy (motifs.cpp:49-123, 145-219).
// There is no CPU counting path here: every count comes from the kernels in
// tm_star.cu / tm_tri.cu, and a missing device is reported as TM_ERR_CUDA.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tmotif_b200.h"
#include "tm_primitives.cuh"

struct tm_graph {
    tmb::DeviceGraph g;
    std::vector<uint32_t> h_off;  // lazily mirrored CSR offsets
};
struct tm_edge_list {
    tmb::ParsedEdges P;
    uint64_t id_bytes = 0;
    bool own_stream = false;
};

namespace tmb {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_timing{0};
std::mutex g_timing_mu;
struct PendingEv {
    std::string name;
    cudaEvent_t a, b;
};
std::vector<PendingEv> g_pending;
std::map<std::string, std::pair<double, uint64_t>> g_ktotals;
}  // namespace

void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        throw tm_error(TM_ERR_CUDA, std::string(cudaGetErrorString(e)) + " at " + file + ":" +
                                        std::to_string(line) + " (" + what + ")");
    }
}

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// With timing on, every launch runs alone (device synchronised on both
// sides), so a kernel's time is its own and not shared with side-stream work.
KernelScope::KernelScope(const char* n, cudaStream_t s) : name(n), stream(s), ev0(nullptr) {
    if (g_timing.load(std::memory_order_relaxed)) {
        cudaDeviceSynchronize();
        cudaEvent_t e;
        if (cudaEventCreate(&e) == cudaSuccess) {
            cudaEventRecord(e, s);
            ev0 = e;
        }
    }
}
KernelScope::~KernelScope() {
    if (!ev0) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, stream);
    cudaDeviceSynchronize();
    std::lock_guard<std::mutex> lk(g_timing_mu);
    g_pending.push_back({name, static_cast<cudaEvent_t>(ev0), e});
}

int sm_count() {
    static int cached = 0;
    if (!cached) {
        int dev = 0;
        cudaGetDevice(&dev);
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached = v > 0 ? v : 148;
    }
    return cached;
}

// ---------------------------------------------------------------------------
// taxonomy (host)
namespace {

struct Universe {
    std::vector<std::string> all;  // 36, lexicographic
    int star_sig[24], pair_sig[8], tri_sig[24];
};

std::string canonical(const uint32_t e[3][2]) {
    uint32_t seen[3];
    int distinct = 0;
    std::string s = "12|12|12";
    for (int k = 0; k < 3; ++k)
        for (int side = 0; side < 2; ++side) {
            int lab = 0;
            for (int q = 0; q < distinct; ++q)
                if (seen[q] == e[k][side]) lab = q + 1;
            if (!lab) {
                seen[distinct++] = e[k][side];
                lab = distinct;
            }
            s[3 * k + side] = char('0' + lab);
        }
    return s;
}
void orient(int d, uint32_t from, uint32_t to, uint32_t out[2]) {
    out[0] = d ? to : from;
    out[1] = d ? from : to;
}
std::string star_sig(int type, int d1, int d2, int d3) {
    uint32_t e[3][2];
    const int d[3] = {d1, d2, d3};
    for (int p = 0; p < 3; ++p) orient(d[p], 0, p == type ? 2 : 1, e[p]);
    return canonical(e);
}
std::string pair_sig(int d1, int d2, int d3) {
    uint32_t e[3][2];
    orient(d1, 0, 1, e[0]);
    orient(d2, 0, 1, e[1]);
    orient(d3, 0, 1, e[2]);
    return canonical(e);
}
std::string tri_sig(int type, int di, int dj, int dk) {
    uint32_t ei[2], ej[2], ek[2];
    orient(di, 0, 1, ei);
    orient(dj, 0, 2, ej);
    orient(dk, 1, 2, ek);
    const uint32_t* ord[3];
    if (type == 0) { ord[0] = ek; ord[1] = ei; ord[2] = ej; }
    else if (type == 1) { ord[0] = ei; ord[1] = ek; ord[2] = ej; }
    else { ord[0] = ei; ord[1] = ej; ord[2] = ek; }
    uint32_t e[3][2];
    for (int k = 0; k < 3; ++k) { e[k][0] = ord[k][0]; e[k][1] = ord[k][1]; }
    return canonical(e);
}

const Universe& universe() {
    static const Universe U = [] {
        Universe u;
        std::set<std::string> all;
        std::string st[24], pr[8], tr[24];
        for (int c = 0; c < 24; ++c) all.insert(st[c] = star_sig(c >> 3, (c >> 2) & 1, (c >> 1) & 1, c & 1));
        for (int c = 0; c < 8; ++c) all.insert(pr[c] = pair_sig(c >> 2, (c >> 1) & 1, c & 1));
        for (int c = 0; c < 24; ++c) all.insert(tr[c] = tri_sig(c >> 3, (c >> 2) & 1, (c >> 1) & 1, c & 1));
        u.all.assign(all.begin(), all.end());
        auto idx = [&](const std::string& s) {
            return int(std::lower_bound(u.all.begin(), u.all.end(), s) - u.all.begin());
        };
        for (int c = 0; c < 24; ++c) u.star_sig[c] = idx(st[c]);
        for (int c = 0; c < 8; ++c) u.pair_sig[c] = idx(pr[c]);
        for (int c = 0; c < 24; ++c) u.tri_sig[c] = idx(tr[c]);
        return u;
    }();
    return U;
}

bool add_checked(uint64_t& cell, uint64_t v) {
    if (cell > UINT64_MAX - v) return false;
    cell += v;
    return true;
}

int merge_census_impl(const uint64_t* star, const uint64_t* pair, const uint64_t* tri, int mode,
                      uint64_t* census) {
    const Universe& u = universe();
    if ((int)u.all.size() != 36) {
        g_last_error = "signature universe is not 36 classes";
        return TM_ERR_CONSISTENCY;
    }
    uint64_t out[36] = {0};
    for (int c = 0; c < 24; ++c)
        if (!add_checked(out[u.star_sig[c]], star[c])) return TM_ERR_OVERFLOW;
    for (int c = 0; c < 4; ++c) {  // d1 = outward; complement flips all bits
        if (pair[c] != pair[7 - c]) {
            g_last_error = "complementary pair cells disagree for " + u.all[u.pair_sig[c]];
            return TM_ERR_CONSISTENCY;
        }
        if (!add_checked(out[u.pair_sig[c]], pair[c])) return TM_ERR_OVERFLOW;
    }
    uint64_t sums[36] = {0};
    bool is_tri[36] = {false};
    for (int c = 0; c < 24; ++c) {
        if (!add_checked(sums[u.tri_sig[c]], tri[c])) return TM_ERR_OVERFLOW;
        is_tri[u.tri_sig[c]] = true;
    }
    for (int k = 0; k < 36; ++k) {
        if (!is_tri[k]) continue;
        if (mode == TM_TRI_COUNT_ALL) {
            if (sums[k] % 3) {
                g_last_error = "triangle class sum not divisible by 3 for " + u.all[k];
                return TM_ERR_CONSISTENCY;
            }
            if (!add_checked(out[k], sums[k] / 3)) return TM_ERR_OVERFLOW;
        } else if (!add_checked(out[k], sums[k])) {
            return TM_ERR_OVERFLOW;
        }
    }
    std::memcpy(census, out, sizeof(out));
    return TM_OK;
}

// A device cell is exact to 128 bits: its u64 sum plus the number of times
// the sum wrapped (tm_primitives.cuh cell_add).  A reference cell that would
// exceed 2^64 - 1 throws CounterOverflowError (checked_increment,
// types.hpp:65-70, via motifs.cpp:131-147 and the merges in executor.cpp:173-179).
using u128 = unsigned __int128;
inline u128 wide(uint64_t lo, uint64_t wraps) { return ((u128)wraps << 64) | lo; }
inline uint64_t narrow_checked(u128 v) {
    if (v >> 64) throw tm_error(TM_ERR_OVERFLOW, "motif counter overflow");
    return (uint64_t)v;
}

// raw star sums (Pair, C, B, A) -> reference Star / Pair cells; wraps: the
// raw cells' wrap counters (nullptr: none)
void finish_star(const uint64_t* raw, uint64_t* star, uint64_t* pair, const uint64_t* wraps = nullptr) {
    auto at = [&](int i) { return wide(raw[i], wraps ? wraps[i] : 0); };
    for (int c = 0; c < 8; ++c) {
        const u128 p = at(c);
        if (pair) pair[c] = narrow_checked(p);
        if (star) {
            star[0 * 8 + c] = narrow_checked(at(8 + c) - p);   // isolated_first  = C - Pair
            star[1 * 8 + c] = narrow_checked(at(16 + c) - p);  // isolated_second = B - Pair
            star[2 * 8 + c] = narrow_checked(at(24 + c) - p);  // isolated_third  = A - Pair
        }
    }
}

// once-counted cells -> count_all cells: every instance lands once in each
// cell of its class (triangle_engine.hpp:57-60)
void expand_count_all(const uint64_t* once, uint64_t* tri, const uint64_t* wraps = nullptr) {
    const Universe& u = universe();
    u128 cls[36] = {0};
    for (int c = 0; c < 24; ++c) cls[u.tri_sig[c]] += wide(once[c], wraps ? wraps[c] : 0);
    for (int c = 0; c < 24; ++c) tri[c] = narrow_checked(cls[u.tri_sig[c]]);
}
void copy_tri_checked(const uint64_t* once, uint64_t* tri, const uint64_t* wraps) {
    for (int c = 0; c < 24; ++c) tri[c] = narrow_checked(wide(once[c], wraps ? wraps[c] : 0));
}

struct PinnedAcc {
    uint64_t* h = nullptr;
    PinnedAcc() {
        if (cudaMallocHost(&h, kAccWords * sizeof(uint64_t)) != cudaSuccess) h = nullptr;
    }
};
// replayed graphs copy their counters into their own entry's pinned buffer
// (two asynchronous censuses can be in flight), everything else into the
// thread's buffer
thread_local uint64_t* g_acc_override = nullptr;
uint64_t* pinned_acc() {
    if (g_acc_override) return g_acc_override;
    static thread_local PinnedAcc p;
    if (!p.h) throw tm_error(TM_ERR_CUDA, "cannot allocate pinned host buffer");
    return p.h;
}
struct AccOverride {
    uint64_t* prev;
    explicit AccOverride(uint64_t* p) : prev(g_acc_override) { g_acc_override = p; }
    ~AccOverride() { g_acc_override = prev; }
};

template <typename F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const tm_error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return TM_ERR_CUDA;
    }
}

void ensure_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        throw tm_error(TM_ERR_CUDA, "no CUDA device: the B200 path has no CPU fallback");
}

const std::vector<uint32_t>& host_off(tm_graph* G) {
    if (G->h_off.size() != G->g.n + 1) {
        G->h_off.resize(G->g.n + 1);
        TM_CUDA(cudaMemcpyAsync(G->h_off.data(), G->g.off, (G->g.n + 1) * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, G->g.stream));
        TM_CUDA(cudaStreamSynchronize(G->g.stream));
    }
    return G->h_off;
}

uint32_t read_u32(const uint32_t* d, uint64_t idx, cudaStream_t s) {
    uint32_t v = 0;
    TM_CUDA(cudaMemcpyAsync(&v, d + idx, sizeof(v), cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    return v;
}

// test hook: every star raw cell starts at this value instead of 0 (Star =
// raw - Pair is unchanged, Pair = bias + count), so the device wrap counters
// and the host's overflow check can be exercised at the 2^64 boundary
thread_local uint64_t g_acc_bias = 0;

// one counting pass into the device accumulator; returns raw on host
struct PassResult {
    uint64_t star_raw[32];
    uint64_t tri_once[24];
    uint64_t star_wraps[32];
    uint64_t tri_wraps[24];
};

// host side of a pass: wait for the counter copy (the whole stream, or just
// up to `done` when later work is already queued behind it) and unpack it
void collect_passes(tm_graph* G, PassResult& r, cudaEvent_t done = nullptr) {
    if (done) TM_CUDA(cudaEventSynchronize(done));
    else TM_CUDA(cudaStreamSynchronize(G->g.stream));
    const uint64_t* h = pinned_acc();
    std::memcpy(r.star_raw, h, 32 * sizeof(uint64_t));
    std::memcpy(r.tri_once, h + 32, 24 * sizeof(uint64_t));
    std::memcpy(G->g.stats, h + 56, 8 * sizeof(uint64_t));
    std::memcpy(r.star_wraps, h + kAccCarry, 32 * sizeof(uint64_t));
    std::memcpy(r.tri_wraps, h + kAccCarry + 32, 24 * sizeof(uint64_t));
}

// inclusive bound on the first edge's t for a time-slice share (INT64_MAX:
// unbounded); `none` when the exclusive end admits no t at all
int64_t first_edge_t_last(const tm_run_config* cfg, bool& none) {
    none = false;
    if (!cfg->has_first_edge_t_end) return INT64_MAX;
    if (cfg->first_edge_t_end == INT64_MIN) {
        none = true;
        return INT64_MIN;
    }
    return cfg->first_edge_t_end - 1;
}

void run_passes(tm_graph* G, int64_t delta, int64_t t_last, bool do_star, bool do_tri, int tri_mode,
                uint32_t cb, uint32_t ce, PassResult& r, tm_phase_timings* tm, bool collect = true) {
    DeviceGraph& g = G->g;
    cudaStream_t s = g.stream;
    if (!g.d_acc) g.d_acc = dalloc<uint64_t>(kAccWords, s);
    TM_CUDA(cudaMemsetAsync(g.d_acc, 0, kAccWords * sizeof(uint64_t), s));
    if (g_acc_bias && collect) {  // test hook (tm_debug_acc_bias): start the 32 star raw cells at the bias
        static thread_local uint64_t bias[32];
        for (auto& b : bias) b = g_acc_bias;
        TM_CUDA(cudaMemcpyAsync(g.d_acc, bias, sizeof(bias), cudaMemcpyHostToDevice, s));
        TM_CUDA(cudaStreamSynchronize(s));
    }
    const bool full = (cb == 0 && ce == g.n);
    cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
    if (tm) {
        TM_CUDA(cudaEventCreate(&e0));
        TM_CUDA(cudaEventCreate(&e1));
        TM_CUDA(cudaEventCreate(&e2));
        TM_CUDA(cudaEventRecord(e0, s));
    }
    // star pass on a side stream, concurrent with the triangle pass on s
    // (both mostly latency-bound gathers; they accumulate into disjoint cells)
    const bool star_on = do_star && g.R;
    cudaStream_t ss = (star_on && g.aux[1]) ? g.aux[1] : s;  // side stream only when used
    if (star_on) {
        stream_after(g, ss, s);
        star_full(g, delta, cb, ce, t_last, g.d_acc, g.d_acc + 56, ss);
    }
    if (tm) TM_CUDA(cudaEventRecord(e1, ss));
    if (do_tri && g.R) {
        const int fm = tri_mode == TM_TRI_REMOVAL ? 1 : 0;
        build_forward(g, fm, s);
        const Forward& f = g.fwd[fm];
        uint32_t fb = 0, fe = (uint32_t)f.len;
        if (!full) {
            fb = read_u32(f.off, cb, s);
            fe = read_u32(f.off, ce, s);
        }
        if (fm == 0 && full && g.pre_tri.valid && g.pre_tri.delta == delta && g.pre_tri.f_begin == fb &&
            g.pre_tri.f_end == fe)
            tri_work_stage(g, f, g.pre_tri, t_last, g.d_acc + 32, g.d_acc + 56);  // filter ran during the build
        else
            tri_oriented(g, f, delta, fb, fe, t_last, g.d_acc + 32, g.d_acc + 56);
    }
    if (ss != s) {
        TM_CUDA(cudaEventRecord(g.ev_join, ss));
        TM_CUDA(cudaStreamWaitEvent(s, g.ev_join, 0));
    }
    if (tm) TM_CUDA(cudaEventRecord(e2, s));
    uint64_t* h = pinned_acc();
    TM_CUDA(cudaMemcpyAsync(h, g.d_acc, kAccWords * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    if (!collect) return;  // (graph capture: the caller launches, synchronises and collects)
    collect_passes(G, r);
    if (tm) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, e0, e1);  // star pass (side stream)
        cudaEventElapsedTime(&b, e0, e2);  // triangle pass, overlapping it
        tm->star_pair_ms = a;
        tm->triangle_ms = b;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaEventDestroy(e2);
    }
}

void check_config(const tm_run_config* cfg) {
    if (!cfg) throw tm_error(TM_ERR_INVALID, "null graph or config");
    if (cfg->workers < 1) throw tm_error(TM_ERR_CONFIG, "workers must be >= 1");
    if (cfg->delta < 0) throw tm_error(TM_ERR_CONFIG, "delta must be >= 0");
    if (cfg->triangle_mode == TM_TRI_REMOVAL && cfg->workers > 1)
        throw tm_error(TM_ERR_CONFIG, "removal triangle mode requires a single worker");
    if (cfg->triangle_mode != TM_TRI_REMOVAL && cfg->triangle_mode != TM_TRI_COUNT_ALL)
        throw tm_error(TM_ERR_CONFIG, "triangle mode must be countall or removal");
}

// raw pass sums -> the reference's counters (+ census for full runs)
void finish_counts(const PassResult& r, const tm_run_config* cfg, bool full, tm_counters* raw,
                   uint64_t* census, tm_phase_timings* tm) {
    const uint32_t motifs = cfg->motifs;
    tm_counters out;
    std::memset(&out, 0, sizeof(out));
    // filtered-out kinds were not counted (their cells are zero, not checked)
    if (motifs & (TM_MOTIF_STAR | TM_MOTIF_PAIR)) finish_star(r.star_raw, out.star, out.pair, r.star_wraps);
    if (!(motifs & TM_MOTIF_TRIANGLE)) {
    } else if (cfg->triangle_mode == TM_TRI_COUNT_ALL) {
        expand_count_all(r.tri_once, out.tri, r.tri_wraps);
    } else {
        copy_tri_checked(r.tri_once, out.tri, r.tri_wraps);
    }
    if (!(motifs & TM_MOTIF_STAR)) std::memset(out.star, 0, sizeof(out.star));
    if (!(motifs & TM_MOTIF_PAIR)) std::memset(out.pair, 0, sizeof(out.pair));
    if (!(motifs & TM_MOTIF_TRIANGLE)) std::memset(out.tri, 0, sizeof(out.tri));
    if (raw) *raw = out;
    auto t1 = std::chrono::steady_clock::now();
    if (census) {
        std::memset(census, 0, 36 * sizeof(uint64_t));
        if (full) {
            int rc = merge_census_impl(out.star, out.pair, out.tri, cfg->triangle_mode, census);
            if (rc) throw tm_error(rc, g_last_error.empty() ? "merge failed" : g_last_error);
        }
    }
    if (tm) tm->merge_ms = std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - t1).count();
}

int run_parallel_impl(tm_graph* G, const tm_run_config* cfg, tm_counters* raw, uint64_t* census,
                      tm_phase_timings* tm) {
    if (!G || !cfg) throw tm_error(TM_ERR_INVALID, "null graph or config");
    if (cfg->workers < 1) throw tm_error(TM_ERR_CONFIG, "workers must be >= 1");
    if (cfg->delta < 0) throw tm_error(TM_ERR_CONFIG, "delta must be >= 0");
    if (cfg->triangle_mode == TM_TRI_REMOVAL && cfg->workers > 1)
        throw tm_error(TM_ERR_CONFIG, "removal triangle mode requires a single worker");
    if (cfg->triangle_mode != TM_TRI_REMOVAL && cfg->triangle_mode != TM_TRI_COUNT_ALL)
        throw tm_error(TM_ERR_CONFIG, "triangle mode must be countall or removal");
    // an empty filter runs nothing and yields the all-zero census
    // (executor.cpp:28-29, 161-163, 204-206)
    const uint32_t motifs = cfg->motifs;
    const uint32_t cb = cfg->center_begin;
    const uint32_t ce = cfg->center_end ? cfg->center_end : (uint32_t)G->g.n;
    if (cb > ce || ce > G->g.n) throw tm_error(TM_ERR_INVALID, "bad center partition");
    const bool full = (cb == 0 && ce == G->g.n) && !cfg->has_first_edge_t_end;

    PassResult r;
    auto t0 = std::chrono::steady_clock::now();
    bool none = false;
    const int64_t t_last = first_edge_t_last(cfg, none);
    run_passes(G, cfg->delta, t_last, !none && (motifs & 3u) != 0, !none && (motifs & 4u) != 0, cfg->triangle_mode,
               cb, ce, r,
               tm);
    finish_counts(r, cfg, full, raw, census, tm);
    (void)t0;
    return TM_OK;
}

tm_graph* build_impl(const uint32_t* src, const uint32_t* dst, const int64_t* t, uint64_t m,
                     uint64_t n, int device_ptrs, void* stream, double* index_ms,
                     const RunHint* hint = nullptr, double* ingest_ms = nullptr) {
    ensure_device();
    if (m && (!src || !dst || !t)) throw tm_error(TM_ERR_INVALID, "null edge arrays");
    auto* G = new tm_graph();
    try {
        if (stream) {
            G->g.stream = static_cast<cudaStream_t>(stream);
        } else {
            TM_CUDA(cudaStreamCreateWithFlags(&G->g.stream, cudaStreamNonBlocking));
            G->g.owns_stream = true;
        }
        cudaStream_t s = G->g.stream;
        static bool pool_set = false;
        if (!pool_set) {  // keep freed blocks in the pool across steps
            int dev = 0;
            cudaGetDevice(&dev);
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            pool_set = true;
        }
        cudaEvent_t e0, e1, ec;
        if (index_ms) {
            TM_CUDA(cudaEventCreate(&e0));
            TM_CUDA(cudaEventCreate(&e1));
            TM_CUDA(cudaEventCreate(&ec));
            TM_CUDA(cudaEventRecord(e0, s));
        }
        const uint32_t *ds = src, *dd = dst;
        const int64_t* dt = t;
        uint32_t *hs = nullptr, *hd = nullptr;
        int64_t* ht = nullptr;
        if (!device_ptrs && m) {
            hs = dalloc<uint32_t>(m, s);
            hd = dalloc<uint32_t>(m, s);
            ht = dalloc<int64_t>(m, s);
            TM_CUDA(cudaMemcpyAsync(hs, src, m * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
            TM_CUDA(cudaMemcpyAsync(hd, dst, m * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
            TM_CUDA(cudaMemcpyAsync(ht, t, m * sizeof(int64_t), cudaMemcpyHostToDevice, s));
            ds = hs;
            dd = hd;
            dt = ht;
        }
        if (index_ms) TM_CUDA(cudaEventRecord(ec, s));  // ingest (host->device copy) | index build
        build_graph(G->g, ds, dd, dt, m, n, hint);
        dfree(hs, s);
        dfree(hd, s);
        dfree(ht, s);
        if (index_ms) {
            TM_CUDA(cudaEventRecord(e1, s));
            TM_CUDA(cudaEventSynchronize(e1));
            float ms = 0, ms_in = 0;
            cudaEventElapsedTime(&ms_in, e0, ec);
            cudaEventElapsedTime(&ms, ec, e1);
            *index_ms = ms;
            if (ingest_ms) *ingest_ms = ms_in;
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            cudaEventDestroy(ec);
        }
    } catch (...) {
        free_graph(G->g);
        if (G->g.owns_stream) cudaStreamDestroy(G->g.stream);
        delete G;
        throw;
    }
    return G;
}

// ---------------------------------------------------------------------------
// Graph replay for repeated one-shot counts (tm_count_edges with the same
// arrays, sizes, stream and config -- a caller streaming batches into fixed
// buffers, or a benchmark loop).  Everything after the pack/validate read-back
// is issued without host synchronisation (build_finish, the counting passes,
// the counter copy and all frees), so it is captured once per (narrow,
// unsorted) variant into a CUDA graph and replayed with one launch: ~40
// kernel launches, ~30 stream-ordered allocations and the side-stream
// fork/joins collapse into cudaGraphLaunch.  The prepare buffers live in a
// per-entry workspace so the replayed graph sees the same addresses.
struct ReplayKey {
    const void* src;
    const void* dst;
    const void* t;
    uint64_t m, n;
    int device_ptrs;
    cudaStream_t stream;
    tm_run_config cfg;
    bool operator==(const ReplayKey& o) const {
        return src == o.src && dst == o.dst && t == o.t && m == o.m && n == o.n &&
               device_ptrs == o.device_ptrs && stream == o.stream &&
               std::memcmp(&cfg, &o.cfg, sizeof(cfg)) == 0;
    }
};
struct ReplayEntry {
    ReplayKey key;
    BuildWorkspace ws;
    uint32_t* hs = nullptr;  // device staging of host arrays
    uint32_t* hd = nullptr;
    int64_t* ht = nullptr;
    cudaGraphExec_t exec[4] = {nullptr, nullptr, nullptr, nullptr};
    uint64_t kernels[4] = {0, 0, 0, 0};  // kernel launches captured in each graph
    int eager_runs[4] = {0, 0, 0, 0};
    // the t range a graph was captured for: its time base (narrow records) and
    // time-sort key width are baked in, so different data re-captures it
    int64_t cap_tmin[4] = {0, 0, 0, 0}, cap_tmax[4] = {0, 0, 0, 0};
    int recaptures = 0;  // data keeps changing under the same buffers: stay eager
    int last_variant = -1;  // replayed by the previous call (speculation target)
    BuildVerdict* verdict = nullptr;  // pinned
    uint64_t* acc = nullptr;          // pinned: the graph's counter read-back
    // speculative replays of this entry launched by the asynchronous API and
    // not yet collected (ReplayPending::E): the entry must outlive them
    int inflight = 0;
    void release() {
        for (auto& e : exec)
            if (e) {
                cudaGraphExecDestroy(e);
                e = nullptr;
            }
        cudaStream_t s = key.stream;
        cudaStreamSynchronize(s);
        dfree(ws.nk0, s); dfree(ws.nk1, s); dfree(ws.nv0, s); dfree(ws.nv1, s); dfree(ws.c0, s); dfree(ws.E, s); dfree(ws.st, s);
        dfree(hs, s); dfree(hd, s); dfree(ht, s);
        cudaStreamSynchronize(s);
        if (verdict) cudaFreeHost(verdict);
        verdict = nullptr;
        if (acc) cudaFreeHost(acc);
        acc = nullptr;
    }
};

constexpr int kPending = 100;  // count_edges_replay left a speculative replay in flight

// A speculative replay launched but not yet collected (asynchronous API):
// completing it synchronises, checks the verdict against the replayed
// variant and unpacks the counters.
struct ReplayPending {
    ReplayEntry* E = nullptr;
    tm_graph G;
    BuildPlan plan;
    int lv = -1;
    bool full = true;
};
struct ReplayCache {
    std::vector<ReplayEntry*> entries;  // most recent last
    cudaStream_t own = nullptr;
    ~ReplayCache() {
        for (auto* e : entries) {
            e->release();
            delete e;
        }
    }
};
thread_local ReplayCache g_replay;
constexpr size_t kReplayEntries = 2;

// the triangle filter of a one-shot count can run while the index builds
RunHint hint_for(const tm_run_config* cfg, uint64_t n) {
    RunHint h;
    const uint32_t motifs = cfg->motifs;
    h.early_tri = (motifs & TM_MOTIF_TRIANGLE) && cfg->triangle_mode == TM_TRI_COUNT_ALL &&
                  cfg->center_begin == 0 && (cfg->center_end == 0 || cfg->center_end == n) && cfg->delta >= 0;
    h.delta = cfg->delta;
    return h;
}

// Graph replay pays off where launch overhead matters; a captured graph also
// keeps its stream-ordered allocations reserved between launches (tens of GB
// at hundreds of millions of edges, per cached entry), so very large inputs
// run eagerly.
constexpr uint64_t kReplayMaxEdges = 128ull << 20;

bool replay_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TM_GRAPHS");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1 && !g_timing.load(std::memory_order_relaxed);
}

int count_edges_replay(const uint32_t* src, const uint32_t* dst, const int64_t* t, uint64_t m, uint64_t n,
                       int device_ptrs, void* stream, const tm_run_config* cfg, tm_counters* raw,
                       uint64_t* census36, ReplayPending* pend = nullptr) {
    ensure_device();
    check_config(cfg);
    if (!src || !dst || !t) throw tm_error(TM_ERR_INVALID, "null edge arrays");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!s) {
        if (!g_replay.own) TM_CUDA(cudaStreamCreateWithFlags(&g_replay.own, cudaStreamNonBlocking));
        s = g_replay.own;
    }
    ReplayKey key{src, dst, t, m, n, device_ptrs, s, *cfg};
    ReplayEntry* E = nullptr;
    for (size_t i = 0; i < g_replay.entries.size(); ++i)
        if (g_replay.entries[i]->key == key) {
            E = g_replay.entries[i];
            g_replay.entries.erase(g_replay.entries.begin() + i);
            break;
        }
    if (!E) {
        // evict the least recently used entry that no pending asynchronous
        // batch still reads (the cache may exceed kReplayEntries while all
        // entries are in flight: at most two per host thread)
        if (g_replay.entries.size() >= kReplayEntries) {
            for (size_t i = 0; i < g_replay.entries.size(); ++i)
                if (g_replay.entries[i]->inflight == 0) {
                    g_replay.entries[i]->release();
                    delete g_replay.entries[i];
                    g_replay.entries.erase(g_replay.entries.begin() + i);
                    break;
                }
        }
        E = new ReplayEntry();
        E->key = key;
    }
    g_replay.entries.push_back(E);

    const uint32_t* ds = src;
    const uint32_t* dd = dst;
    const int64_t* dt = t;
    if (!device_ptrs) {
        if (!E->hs) {
            E->hs = dalloc<uint32_t>(m, s);
            E->hd = dalloc<uint32_t>(m, s);
            E->ht = dalloc<int64_t>(m, s);
        }
        TM_CUDA(cudaMemcpyAsync(E->hs, src, m * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        TM_CUDA(cudaMemcpyAsync(E->hd, dst, m * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        TM_CUDA(cudaMemcpyAsync(E->ht, t, m * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        ds = E->hs;
        dd = E->hd;
        dt = E->ht;
    }
    const uint32_t motifs = cfg->motifs;
    bool none = false;
    const int64_t t_last = first_edge_t_last(cfg, none);
    const bool full = !cfg->has_first_edge_t_end;
    PassResult r;
    if (!E->verdict) TM_CUDA(cudaMallocHost(&E->verdict, sizeof(BuildVerdict)));
    if (!E->acc) TM_CUDA(cudaMallocHost(&E->acc, kAccWords * sizeof(uint64_t)));
    AccOverride acc_scope(E->acc);
    // Speculative replay: when the previous call of this entry replayed a
    // graph, pack + validate and launch that graph back to back without the
    // verdict read-back in between; the verdict is checked afterwards (the
    // pack clamps invalid ids, so even rejected input stays in bounds) and a
    // call whose data changed variant or t range falls through to the
    // checked path below.
    if (E->last_variant >= 0 && E->exec[E->last_variant]) {
        const int lv = E->last_variant;
        tm_graph G;
        G.g.stream = s;
        BuildPlan plan;
        try {
            plan = build_prepare(G.g, ds, dd, dt, m, n, &E->ws, E->verdict);
            TM_CUDA(cudaGraphLaunch(E->exec[lv], s));
            if (pend) {  // asynchronous: collected by complete_pending
                g_launches.fetch_add(E->kernels[lv]);
                ++E->inflight;
                pend->E = E;
                pend->G.g = G.g;
                G.g = DeviceGraph();
                pend->plan = plan;
                pend->lv = lv;
                pend->full = full;
                return kPending;
            }
            collect_passes(&G, r);
            plan_from_verdict(G.g, plan, *E->verdict);
        } catch (...) {
            free_graph(G.g);
            throw;
        }
        free_graph(G.g);
        const int v = (plan.narrow ? 2 : 0) | (plan.unsorted ? 1 : 0);
        if (v == lv && E->cap_tmin[lv] == plan.tmin && E->cap_tmax[lv] == plan.tmax) {
            g_launches.fetch_add(E->kernels[lv]);
            finish_counts(r, cfg, full, raw, census36, nullptr);
            return TM_OK;
        }
        E->last_variant = -1;  // the data moved: redo with the verdict first
    }
    tm_graph G;
    G.g.stream = s;
    BuildPlan plan;
    try {
        plan = build_prepare(G.g, ds, dd, dt, m, n, &E->ws);
    } catch (...) {
        free_graph(G.g);
        throw;
    }
    const int variant = (plan.narrow ? 2 : 0) | (plan.unsorted ? 1 : 0);
    const RunHint hint = hint_for(cfg, n);
    auto issue = [&](bool collect) {
        build_finish(G.g, plan, ds, dd, dt, &hint);
        run_passes(&G, cfg->delta, t_last, !none && (motifs & 3u) != 0, !none && (motifs & 4u) != 0,
                   cfg->triangle_mode, 0,
                   (uint32_t)n, r, nullptr, collect);
    };
    if (E->exec[variant] && (E->cap_tmin[variant] != plan.tmin || E->cap_tmax[variant] != plan.tmax)) {
        cudaGraphExecDestroy(E->exec[variant]);
        E->exec[variant] = nullptr;
        E->eager_runs[variant] = 0;
        ++E->recaptures;
    }
    if (!E->exec[variant] && (E->eager_runs[variant] == 0 || E->recaptures > 2)) {
        // first run of this shape: eager (also initialises every lazy static)
        ++E->eager_runs[variant];
        try {
            issue(true);
        } catch (...) {
            free_graph(G.g);
            throw;
        }
        free_graph(G.g);
        TM_CUDA(cudaStreamSynchronize(s));
        finish_counts(r, cfg, full, raw, census36, nullptr);
        return TM_OK;
    }
    if (!E->exec[variant]) {
        cudaGraph_t graph = nullptr;
        const uint64_t l0 = g_launches.load();
        TM_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
            issue(false);
            free_graph(G.g);
        } catch (...) {
            cudaStreamEndCapture(s, &graph);
            if (graph) cudaGraphDestroy(graph);
            free_graph(G.g);
            throw;
        }
        TM_CUDA(cudaStreamEndCapture(s, &graph));
        E->kernels[variant] = g_launches.load() - l0;
        g_launches.fetch_sub(E->kernels[variant]);  // counted when launched, below
        cudaGraphExec_t ex = nullptr;
        const cudaError_t ie = cudaGraphInstantiate(&ex, graph, 0);
        cudaGraphDestroy(graph);
        TM_CUDA(ie);
        E->exec[variant] = ex;
        E->cap_tmin[variant] = plan.tmin;
        E->cap_tmax[variant] = plan.tmax;
    } else {
        free_graph(G.g);  // (only returns the side streams: nothing was allocated)
    }
    TM_CUDA(cudaGraphLaunch(E->exec[variant], s));
    g_launches.fetch_add(E->kernels[variant]);  // the graph's kernels, launched from the device queue
    collect_passes(&G, r);
    finish_counts(r, cfg, full, raw, census36, nullptr);
    E->last_variant = variant;
    return TM_OK;
}

// node-id tokens joined by '\n' in id order
struct IdLenLoad {
    const uint32_t* len;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return (uint64_t)len[i] + 1; }
};
__global__ void gather_ids_kernel(const unsigned char* __restrict__ text, const uint64_t* __restrict__ off,
                                  const uint32_t* __restrict__ len, const uint64_t* __restrict__ pos, uint64_t n,
                                  char* __restrict__ out) {
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p = pos[u];
        for (uint32_t k = 0; k < len[u]; ++k) out[p + k] = (char)text[off[u] + k];
        if (u + 1 < n) out[p + len[u]] = '\n';
    }
}
thread_local uint64_t g_parse_line = 0;

// Finish a speculative replay: wait, check the verdict against the replayed
// variant and t range, unpack.  Returns false when the data did not match the
// graph (the caller re-runs the checked path on the same device arrays).
bool complete_pending(ReplayPending& P, cudaEvent_t done, const tm_run_config* cfg, tm_counters* raw,
                      uint64_t* census36) {
    ReplayEntry* E = P.E;
    --E->inflight;  // (the entry stays cached; it is only pinned while pending)
    PassResult r;
    bool ok = false;
    try {
        AccOverride acc_scope(E->acc);
        collect_passes(&P.G, r, done);
        plan_from_verdict(P.G.g, P.plan, *E->verdict);
        const int v = (P.plan.narrow ? 2 : 0) | (P.plan.unsorted ? 1 : 0);
        ok = v == P.lv && E->cap_tmin[v] == P.plan.tmin && E->cap_tmax[v] == P.plan.tmax;
    } catch (...) {
        free_graph(P.G.g);
        throw;
    }
    free_graph(P.G.g);
    if (!ok) {
        E->last_variant = -1;
        return false;
    }
    finish_counts(r, cfg, P.full, raw, census36, nullptr);
    return true;
}

// Per-host-thread pipeline of the asynchronous API: two staging slots of
// device input buffers, filled on a copy stream while the other slot's
// census runs.
// ---- host-side timestamp packing for the pipelined batches ----------------
//
// A batch's PCIe bytes are 16 per edge (u32 src, u32 dst, i64 t), and the
// pipelined census of a large batch is bound by that copy (config 4: 9.6 GB at
// ~53 GB/s = 182 ms against a 151 ms census).  Timestamps of 65536 consecutive
// edges almost always span less than 2^32, so host worker threads rewrite t as
// a per-block i64 base + u32 offsets into a pinned staging buffer while the
// src / dst copies are on the wire; the copy stream waits for each packed piece
// with a host function, copies it (4 bytes per edge) and one kernel expands the
// offsets into the i64 array the census reads.  A block whose span does not fit
// marks the batch, and its census then waits for a plain copy of t.
// A pipeline starts with u16 offsets from a base per 4096 edges (10 bytes per
// edge on the link: a dense stream's 4096 consecutive edges span far less than
// 2^16); the first batch with a block that does not fit takes the plain copy
// and moves the pipeline to u32 offsets for good (TM_H2D_PACK16=0 starts there).
constexpr uint64_t kPackBlock = 1u << 16;   // edges per base, u32 offsets
constexpr uint64_t kPackBlock16 = 1u << 12; // edges per base, u16 offsets
constexpr uint64_t kPackTask = 1u << 20;    // edges per worker task
constexpr uint64_t kPackPiece = 1u << 26;   // edges per staged copy
constexpr uint64_t kPackMinEdges = 1u << 24;  // smaller batches: plain copies (TM_H2D_PACK_MIN overrides, tests)

class HostPool {
  public:
    static HostPool& get() {
        static HostPool* p = new HostPool();  // never destroyed: no join at process exit
        return *p;
    }
    void submit(std::function<void()> f) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            q_.push_back(std::move(f));
        }
        cv_.notify_one();
    }

  private:
    HostPool() {
        int n = (int)std::thread::hardware_concurrency();
        if (const char* e = std::getenv("TM_HOST_THREADS")) n = std::atoi(e);
        n_ = std::max(1, std::min(n, 32));
        for (int i = 0; i < n_; ++i) std::thread([this] { run(); }).detach();
    }
    void run() {
        for (;;) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return !q_.empty(); });
                f = std::move(q_.front());
                q_.pop_front();
            }
            f();
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    int n_ = 1;
};

struct PackPiece {
    std::atomic<uint32_t> left{0};
};
struct PackJob {
    const int64_t* t = nullptr;
    uint64_t m = 0;
    uint32_t* off = nullptr;   // pinned staging (u16 offsets when width == 2)
    int64_t* base = nullptr;   // pinned staging, one per kPackBlock / kPackBlock16 edges
    int width = 4;             // bytes per offset
    std::unique_ptr<PackPiece[]> piece;
    uint64_t pieces = 0;
    std::atomic<uint32_t> bad{0};
    std::mutex mu;
    std::condition_variable cv;
    void wait_piece(uint64_t i) {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return piece[i].left.load(std::memory_order_acquire) == 0; });
    }
    void wait_all() {
        for (uint64_t i = 0; i < pieces; ++i) wait_piece(i);
    }
};

// offsets of one block from its first timestamp; a second pass from the
// block's minimum when an edge falls outside [t0, t0 + 2^32)
template <typename O>
bool pack_block(const int64_t* t, uint64_t cnt, O* off, int64_t* base) {
    constexpr uint64_t kMax = (uint64_t)(O)~(O)0;  // 2^k - 1: the OR of the offsets exceeds it iff one of them does
    const int64_t t0 = t[0];
    uint64_t over = 0;
    for (uint64_t i = 0; i < cnt; ++i) {
        const uint64_t d = (uint64_t)t[i] - (uint64_t)t0;  // wraps for t[i] < t0: caught by the range test
        off[i] = (O)d;
        over |= d;
    }
    *base = t0;
    if (over <= kMax) return true;
    int64_t lo = t0, hi = t0;
    for (uint64_t i = 0; i < cnt; ++i) {
        lo = std::min(lo, t[i]);
        hi = std::max(hi, t[i]);
    }
    if ((uint64_t)hi - (uint64_t)lo > kMax) return false;
    for (uint64_t i = 0; i < cnt; ++i) off[i] = (O)((uint64_t)t[i] - (uint64_t)lo);
    *base = lo;
    return true;
}

void pack_start(PackJob& J) {
    J.pieces = (J.m + kPackPiece - 1) / kPackPiece;
    J.piece.reset(new PackPiece[J.pieces]);
    J.bad.store(0);
    for (uint64_t p = 0; p < J.pieces; ++p) {
        const uint64_t b = p * kPackPiece, e = std::min(J.m, b + kPackPiece);
        J.piece[p].left.store((uint32_t)((e - b + kPackTask - 1) / kPackTask));
    }
    HostPool& pool = HostPool::get();
    for (uint64_t b = 0; b < J.m; b += kPackTask) {
        const uint64_t e = std::min(J.m, b + kPackTask);
        PackJob* j = &J;
        pool.submit([j, b, e] {
            if (j->width == 2) {
                uint16_t* off16 = reinterpret_cast<uint16_t*>(j->off);
                for (uint64_t x = b; x < e; x += kPackBlock16) {
                    const uint64_t c = std::min(kPackBlock16, e - x);
                    if (!pack_block(j->t + x, c, off16 + x, j->base + x / kPackBlock16)) {
                        j->bad.store(1);
                        break;  // the batch takes the plain copy
                    }
                }
            } else {
                for (uint64_t x = b; x < e; x += kPackBlock) {
                    const uint64_t c = std::min(kPackBlock, e - x);
                    if (!pack_block(j->t + x, c, j->off + x, j->base + x / kPackBlock)) j->bad.store(1);
                }
            }
            PackPiece& pc = j->piece[b / kPackPiece];
            if (pc.left.fetch_sub(1, std::memory_order_acq_rel) == 1) {
                std::lock_guard<std::mutex> lk(j->mu);
                j->cv.notify_all();
            }
        });
    }
}

struct PieceWait {
    PackJob* job;
    uint64_t piece;
};
void CUDART_CB pack_wait_cb(void* arg) {
    PieceWait* w = static_cast<PieceWait*>(arg);
    w->job->wait_piece(w->piece);
}

template <typename O, uint64_t kBlock>
__global__ void unpack_t_kernel(const O* __restrict__ off, const int64_t* __restrict__ base, uint64_t m,
                                int64_t* __restrict__ t) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        t[i] = base[i / kBlock] + (int64_t)off[i];
}

bool pack_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TM_H2D_PACK");
        return !(e && e[0] == '0');
    }();
    return on;
}
bool pack16_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TM_H2D_PACK16");
        return !(e && e[0] == '0');
    }();
    return on;
}
uint64_t pack_min_edges() {
    static const uint64_t v = [] {
        const char* e = std::getenv("TM_H2D_PACK_MIN");
        return e ? (uint64_t)std::strtoull(e, nullptr, 10) : kPackMinEdges;
    }();
    return v;
}
std::atomic<uint64_t> g_h2d_bytes{0};  // input bytes the last submitted batch put on the wire

struct AsyncResult {
    int rc = TM_OK;
    std::string err;
    tm_counters raw;
    uint64_t census[36];
};
struct AsyncSlot {
    uint32_t* ds = nullptr;
    uint32_t* dd = nullptr;
    int64_t* dt = nullptr;
    uint64_t cap = 0;
    cudaEvent_t copied = nullptr, done = nullptr;
    bool busy = false, pending = false;
    bool deferred = false;  // large batch: census not yet issued (runs when the next batch is submitted)
    // packed timestamps (large batches): pinned staging, device copies, the running job
    uint32_t* h_off = nullptr;
    int64_t* h_base = nullptr;
    uint32_t* d_off = nullptr;
    int64_t* d_base = nullptr;
    uint64_t pack_cap = 0;
    bool packed = false;
    const int64_t* host_t = nullptr;
    std::unique_ptr<PackJob> job;
    std::vector<PieceWait> waits;
    uint64_t ticket = 0, m = 0, n = 0;
    cudaStream_t s = nullptr;
    tm_run_config cfg;
    ReplayPending P;
    AsyncResult res;  // when !pending
};
struct AsyncPipe {
    cudaStream_t copy = nullptr;
    AsyncSlot slot[2];
    uint64_t next = 1;
    int t_width = 2;  // bytes per packed timestamp offset: 2 until a batch does not fit, then 4
    std::vector<std::pair<uint64_t, AsyncResult>> finished;  // completed, not yet waited
    ~AsyncPipe() {
        for (auto& sl : slot) {
            if (sl.copied) cudaEventDestroy(sl.copied);
            if (sl.done) cudaEventDestroy(sl.done);
            if (sl.job) sl.job->wait_all();
            if (sl.ds) {
                cudaFree(sl.ds);
                cudaFree(sl.dd);
                cudaFree(sl.dt);
            }
            if (sl.h_off) {
                cudaFreeHost(sl.h_off);
                cudaFreeHost(sl.h_base);
                cudaFree(sl.d_off);
                cudaFree(sl.d_base);
            }
        }
        if (copy) cudaStreamDestroy(copy);
    }
};
thread_local AsyncPipe g_async;

// A batch above the replay size is counted eagerly, and an eager count syncs
// the host (the build verdict).  Its census is therefore issued only when the
// next batch has been submitted -- after that batch's host->device copy is
// queued on the copy stream -- so the copy of batch i+1 overlaps the census of
// batch i.
void run_deferred(AsyncSlot& sl) {
    if (!sl.deferred) return;
    sl.deferred = false;
    if (sl.packed) {
        sl.job->wait_all();  // long done: the copy stream already waited for every piece
        if (sl.job->bad.load()) {  // a block's span did not fit the offsets: plain copy of t
            AsyncPipe& A = g_async;
            if (sl.job->width == 2) A.t_width = 4;  // later batches pack u32 offsets
            TM_CUDA(cudaMemcpyAsync(sl.dt, sl.host_t, sl.m * sizeof(int64_t), cudaMemcpyHostToDevice, A.copy));
            TM_CUDA(cudaEventRecord(sl.copied, A.copy));
            TM_CUDA(cudaStreamWaitEvent(sl.s, sl.copied, 0));
            g_h2d_bytes.fetch_add(sl.m * sizeof(int64_t));
        }
        sl.packed = false;
    }
    const int rc = tm_count_edges(sl.ds, sl.dd, sl.dt, sl.m, sl.n, 1, sl.s, &sl.cfg, &sl.res.raw, sl.res.census,
                                  nullptr);
    sl.res.rc = rc;
    if (rc != TM_OK) sl.res.err = g_last_error;
    TM_CUDA(cudaEventRecord(sl.done, sl.s));
}

// run the slot's census to completion (speculation checked, re-run if needed)
AsyncResult finish_slot(AsyncSlot& sl) {
    AsyncResult out;
    try {
        run_deferred(sl);
    } catch (const tm_error& e) {
        sl.res.rc = e.code;
        sl.res.err = e.what();
    }
    try {
        if (sl.pending) {
            sl.pending = false;
            if (!complete_pending(sl.P, sl.done, &sl.cfg, &out.raw, out.census))
                count_edges_replay(sl.ds, sl.dd, sl.dt, sl.m, sl.n, 1, sl.s, &sl.cfg, &out.raw, out.census);
        } else {
            out = sl.res;
        }
    } catch (const tm_error& e) {
        out.rc = e.code;
        out.err = e.what();
    } catch (const std::exception& e) {
        out.rc = TM_ERR_CUDA;
        out.err = e.what();
    }
    sl.busy = false;
    return out;
}

void free_impl(tm_graph* G) {
    if (!G) return;
    free_graph(G->g);
    cudaStreamSynchronize(G->g.stream);
    if (G->g.owns_stream) cudaStreamDestroy(G->g.stream);
    delete G;
}

}  // namespace
}  // namespace tmb

using namespace tmb;

extern "C" {

int tm_graph_build(const uint32_t* src, const uint32_t* dst, const int64_t* t, uint64_t m,
                   uint64_t n, int device_ptrs, void* stream, tm_graph** out) {
    return guarded([&] {
        if (!out) throw tm_error(TM_ERR_INVALID, "null output handle");
        *out = build_impl(src, dst, t, m, n, device_ptrs, stream, nullptr);
        return TM_OK;
    });
}

void tm_graph_free(tm_graph* g) {
    try {
        free_impl(g);
    } catch (...) {
    }
}

uint64_t tm_graph_node_count(const tm_graph* g) { return g ? g->g.n : 0; }
uint64_t tm_graph_edge_count(const tm_graph* g) { return g ? g->g.m : 0; }
void* tm_graph_stream(const tm_graph* g) { return g ? (void*)g->g.stream : nullptr; }

int tm_graph_degrees(const tm_graph* g, uint64_t* out) {
    return guarded([&] {
        auto* G = const_cast<tm_graph*>(g);
        const auto& off = host_off(G);
        for (uint64_t u = 0; u < G->g.n; ++u) out[u] = off[u + 1] - off[u];
        return TM_OK;
    });
}

namespace {
// host copy of timestamps [b, b + cnt) of a TimeBuf as absolute int64
void copy_times(const TimeBuf& tb, int64_t base, uint64_t b, uint64_t cnt, int64_t* out, cudaStream_t st) {
    if (!cnt) return;
    if (tb.n) {
        std::vector<uint32_t> tmp(cnt);
        TM_CUDA(cudaMemcpyAsync(tmp.data(), tb.n + b, cnt * 4, cudaMemcpyDeviceToHost, st));
        TM_CUDA(cudaStreamSynchronize(st));
        for (uint64_t i = 0; i < cnt; ++i) out[i] = base + (int64_t)tmp[i];
    } else {
        TM_CUDA(cudaMemcpyAsync(out, tb.w + b, cnt * 8, cudaMemcpyDeviceToHost, st));
    }
}
}  // namespace

int tm_graph_sequence(const tm_graph* g, uint32_t u, int64_t* t, uint64_t* ordinal, uint32_t* other,
                      uint8_t* dir, uint64_t cap, uint64_t* len) {
    return guarded([&] {
        auto* G = const_cast<tm_graph*>(g);
        if (u >= G->g.n) throw tm_error(TM_ERR_INVALID, "node out of range");
        const auto& off = host_off(G);
        const uint64_t b = off[u], s = off[u + 1] - off[u];
        if (len) *len = s;
        if (s > cap) return TM_ERR_INVALID;
        std::vector<int64_t> ht(s);
        std::vector<uint32_t> hn(s), ho(s);
        cudaStream_t st = G->g.stream;
        if (s) {
            copy_times(G->g.S_t, G->g.tbase, b, s, ht.data(), st);
            TM_CUDA(cudaMemcpyAsync(hn.data(), G->g.S_nbr + b, s * 4, cudaMemcpyDeviceToHost, st));
            TM_CUDA(cudaMemcpyAsync(ho.data(), G->g.S_ord + b, s * 4, cudaMemcpyDeviceToHost, st));
            TM_CUDA(cudaStreamSynchronize(st));
        }
        for (uint64_t k = 0; k < s; ++k) {
            if (t) t[k] = ht[k];
            if (ordinal) ordinal[k] = ho[k] & kNodeMask;
            if (other) other[k] = hn[k] & kNodeMask;
            if (dir) dir[k] = (uint8_t)(hn[k] >> 31);
        }
        return TM_OK;
    });
}

int tm_pair_window(const tm_graph* g, uint32_t v, uint32_t w, int64_t lo, int64_t hi, int64_t* t,
                   uint64_t* ordinal, uint8_t* dir_rel_v, uint64_t cap, uint64_t* len) {
    return guarded([&] {
        auto* G = const_cast<tm_graph*>(g);
        if (v >= G->g.n || w >= G->g.n) throw tm_error(TM_ERR_INVALID, "node out of range");
        if (len) *len = 0;
        if (v == w || lo > hi) return TM_OK;
        cudaStream_t st = G->g.stream;
        // the pair's P block is its lower endpoint's in (degree class, id) order
        uint8_t cv = 0, cw = 0;
        TM_CUDA(cudaMemcpyAsync(&cv, G->g.cls + v, 1, cudaMemcpyDeviceToHost, st));
        TM_CUDA(cudaMemcpyAsync(&cw, G->g.cls + w, 1, cudaMemcpyDeviceToHost, st));
        TM_CUDA(cudaStreamSynchronize(st));
        const bool vlow = cv < cw || (cv == cw && v < w);
        const uint32_t a = vlow ? v : w, b = vlow ? w : v;
        const uint32_t k0 = read_u32(G->g.pofs, a, st), k1 = read_u32(G->g.pofs, a + 1, st);
        std::vector<uint32_t> mx(k1 - k0);
        if (k1 > k0) {
            TM_CUDA(cudaMemcpyAsync(mx.data(), G->g.P_max + k0, (k1 - k0) * 4, cudaMemcpyDeviceToHost, st));
            TM_CUDA(cudaStreamSynchronize(st));
        }
        auto lo_it = std::lower_bound(mx.begin(), mx.end(), b);
        auto hi_it = std::upper_bound(lo_it, mx.end(), b);
        const uint32_t kb = k0 + (uint32_t)(lo_it - mx.begin()), ke = k0 + (uint32_t)(hi_it - mx.begin());
        if (ke == kb) return TM_OK;
        std::vector<int64_t> ht(ke - kb);
        std::vector<uint32_t> ho(ke - kb), hw(ke - kb);
        copy_times(G->g.P_t, G->g.tbase, kb, ke - kb, ht.data(), st);
        TM_CUDA(cudaMemcpyAsync(ho.data(), G->g.P_ord + kb, (ke - kb) * 4, cudaMemcpyDeviceToHost, st));
        TM_CUDA(cudaMemcpyAsync(hw.data(), G->g.P_w + kb, (ke - kb) * 4, cudaMemcpyDeviceToHost, st));
        TM_CUDA(cudaStreamSynchronize(st));
        const uint32_t flip = v == a ? 0u : 1u;
        uint64_t k = 0;
        for (uint32_t x = 0; x < ke - kb; ++x) {
            if (ht[x] < lo || ht[x] > hi) continue;
            if (k < cap) {
                if (t) t[k] = ht[x];
                if (ordinal) ordinal[k] = ho[x];
                if (dir_rel_v) dir_rel_v[k] = (uint8_t)((hw[x] >> 31) ^ flip);
            }
            ++k;
        }
        if (len) *len = k;
        return k > cap ? TM_ERR_INVALID : TM_OK;
    });
}

int tm_auto_degree_threshold(const tm_graph* g, uint64_t* out) {
    return guarded([&] {
        auto* G = const_cast<tm_graph*>(g);
        const auto& off = host_off(G);
        std::vector<uint64_t> d(G->g.n);
        for (uint64_t u = 0; u < G->g.n; ++u) d[u] = off[u + 1] - off[u];
        if (d.empty()) {
            *out = 0;
            return TM_OK;
        }
        if (d.size() < 20) {
            *out = *std::max_element(d.begin(), d.end());
            return TM_OK;
        }
        std::nth_element(d.begin(), d.begin() + 19, d.end(), std::greater<uint64_t>());
        *out = d[19];
        return TM_OK;
    });
}

int tm_count_star_pair(tm_graph* g, int64_t delta, uint64_t* star24, uint64_t* pair8) {
    return guarded([&] {
        if (delta < 0) throw tm_error(TM_ERR_CONFIG, "delta must be >= 0");
        PassResult r;
        run_passes(g, delta, INT64_MAX, true, false, 0, 0, (uint32_t)g->g.n, r, nullptr);
        finish_star(r.star_raw, star24, pair8, r.star_wraps);
        return TM_OK;
    });
}

int tm_count_triangles(tm_graph* g, int64_t delta, int mode, uint64_t* tri24) {
    return guarded([&] {
        if (delta < 0) throw tm_error(TM_ERR_CONFIG, "delta must be >= 0");
        if (mode != TM_TRI_COUNT_ALL && mode != TM_TRI_REMOVAL)
            throw tm_error(TM_ERR_CONFIG, "triangle mode must be countall or removal");
        PassResult r;
        run_passes(g, delta, INT64_MAX, false, true, mode, 0, (uint32_t)g->g.n, r, nullptr);
        if (mode == TM_TRI_COUNT_ALL) expand_count_all(r.tri_once, tri24, r.tri_wraps);
        else copy_tri_checked(r.tri_once, tri24, r.tri_wraps);
        return TM_OK;
    });
}

int tm_count_star_pair_items(tm_graph* g, int64_t delta, uint64_t n_items, const uint32_t* nodes,
                             const uint64_t* begin, const uint64_t* end, uint64_t* star_out,
                             uint64_t* pair_out) {
    return guarded([&] {
        if (delta < 0) throw tm_error(TM_ERR_CONFIG, "delta must be >= 0");
        const auto& off = host_off(g);
        std::vector<uint64_t> fo(n_items + 1, 0), to(n_items + 1, 0), b(n_items), e(n_items);
        for (uint64_t it = 0; it < n_items; ++it) {
            if (nodes[it] >= g->g.n) throw tm_error(TM_ERR_INVALID, "node out of range");
            const uint64_t s = off[nodes[it] + 1] - off[nodes[it]];
            b[it] = std::min<uint64_t>(begin[it], s);
            e[it] = std::min<uint64_t>(std::max(end[it], b[it]), s);
            fo[it + 1] = fo[it] + (e[it] - b[it]);
            to[it + 1] = to[it] + (s > b[it] + 1 ? s - b[it] - 1 : 0);
            if (end[it] <= begin[it]) to[it + 1] = to[it];  // empty range counts nothing
        }
        cudaStream_t s = g->g.stream;
        uint32_t* dn = dalloc<uint32_t>(n_items, s);
        uint64_t *db = dalloc<uint64_t>(n_items, s), *de = dalloc<uint64_t>(n_items, s);
        uint64_t *dfo = dalloc<uint64_t>(n_items + 1, s), *dto = dalloc<uint64_t>(n_items + 1, s);
        uint64_t* dout = dalloc<uint64_t>(n_items * 64, s);  // per item: 32 cells + 32 wrap counters
        TM_CUDA(cudaMemcpyAsync(dn, nodes, n_items * 4, cudaMemcpyHostToDevice, s));
        TM_CUDA(cudaMemcpyAsync(db, b.data(), n_items * 8, cudaMemcpyHostToDevice, s));
        TM_CUDA(cudaMemcpyAsync(de, e.data(), n_items * 8, cudaMemcpyHostToDevice, s));
        TM_CUDA(cudaMemcpyAsync(dfo, fo.data(), (n_items + 1) * 8, cudaMemcpyHostToDevice, s));
        TM_CUDA(cudaMemcpyAsync(dto, to.data(), (n_items + 1) * 8, cudaMemcpyHostToDevice, s));
        TM_CUDA(cudaMemsetAsync(dout, 0, n_items * 64 * 8, s));
        build_s_pidx(g->g);
        star_items(g->g, delta, n_items, dn, db, de, dfo, fo[n_items], to[n_items], dto, dout);
        std::vector<uint64_t> raw(n_items * 64);
        TM_CUDA(cudaMemcpyAsync(raw.data(), dout, n_items * 64 * 8, cudaMemcpyDeviceToHost, s));
        dfree(dn, s); dfree(db, s); dfree(de, s); dfree(dfo, s); dfree(dto, s); dfree(dout, s);
        TM_CUDA(cudaStreamSynchronize(s));
        for (uint64_t it = 0; it < n_items; ++it)
            finish_star(&raw[it * 64], star_out ? star_out + it * 24 : nullptr,
                        pair_out ? pair_out + it * 8 : nullptr, &raw[it * 64 + 32]);
        return TM_OK;
    });
}

int tm_count_triangles_items(tm_graph* g, int64_t delta, uint64_t n_items, const uint32_t* nodes,
                             const uint64_t* begin, const uint64_t* end, const uint8_t* live,
                             uint64_t* tri_out) {
    return guarded([&] {
        if (delta < 0) throw tm_error(TM_ERR_CONFIG, "delta must be >= 0");
        const auto& off = host_off(g);
        std::vector<uint64_t> io(n_items + 1, 0), b(n_items);
        for (uint64_t it = 0; it < n_items; ++it) {
            if (nodes[it] >= g->g.n) throw tm_error(TM_ERR_INVALID, "node out of range");
            const uint64_t s = off[nodes[it] + 1] - off[nodes[it]];
            const uint64_t lim = s >= 2 ? s - 1 : 0;
            b[it] = std::min<uint64_t>(begin[it], lim);
            const uint64_t e = std::min<uint64_t>(std::max(end[it], b[it]), lim);
            io[it + 1] = io[it] + (e - b[it]);
        }
        cudaStream_t s = g->g.stream;
        uint32_t* dn = dalloc<uint32_t>(n_items, s);
        uint64_t *db = dalloc<uint64_t>(n_items, s), *dio = dalloc<uint64_t>(n_items + 1, s);
        uint64_t* dout = dalloc<uint64_t>(n_items * 48, s);  // per item: 24 cells + 24 wrap counters
        uint8_t* dl = nullptr;
        TM_CUDA(cudaMemcpyAsync(dn, nodes, n_items * 4, cudaMemcpyHostToDevice, s));
        TM_CUDA(cudaMemcpyAsync(db, b.data(), n_items * 8, cudaMemcpyHostToDevice, s));
        TM_CUDA(cudaMemcpyAsync(dio, io.data(), (n_items + 1) * 8, cudaMemcpyHostToDevice, s));
        TM_CUDA(cudaMemsetAsync(dout, 0, n_items * 48 * 8, s));
        if (live) {
            dl = dalloc<uint8_t>(g->g.n, s);
            TM_CUDA(cudaMemcpyAsync(dl, live, g->g.n, cudaMemcpyHostToDevice, s));
        }
        tri_items(g->g, delta, n_items, dn, db, dio, io[n_items], dl, dout);
        std::vector<uint64_t> raw(n_items * 48);
        TM_CUDA(cudaMemcpyAsync(raw.data(), dout, n_items * 48 * 8, cudaMemcpyDeviceToHost, s));
        dfree(dn, s); dfree(db, s); dfree(dio, s); dfree(dout, s); dfree(dl, s);
        TM_CUDA(cudaStreamSynchronize(s));
        for (uint64_t it = 0; it < n_items; ++it) copy_tri_checked(&raw[it * 48], tri_out + it * 24, &raw[it * 48 + 24]);
        return TM_OK;
    });
}

int tm_run_parallel(tm_graph* g, const tm_run_config* cfg, tm_counters* raw, uint64_t* census36,
                    tm_phase_timings* timings) {
    return guarded([&] { return run_parallel_impl(g, cfg, raw, census36, timings); });
}

int tm_count_edges(const uint32_t* src, const uint32_t* dst, const int64_t* t, uint64_t m,
                   uint64_t n, int device_ptrs, void* stream, const tm_run_config* cfg,
                   tm_counters* raw, uint64_t* census36, tm_phase_timings* timings) {
    return guarded([&] {
        if (!timings && m && m <= kReplayMaxEdges && cfg && cfg->center_begin == 0 &&
            (cfg->center_end == 0 || cfg->center_end == n) && replay_enabled())
            return count_edges_replay(src, dst, t, m, n, device_ptrs, stream, cfg, raw, census36);
        double index_ms = 0, ingest_ms = 0;
        RunHint hint;
        if (cfg) hint = hint_for(cfg, n);
        tm_graph* G = build_impl(src, dst, t, m, n, device_ptrs, stream, timings ? &index_ms : nullptr,
                                 cfg ? &hint : nullptr, &ingest_ms);
        int rc;
        try {
            rc = run_parallel_impl(G, cfg, raw, census36, timings);
        } catch (...) {
            free_impl(G);
            throw;
        }
        free_impl(G);
        if (timings) {
            timings->index_ms = index_ms;
            timings->ingest_ms = ingest_ms;
        }
        return rc;
    });
}

int tm_parse_edge_list(const char* text, uint64_t bytes, int device_text, int drop_self_loops, void* stream,
                       tm_edge_list** out) {
    return guarded([&] {
        if (!out || (bytes && !text)) throw tm_error(TM_ERR_INVALID, "null argument");
        ensure_device();
        auto* el = new tm_edge_list();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (!s) {
            TM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            el->own_stream = true;
        }
        el->P.stream = s;
        try {
            // a private copy of the text: the node-id tokens point into it
            unsigned char* d_text = dalloc<unsigned char>(bytes + 16, s);
            if (bytes)
                TM_CUDA(cudaMemcpyAsync(d_text, text, bytes,
                                        device_text ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
            try {
                el->P = parse_edge_list_device(d_text, bytes, drop_self_loops != 0, s);
            } catch (...) {
                dfree(d_text, s);
                throw;
            }
            el->P.text = d_text;
            el->P.bytes = bytes;
            el->P.stream = s;
            if (el->P.n) {  // sum of token lengths + separators
                uint64_t ib = 0;
                uint64_t* pos = dalloc<uint64_t>(el->P.n + 1, s);
                exclusive_scan<uint64_t>(IdLenLoad{el->P.node_len}, el->P.n, pos, s);
                TM_CUDA(cudaMemcpyAsync(&ib, pos + el->P.n, 8, cudaMemcpyDeviceToHost, s));
                dfree(pos, s);
                TM_CUDA(cudaStreamSynchronize(s));
                el->id_bytes = ib - 1;
            }
        } catch (const parse_error& e) {
            g_parse_line = e.line;
            cudaStreamSynchronize(s);
            if (el->own_stream) cudaStreamDestroy(s);
            delete el;
            throw;
        } catch (...) {
            cudaStreamSynchronize(s);
            if (el->own_stream) cudaStreamDestroy(s);
            delete el;
            throw;
        }
        *out = el;
        return TM_OK;
    });
}

int tm_edge_list_info(const tm_edge_list* el, uint64_t* nodes, uint64_t* edges, uint64_t* dropped,
                      uint64_t* id_bytes) {
    if (!el) return TM_ERR_INVALID;
    if (nodes) *nodes = el->P.n;
    if (edges) *edges = el->P.m;
    if (dropped) *dropped = el->P.dropped;
    if (id_bytes) *id_bytes = el->id_bytes;
    return TM_OK;
}

int tm_edge_list_device_arrays(const tm_edge_list* el, const uint32_t** src, const uint32_t** dst,
                               const int64_t** t) {
    if (!el) return TM_ERR_INVALID;
    if (src) *src = el->P.src;
    if (dst) *dst = el->P.dst;
    if (t) *t = el->P.t;
    return TM_OK;
}

int tm_edge_list_copy(const tm_edge_list* el, uint32_t* src, uint32_t* dst, int64_t* t, char* ids) {
    return guarded([&] {
        if (!el) throw tm_error(TM_ERR_INVALID, "null edge list");
        const ParsedEdges& P = el->P;
        cudaStream_t s = P.stream;
        if (src && P.m) TM_CUDA(cudaMemcpyAsync(src, P.src, P.m * 4, cudaMemcpyDeviceToHost, s));
        if (dst && P.m) TM_CUDA(cudaMemcpyAsync(dst, P.dst, P.m * 4, cudaMemcpyDeviceToHost, s));
        if (t && P.m) TM_CUDA(cudaMemcpyAsync(t, P.t, P.m * 8, cudaMemcpyDeviceToHost, s));
        if (ids && P.n) {
            uint64_t* pos = dalloc<uint64_t>(P.n + 1, s);
            exclusive_scan<uint64_t>(IdLenLoad{P.node_len}, P.n, pos, s);
            char* d_ids = dalloc<char>(el->id_bytes + 1, s);
            const unsigned g = (unsigned)std::min<uint64_t>((P.n + 255) / 256, (uint64_t)sm_count() * 8);
            TM_LAUNCH("parse_gather_ids", s, gather_ids_kernel, g, 256, 0, P.text, P.node_off, P.node_len, pos, P.n,
                      d_ids);
            TM_CUDA(cudaMemcpyAsync(ids, d_ids, el->id_bytes, cudaMemcpyDeviceToHost, s));
            dfree(d_ids, s);
            dfree(pos, s);
        }
        TM_CUDA(cudaStreamSynchronize(s));
        return TM_OK;
    });
}

uint64_t tm_parse_error_line(void) { return g_parse_line; }

int tm_write_edge_list(const uint32_t* src, const uint32_t* dst, const int64_t* t, uint64_t m, int device_ptrs,
                       void* stream, char* out, int device_out, uint64_t* bytes) {
    return guarded([&] {
        if (!bytes || (m && (!src || !dst || !t))) throw tm_error(TM_ERR_INVALID, "null argument");
        ensure_device();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        bool own = false;
        if (!s) {
            TM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            own = true;
        }
        const uint32_t *ds = src, *dd = dst;
        const int64_t* dt = t;
        uint32_t *hs = nullptr, *hd = nullptr;
        int64_t* ht = nullptr;
        if (!device_ptrs && m) {
            hs = dalloc<uint32_t>(m, s);
            hd = dalloc<uint32_t>(m, s);
            ht = dalloc<int64_t>(m, s);
            TM_CUDA(cudaMemcpyAsync(hs, src, m * 4, cudaMemcpyHostToDevice, s));
            TM_CUDA(cudaMemcpyAsync(hd, dst, m * 4, cudaMemcpyHostToDevice, s));
            TM_CUDA(cudaMemcpyAsync(ht, t, m * 8, cudaMemcpyHostToDevice, s));
            ds = hs;
            dd = hd;
            dt = ht;
        }
        const uint64_t nb = edge_list_text_bytes(ds, dd, dt, m, s);
        *bytes = nb;
        if (out && nb) {
            char* d_out = device_out ? out : dalloc<char>(nb, s);
            write_edge_list_device(ds, dd, dt, m, d_out, s);
            if (!device_out) {
                TM_CUDA(cudaMemcpyAsync(out, d_out, nb, cudaMemcpyDeviceToHost, s));
                dfree(d_out, s);
            }
        }
        dfree(hs, s);
        dfree(hd, s);
        dfree(ht, s);
        TM_CUDA(cudaStreamSynchronize(s));
        if (own) cudaStreamDestroy(s);
        return TM_OK;
    });
}

void tm_edge_list_free(tm_edge_list* el) {
    if (!el) return;
    cudaStream_t s = el->P.stream;
    free_parsed(el->P);
    cudaStreamSynchronize(s);
    if (el->own_stream) cudaStreamDestroy(s);
    delete el;
}

int tm_count_edges_async(const uint32_t* src, const uint32_t* dst, const int64_t* t, uint64_t m,
                         uint64_t n, void* stream, const tm_run_config* cfg, uint64_t* ticket) {
    return guarded([&] {
        ensure_device();
        check_config(cfg);
        if (!ticket || (m && (!src || !dst || !t))) throw tm_error(TM_ERR_INVALID, "null argument");
        if (cfg->center_begin != 0 || (cfg->center_end != 0 && cfg->center_end != n))
            throw tm_error(TM_ERR_CONFIG, "asynchronous census: whole-graph runs only");
        AsyncPipe& A = g_async;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (!s) {
            if (!g_replay.own) TM_CUDA(cudaStreamCreateWithFlags(&g_replay.own, cudaStreamNonBlocking));
            s = g_replay.own;
        }
        if (!A.copy) TM_CUDA(cudaStreamCreateWithFlags(&A.copy, cudaStreamNonBlocking));
        const uint64_t tk = A.next++;
        AsyncSlot& sl = A.slot[tk & 1];
        if (sl.busy) A.finished.emplace_back(sl.ticket, finish_slot(sl));  // oldest batch first
        if (!sl.copied) {
            TM_CUDA(cudaEventCreateWithFlags(&sl.copied, cudaEventDisableTiming));
            TM_CUDA(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
            TM_CUDA(cudaEventRecord(sl.done, s));
        }
        if (sl.cap < m) {  // (re)size the staging buffers once the slot is idle
            TM_CUDA(cudaEventSynchronize(sl.done));
            if (sl.ds) {
                cudaFree(sl.ds);
                cudaFree(sl.dd);
                cudaFree(sl.dt);
            }
            TM_CUDA(cudaMalloc(&sl.ds, m * sizeof(uint32_t)));
            TM_CUDA(cudaMalloc(&sl.dd, m * sizeof(uint32_t)));
            TM_CUDA(cudaMalloc(&sl.dt, m * sizeof(int64_t)));
            sl.cap = m;
        }
        sl.busy = true;
        sl.ticket = tk;
        sl.m = m;
        sl.n = n;
        sl.s = s;
        sl.cfg = *cfg;
        sl.pending = false;
        sl.deferred = false;
        sl.res = AsyncResult();
        // copy stream: wait until the slot's previous census stopped reading it
        TM_CUDA(cudaStreamWaitEvent(A.copy, sl.done, 0));
        const bool eager = m && !(m <= kReplayMaxEdges && replay_enabled());
        bool pack = eager && m >= pack_min_edges() && pack_enabled();
        if (pack && sl.pack_cap < m) {  // pinned staging + device copies of the packed timestamps
            if (sl.h_off) {
                cudaFreeHost(sl.h_off);
                cudaFreeHost(sl.h_base);
                cudaFree(sl.d_off);
                cudaFree(sl.d_base);
                sl.h_off = nullptr;
                sl.pack_cap = 0;
            }
            const uint64_t nb = (m + kPackBlock16 - 1) / kPackBlock16;  // room for either block size
            if (cudaHostAlloc(&sl.h_off, m * sizeof(uint32_t), cudaHostAllocDefault) == cudaSuccess &&
                cudaHostAlloc(&sl.h_base, nb * sizeof(int64_t), cudaHostAllocDefault) == cudaSuccess &&
                cudaMalloc(&sl.d_off, m * sizeof(uint32_t)) == cudaSuccess &&
                cudaMalloc(&sl.d_base, nb * sizeof(int64_t)) == cudaSuccess) {
                sl.pack_cap = m;
            } else {  // no room for the staging: plain copies
                cudaGetLastError();
                if (sl.h_off) cudaFreeHost(sl.h_off);
                if (sl.h_base) cudaFreeHost(sl.h_base);
                if (sl.d_off) cudaFree(sl.d_off);
                if (sl.d_base) cudaFree(sl.d_base);
                sl.h_off = nullptr;
                sl.h_base = nullptr;
                sl.d_off = nullptr;
                sl.d_base = nullptr;
                pack = false;
            }
        }
        sl.packed = pack;
        sl.host_t = t;
        if (pack) {  // workers pack t while src / dst are on the wire
            sl.job.reset(new PackJob());
            sl.job->t = t;
            sl.job->m = m;
            sl.job->off = sl.h_off;
            sl.job->base = sl.h_base;
            sl.job->width = (A.t_width == 2 && pack16_enabled()) ? 2 : 4;
            pack_start(*sl.job);
        }
        if (m) {
            TM_CUDA(cudaMemcpyAsync(sl.ds, src, m * sizeof(uint32_t), cudaMemcpyHostToDevice, A.copy));
            TM_CUDA(cudaMemcpyAsync(sl.dd, dst, m * sizeof(uint32_t), cudaMemcpyHostToDevice, A.copy));
            if (pack) {
                const uint64_t w = (uint64_t)sl.job->width, blk = w == 2 ? kPackBlock16 : kPackBlock;
                const uint64_t nb = (m + blk - 1) / blk;
                sl.waits.resize(sl.job->pieces);
                for (uint64_t p = 0; p < sl.job->pieces; ++p) {
                    const uint64_t b = p * kPackPiece, e = std::min(m, b + kPackPiece);
                    sl.waits[p] = PieceWait{sl.job.get(), p};
                    TM_CUDA(cudaLaunchHostFunc(A.copy, pack_wait_cb, &sl.waits[p]));
                    TM_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(sl.d_off) + b * w,
                                            reinterpret_cast<const char*>(sl.h_off) + b * w, (e - b) * w,
                                            cudaMemcpyHostToDevice, A.copy));
                }
                TM_CUDA(cudaMemcpyAsync(sl.d_base, sl.h_base, nb * sizeof(int64_t), cudaMemcpyHostToDevice, A.copy));
                const unsigned ugrid = (unsigned)std::min<uint64_t>((m + 255) / 256, (uint64_t)sm_count() * 8);
                if (w == 2) {
                    TM_LAUNCH("unpack_t", A.copy, (unpack_t_kernel<uint16_t, kPackBlock16>), ugrid, 256, 0,
                              reinterpret_cast<const uint16_t*>(sl.d_off), sl.d_base, m, sl.dt);
                } else {
                    TM_LAUNCH("unpack_t", A.copy, (unpack_t_kernel<uint32_t, kPackBlock>), ugrid, 256, 0, sl.d_off,
                              sl.d_base, m, sl.dt);
                }
                g_h2d_bytes.store(m * (8 + w) + nb * 8);
            } else {
                TM_CUDA(cudaMemcpyAsync(sl.dt, t, m * sizeof(int64_t), cudaMemcpyHostToDevice, A.copy));
                g_h2d_bytes.store(m * 16);
            }
        } else {
            g_h2d_bytes.store(0);
        }
        TM_CUDA(cudaEventRecord(sl.copied, A.copy));
        // the previous batch's deferred census runs now, while this copy is in
        // flight -- before `s` is made to wait for it
        AsyncSlot& prev = A.slot[(tk & 1) ^ 1];
        if (prev.busy && prev.deferred) {
            try {
                run_deferred(prev);
            } catch (const tm_error& e) {
                prev.res.rc = e.code;
                prev.res.err = e.what();
            }
        }
        TM_CUDA(cudaStreamWaitEvent(s, sl.copied, 0));
        if (eager) {
            sl.deferred = true;  // eager (host-synchronous) count: issued with the next submission or the wait
            *ticket = tk;
            return TM_OK;
        }
        try {
            const int rc = m ? count_edges_replay(sl.ds, sl.dd, sl.dt, m, n, 1, s, cfg, &sl.res.raw, sl.res.census,
                                                  &sl.P)
                             : tm_count_edges(sl.ds, sl.dd, sl.dt, m, n, 1, s, cfg, &sl.res.raw, sl.res.census,
                                              nullptr);
            sl.pending = rc == kPending;
            if (!sl.pending) {
                sl.res.rc = rc;
                if (rc != TM_OK) sl.res.err = g_last_error;
            }
        } catch (const tm_error& e) {
            sl.res.rc = e.code;
            sl.res.err = e.what();
        }
        TM_CUDA(cudaEventRecord(sl.done, s));
        *ticket = tk;
        return TM_OK;
    });
}

int tm_async_h2d_bytes(uint64_t* bytes) {
    if (!bytes) return TM_ERR_INVALID;
    *bytes = g_h2d_bytes.load();
    return TM_OK;
}

int tm_count_edges_wait(uint64_t ticket, tm_counters* raw, uint64_t* census36) {
    return guarded([&] {
        AsyncPipe& A = g_async;
        AsyncResult res;
        bool found = false;
        for (size_t i = 0; i < A.finished.size(); ++i)
            if (A.finished[i].first == ticket) {
                res = A.finished[i].second;
                A.finished.erase(A.finished.begin() + i);
                found = true;
                break;
            }
        if (!found) {
            AsyncSlot& sl = A.slot[ticket & 1];
            if (!sl.busy || sl.ticket != ticket) throw tm_error(TM_ERR_INVALID, "unknown or already collected ticket");
            res = finish_slot(sl);
        }
        if (res.rc != TM_OK) throw tm_error(res.rc, res.err.empty() ? "census failed" : res.err);
        if (raw) *raw = res.raw;
        if (census36) std::memcpy(census36, res.census, sizeof(res.census));
        return TM_OK;
    });
}

int tm_count_edges_time_slice(const uint32_t* src, const uint32_t* dst, const int64_t* t, uint64_t m,
                              uint64_t n, int device_ptrs, void* stream, const tm_run_config* cfg,
                              int has_lo, int64_t t_lo, int has_hi, int64_t t_hi, tm_counters* raw,
                              tm_phase_timings* timings) {
    return guarded([&] {
        if (!cfg) throw tm_error(TM_ERR_INVALID, "null config");
        if (cfg->delta < 0) throw tm_error(TM_ERR_CONFIG, "delta must be >= 0");
        ensure_device();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        bool own = false;
        if (!s) {
            TM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            own = true;
        }
        const uint32_t *ds = src, *dd = dst;
        const int64_t* dt = t;
        uint32_t *hs = nullptr, *hd = nullptr, *os = nullptr, *od = nullptr;
        int64_t *ht = nullptr, *ot = nullptr;
        tm_graph* G = nullptr;
        int rc = TM_OK;
        try {
            if (!device_ptrs && m) {
                hs = dalloc<uint32_t>(m, s);
                hd = dalloc<uint32_t>(m, s);
                ht = dalloc<int64_t>(m, s);
                TM_CUDA(cudaMemcpyAsync(hs, src, m * 4, cudaMemcpyHostToDevice, s));
                TM_CUDA(cudaMemcpyAsync(hd, dst, m * 4, cudaMemcpyHostToDevice, s));
                TM_CUDA(cudaMemcpyAsync(ht, t, m * 8, cudaMemcpyHostToDevice, s));
                ds = hs;
                dd = hd;
                dt = ht;
            }
            // edges of instances whose first edge starts in [t_lo, t_hi):
            // t_lo <= t <= t_hi - 1 + delta (saturating; an open end keeps every t)
            const int64_t lo = has_lo ? t_lo : INT64_MIN;
            const int64_t hi = !has_hi ? INT64_MAX : t_hi == INT64_MIN ? INT64_MIN : sat_add(t_hi - 1, cfg->delta);
            uint64_t ms = 0;
            if (has_lo || has_hi) ms = slice_edges(ds, dd, dt, m, lo, hi, &os, &od, &ot, s);
            tm_run_config c = *cfg;
            c.has_first_edge_t_end = has_hi ? 1 : 0;
            c.first_edge_t_end = t_hi;
            double index_ms = 0;
            if (has_lo || has_hi)
                G = build_impl(os, od, ot, ms, n, 1, s, timings ? &index_ms : nullptr);
            else
                G = build_impl(ds, dd, dt, m, n, 1, s, timings ? &index_ms : nullptr);
            rc = run_parallel_impl(G, &c, raw, nullptr, timings);
            if (timings) timings->index_ms = index_ms;
        } catch (...) {
            if (G) free_impl(G);
            dfree(os, s); dfree(od, s); dfree(ot, s); dfree(hs, s); dfree(hd, s); dfree(ht, s);
            if (own) cudaStreamDestroy(s);
            throw;
        }
        free_impl(G);
        dfree(os, s); dfree(od, s); dfree(ot, s); dfree(hs, s); dfree(hd, s); dfree(ht, s);
        TM_CUDA(cudaStreamSynchronize(s));
        if (own) cudaStreamDestroy(s);
        return rc;
    });
}

int tm_partition_centers(const tm_graph* g, uint32_t world, uint32_t rank, uint32_t* begin,
                         uint32_t* end) {
    return guarded([&] {
        if (world == 0 || rank >= world) throw tm_error(TM_ERR_INVALID, "bad rank/world");
        auto* G = const_cast<tm_graph*>(g);
        const uint64_t n = G->g.n;
        const auto& off = host_off(G);
        // cost(u) = |S_u| + |F_u| (star records + forward wedges' first edges)
        build_forward(G->g, 0, G->g.stream);
        std::vector<uint32_t> foff(n + 1);
        TM_CUDA(cudaMemcpyAsync(foff.data(), G->g.fwd[0].off, (n + 1) * 4, cudaMemcpyDeviceToHost,
                                G->g.stream));
        TM_CUDA(cudaStreamSynchronize(G->g.stream));
        const uint64_t total = (uint64_t)off[n] + foff[n];
        auto bound = [&](uint64_t r) -> uint32_t {
            if (r == 0) return 0;
            if (r >= world) return (uint32_t)n;
            const uint64_t target = total * r / world;
            uint64_t lo = 0, hi = n;  // first u with cost prefix >= target
            while (lo < hi) {
                const uint64_t mid = (lo + hi) / 2;
                if ((uint64_t)off[mid] + foff[mid] < target) lo = mid + 1; else hi = mid;
            }
            return (uint32_t)lo;
        };
        *begin = bound(rank);
        *end = bound(rank + 1);
        return TM_OK;
    });
}

void tm_debug_acc_bias(uint64_t bias) { g_acc_bias = bias; }

int tm_merge_census(const uint64_t* star24, const uint64_t* pair8, const uint64_t* tri24, int mode,
                    uint64_t* census36) {
    return guarded([&] { return merge_census_impl(star24, pair8, tri24, mode, census36); });
}

int tm_signature(int idx, char* out9) {
    const auto& u = universe();
    if (idx < 0 || idx >= (int)u.all.size()) return TM_ERR_INVALID;
    std::memcpy(out9, u.all[idx].c_str(), 9);
    return TM_OK;
}

int tm_cell_signature(int kind, int cell) {
    const auto& u = universe();
    if (kind == 0 && cell >= 0 && cell < 24) return u.star_sig[cell];
    if (kind == 1 && cell >= 0 && cell < 8) return u.pair_sig[cell];
    if (kind == 2 && cell >= 0 && cell < 24) return u.tri_sig[cell];
    return -1;
}

int tm_signature_label(int idx, char* out16) {
    // anchored M_ij names (motifs.cpp:207-219); others label as themselves
    static const std::map<std::string, std::string> anchors = {
        {"12|23|32", "M_24"}, {"12|31|23", "M_25"}, {"12|23|31", "M_26"},
        {"12|32|31", "M_46"}, {"12|12|12", "M_55"}, {"12|21|21", "M_56"},
        {"12|12|31", "M_63"}, {"12|21|12", "M_65"}, {"12|12|21", "M_66"},
    };
    const auto& u = universe();
    if (idx < 0 || idx >= (int)u.all.size()) return TM_ERR_INVALID;
    auto it = anchors.find(u.all[idx]);
    const std::string& s = it != anchors.end() ? it->second : u.all[idx];
    std::memcpy(out16, s.c_str(), s.size() + 1);
    return TM_OK;
}

int tm_generate_random_graph(uint64_t nodes, uint64_t m, int64_t t_max, uint64_t seed, uint32_t* src,
                             uint32_t* dst, int64_t* t) {
    if (m > 0 && nodes < 2) {
        g_last_error = "need at least 2 nodes to place edges";
        return TM_ERR_INVALID;
    }
    if (t_max < 0) {
        g_last_error = "t_max must be non-negative";
        return TM_ERR_INVALID;
    }
    std::mt19937_64 rng(seed);
    auto draw = [&](uint64_t bound) -> uint64_t {
        if (bound == 0) return 0;
        const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
        uint64_t x;
        do {
            x = rng();
        } while (x >= limit);
        return x % bound;
    };
    for (uint64_t i = 0; i < m; ++i) {
        const uint32_t s = (uint32_t)draw(nodes);
        const uint32_t o = (uint32_t)draw(nodes - 1);
        src[i] = s;
        dst[i] = o + (o >= s ? 1 : 0);
        t[i] = (int64_t)draw((uint64_t)t_max + 1);
    }
    return TM_OK;
}

int tm_run_stats(const tm_graph* g, uint64_t* out8) {
    if (!g || !out8) return TM_ERR_INVALID;
    std::memcpy(out8, g->g.stats, 8 * sizeof(uint64_t));
    return TM_OK;
}

const char* tm_last_error(void) { return g_last_error.c_str(); }
uint64_t tm_kernel_launches(void) { return g_launches.load(); }
void tm_kernel_timing_enable(int on) { g_timing.store(on ? 1 : 0); }

void tm_kernel_timing_reset(void) {
    std::lock_guard<std::mutex> lk(g_timing_mu);
    for (auto& p : g_pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    g_pending.clear();
    g_ktotals.clear();
}

int tm_kernel_timing_get(const char* name, double* total_ms, uint64_t* launches) {
    std::lock_guard<std::mutex> lk(g_timing_mu);
    for (auto& p : g_pending) {
        cudaEventSynchronize(p.b);
        float ms = 0;
        cudaEventElapsedTime(&ms, p.a, p.b);
        auto& tot = g_ktotals[p.name];
        tot.first += ms;
        tot.second += 1;
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    g_pending.clear();
    auto it = g_ktotals.find(name);
    if (total_ms) *total_ms = it == g_ktotals.end() ? 0.0 : it->second.first;
    if (launches) *launches = it == g_ktotals.end() ? 0 : it->second.second;
    return TM_OK;
}

}  // extern "C"
