// tm_tri.cu -- FAST-Tri (Algorithm 2, triangle_engine.cpp:20-62) on B200.
//
// Per center u, every in-window pair (e_i, e_j) of incident edges to distinct
// neighbours v, w is a wedge; the closing edges are the v-w records with
// t in [t_j - delta, t_i + delta], typed I/II/III by their (t, ordinal) place
// relative to e_i and e_j (triangle_engine.cpp:10-16, 43-51).  The v-w list
// is the P group {min, max} (PairEdgeIndex), found by a binary search of max
// in min's block; short groups are classified record by record, long ones by
// four binary searches for the window and the I/II/III boundaries.
//
// Full-graph passes run on the forward-oriented sequences F (each edge kept
// at one endpoint under a strict total order), so every triangle instance is
// enumerated exactly once, at its lowest-ranked vertex:
//   * node-index order  == the reference's removal mode (alive = later nodes),
//     giving Tri cells identical to count_triangles(removal);
//   * (degree class, id) order == the same instances with hubs last, used for
//     count_all: each instance lands once in every cell of its isomorphism
//     class (one per type, motifs.cpp fibers), so the host expands class sums
//     into the reference's count_all cells.
// Per-center work items (count_triangles_at_center with ranges / live mask)
// use the unoriented S sequences exactly as the reference does.
#include "tm_primitives.cuh"

namespace tmb {

namespace {

// counts of closing records for one wedge: c[type*2 + dk], dk relative to v.
// The v-w list is the P group {min, max}: lower_bound of max in min's block.
// t_last restricts to instances whose earliest edge has t <= t_last (time-slice
// partitions; INT64_MAX = no bound): the closing edge itself for type I, e_i
// otherwise.
constexpr uint32_t kTableMinBlock = 256;

// (t, ordinal) strict order of P record k before the record key
__device__ __forceinline__ bool p_before(const PView& P, uint32_t k, const RecKey& key) {
    const int c = P.t.cmp(k, key);
    return c < 0 || (c == 0 && P.ord[k] < key.ord);
}
// first k in [from, end) with (t, ord) >= the record key, galloping up from
// `from` (the boundaries of one window are close together)
__device__ __forceinline__ uint32_t p_gallop_rec(const PView& P, uint32_t from, uint32_t end, const RecKey& key) {
    uint32_t lo = from, hi = end;
    for (uint32_t span = 1;; span <<= 1) {
        const uint64_t probe = (uint64_t)lo + span - 1;
        if (probe >= end) break;
        if (!p_before(P, (uint32_t)probe, key)) {
            hi = (uint32_t)probe;
            break;
        }
        lo = (uint32_t)probe + 1;
    }
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (p_before(P, mid, key)) lo = mid + 1; else hi = mid;
    }
    return lo;
}
// first k in [from, end) whose time is not below the threshold key (key_below(x):
// first t >= x; key_upto(x): first t > x), galloping up from `from`
__device__ __forceinline__ uint32_t p_gallop_t(const PView& P, uint32_t from, uint32_t end, const TimeKey& key) {
    uint32_t lo = from, hi = end;
    for (uint32_t span = 1;; span <<= 1) {
        const uint64_t probe = (uint64_t)lo + span - 1;
        if (probe >= end) break;
        if (!P.t.below(probe, key)) {
            hi = (uint32_t)probe;
            break;
        }
        lo = (uint32_t)probe + 1;
    }
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (P.t.below(mid, key)) lo = mid + 1; else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ uint32_t p_gallop_tupper(const PView& P, uint32_t from, uint32_t end, int64_t x) {
    return p_gallop_t(P, from, end, P.t.key_upto(x));
}

// One path for every group, short or long: the lanes of a warp hold wedges
// whose closing groups range from one record to hundreds of thousands (hub
// pairs), and a per-length special case made the warp execute both paths.
// Group [kb, ke) by the fenced block search and the group end; then the
// window [k1, k4) = [t_j - delta, t_i + delta] and the type boundaries k2 =
// (t_i, o_i), k3 = (t_j, o_j) (triangle_engine.cpp:43-51): k1 by the fenced
// search, k2, k3, k4 each by a gallop from the previous boundary.
// A wedge's closing group, found (locate_closing) and counted (count_closing).
// (Parking the located wedges in shared memory and counting them 32 at a time,
// so that count_closing runs with every lane busy, measured slower: config 4
// delta 3600 tri_wedge 18.5 -> 27.3 ms, tri_mid 17.4 -> 21.8 ms.)
struct GroupRef {
    uint32_t kb;   // first record of the v-w group
    uint32_t aux;  // the end of its block, or (bit 31 set) the group end itself
};
constexpr uint32_t kGroupEndKnown = 0x80000000u;

__device__ __forceinline__ bool locate_closing(const PView& P, uint32_t v, uint32_t w, GroupRef& g) {
    const bool vlow = ranks_below(P.cls, v, w);
    const uint32_t a = vlow ? v : w, b = vlow ? w : v;  // the pair's lower / upper endpoint (P block of a)
    const uint32_t blk_end = P.pofs[a + 1];
    if (P.pt_keys && blk_end - P.pofs[a] > kTableMinBlock) {  // optional pair table (TM_PAIR_TABLE)
        const unsigned long long key = ((unsigned long long)a << 32) | b;
        uint64_t slot = pair_slot(a, b) & P.pt_mask;
        for (;;) {
            const unsigned long long kk = P.pt_keys[slot];
            if (kk == key) break;
            if (kk == kPairEmpty) return false;  // no v-w record
            slot = (slot + 1) & P.pt_mask;
        }
        const unsigned long long val = P.pt_vals[slot];
        g.kb = (uint32_t)(val >> 32);
        g.aux = (g.kb + (uint32_t)val) | kGroupEndKnown;
        return true;
    }
    g.kb = p_max_lower(P, P.pofs[a], blk_end, b);
    g.aux = blk_end;
    return g.kb < blk_end && P.max[g.kb] == b;
}

__device__ __forceinline__ void count_closing(const PView& P, uint32_t v, uint32_t w, const GroupRef g, int64_t lo,
                                              int64_t hi, int64_t ti, uint32_t oi, int64_t tj, uint32_t oj,
                                              int64_t t_last, uint32_t c[6]) {
    const bool vlow = ranks_below(P.cls, v, w);
    const uint32_t flip = vlow ? 0u : 1u;  // dir_rel_lower -> dir relative to v
    const uint32_t kb = g.kb;
    const uint32_t ke = (g.aux & kGroupEndKnown) ? (g.aux & ~kGroupEndKnown)
                        : P.gend                 ? p_group_end(P, kb)
                                                 : p_max_upper(P, kb, g.aux, vlow ? w : v);
    const uint32_t k1 = p_t_lower(P, kb, ke, lo);
    const uint32_t k2 = p_gallop_rec(P, k1, ke, P.t.rec_key(ti, oi));
    const uint32_t k3 = p_gallop_rec(P, k2, ke, P.t.rec_key(tj, oj));
    const uint32_t k4 = p_gallop_tupper(P, k3, ke, hi);
    uint32_t k2e = k2;  // type I records whose own t is at most t_last
    if (t_last != INT64_MAX) {
        uint32_t l = k1, r = k2;
        while (l < r) { const uint32_t mid = (l + r) >> 1; if (P.t[mid] <= t_last) l = mid + 1; else r = mid; }
        k2e = l;
    }
    // direction split of each type range from the P direction prefix
    auto add_range = [&](int type, uint32_t x0, uint32_t x1) {
        if (x1 <= x0) return;
        const uint32_t n1 = p_dir_before(P, x1) - p_dir_before(P, x0);  // dir_rel_min = 1
        const uint32_t n0 = (x1 - x0) - n1;
        c[type * 2] += flip ? n1 : n0;  // static cell indices: c[] stays in registers
        c[type * 2 + 1] += flip ? n0 : n1;
    };
    add_range(0, k1, k2e);
    if (ti <= t_last) {
        add_range(1, k2, k3);
        add_range(2, k3, k4);
    }
}

__device__ __forceinline__ void closing_counts(const PView& P, uint32_t v, uint32_t w, int64_t lo,
                                               int64_t hi, int64_t ti, uint32_t oi, int64_t tj,
                                               uint32_t oj, int64_t t_last, uint32_t c[6]) {
#pragma unroll
    for (int j = 0; j < 6; ++j) c[j] = 0;
    GroupRef g;
    if (!locate_closing(P, v, w, g)) return;
    count_closing(P, v, w, g, lo, hi, ti, oi, tj, oj, t_last, c);
}

// all wedges with first edge i in sequence arrays (T, NBR, ORD) ending at end
template <typename Sink>
__device__ __forceinline__ void wedges_from(const PView& P, const TimeArr& T,
                                            const uint32_t* __restrict__ NBR,
                                            const uint32_t* __restrict__ ORD, uint32_t i,
                                            uint32_t end, int64_t delta,
                                            const uint8_t* __restrict__ live, const Sink& acc) {
    const uint32_t ni = NBR[i];
    const uint32_t v = ni & kNodeMask, di = ni >> 31;
    if (live && !live[v]) return;
    const int64_t ti = T[i];
    const uint32_t oi = ORD[i] & kNodeMask;
    const int64_t lim = sat_add(ti, delta);
    uint64_t a0[6] = {0, 0, 0, 0, 0, 0}, a1[6] = {0, 0, 0, 0, 0, 0};
    for (uint32_t j = i + 1; j < end; ++j) {
        const int64_t tj = T[j];
        if (tj > lim) break;
        const uint32_t nj = NBR[j];
        const uint32_t w = nj & kNodeMask;
        if (w == v) continue;
        if (live && !live[w]) continue;
        uint32_t c[6];
        closing_counts(P, v, w, sat_sub(tj, delta), lim, ti, oi, tj, ORD[j] & kNodeMask, INT64_MAX, c);
        const uint64_t m1 = (nj >> 31) ? ~0ull : 0ull, m0 = ~m1;
#pragma unroll
        for (int x = 0; x < 6; ++x) {
            a0[x] += c[x] & m0;
            a1[x] += c[x] & m1;
        }
    }
#pragma unroll
    for (int ty = 0; ty < 3; ++ty)
#pragma unroll
        for (int dk = 0; dk < 2; ++dk) {
            acc.add(ty * 8 + (int)di * 4 + 0 + dk, a0[ty * 2 + dk]);
            acc.add(ty * 8 + (int)di * 4 + 2 + dk, a1[ty * 2 + dk]);
        }
}

// Filter + wedge expansion: one pass over F.  Thread i scans the next
// kWedgeScan forward records of its center; every in-window record to a
// different neighbour is a wedge (i, j), reserved warp-aggregated in one
// atomic per warp and written to the wedge list.  A first edge whose window
// runs past kWedgeScan records (or whose wedges do not fit the list) goes to
// the long list instead and is enumerated by tri_long_kernel.
constexpr int kWedgeScan = 8;
#ifndef TM_GCACHE_BITS
#define TM_GCACHE_BITS 7
#endif
#ifndef TM_CACHE_MINB
#define TM_CACHE_MINB 3  // tri_window: config 4 delta 86400 tri_long 884.9 -> 878.6 ms against 4 (profiles/r02/ab)
#endif
constexpr int kGroupCache = 1 << TM_GCACHE_BITS;  // entries per warp (dynamic shared memory)
#ifndef TM_CACHE_MINWIN
#define TM_CACHE_MINWIN 64
#endif
constexpr uint32_t kGroupCacheMinWindow = TM_CACHE_MINWIN;  // shorter windows repeat few groups: plain path

#ifndef TM_WEDGE_MINB
#define TM_WEDGE_MINB 5
#endif
#ifndef TM_LONG_MINB
#define TM_LONG_MINB 5  // tri_mid: 17.6 -> 17.2 ms at config 4 delta 3600, 898 -> 885 ms at 86400 against 6; 4 and 7 lose at 3600
#endif
constexpr int kFilterItems = 4;  // first edges per thread per block iteration (one reservation)
__global__ void __launch_bounds__(256) tri_filter_kernel(TimeArr FT,
                                                         const uint32_t* __restrict__ FN,
                                                         const uint32_t* __restrict__ Fnode,
                                                         int64_t delta, uint32_t fb, uint32_t fe,
                                                         uint64_t* __restrict__ wedges,
                                                         uint64_t wedge_cap,
                                                         uint32_t* __restrict__ long_list,
                                                         uint32_t long_cap,
                                                         unsigned long long* __restrict__ wcount,
                                                         uint32_t* __restrict__ lcount) {
    constexpr uint64_t kStep = 256 * kFilterItems;
    for (uint64_t base = (uint64_t)fb + (uint64_t)blockIdx.x * kStep; base < fe;
         base += (uint64_t)gridDim.x * kStep) {
        uint32_t hits4 = 0;   // byte j: partners (bit s-1 = record i+s) of first edge j
        uint32_t longs = 0;   // bit j: first edge j goes to the long list
#pragma unroll
        for (int jj = 0; jj < kFilterItems; ++jj) {
            const uint64_t i = base + (uint64_t)jj * 256 + threadIdx.x;
            if (i + 1 >= fe) continue;
            const uint32_t node = Fnode[i];
            const uint32_t v = FN[i] & kNodeMask;
            const TimeKey limk = FT.key_upto(sat_add(FT[i], delta));  // in-window: t <= t_i + delta
            bool alive = true;
            uint32_t hits = 0;
#pragma unroll
            for (int s = 1; s <= kWedgeScan; ++s) {
                const uint64_t j = i + s;
                if (alive) {
                    if (j >= fe || Fnode[j] != node || !FT.below(j, limk)) {
                        alive = false;
                    } else if ((FN[j] & kNodeMask) != v) {
                        hits |= 1u << (s - 1);
                    }
                }
            }
            if (alive && i + kWedgeScan + 1 < fe && Fnode[i + kWedgeScan + 1] == node &&
                FT.below(i + kWedgeScan + 1, limk)) {
                // a window past kGroupCacheMinWindow records goes to the very-long
                // list, filled from the back of the same buffer (lcount[1])
                const uint64_t x = i + 1 + kGroupCacheMinWindow;
                if (x < fe && Fnode[x] == node && FT.below(x, limk))
                    long_list[long_cap - 1 - atomicAdd(lcount + 1, 1u)] = (uint32_t)i;
                else
                    longs |= 1u << jj;
            } else
                hits4 |= hits << (8 * jj);
        }
        const uint32_t nw = (uint32_t)__popc(hits4);
        // one block-wide reservation for the wedge slots and the long list
        unsigned long long wo;
        uint32_t lo;
        block_reserve2<8>(nw, (uint32_t)__popc(longs), wcount, lcount, wo, lo);
        for (uint32_t lb = longs; lb; lb &= lb - 1)
            long_list[lo++] = (uint32_t)(base + (uint64_t)(__ffs(lb) - 1) * 256 + threadIdx.x);
        // a reservation past the capacity goes to the long list instead; the
        // lowest such start bounds the valid wedge prefix (every slot below it
        // belongs to a reservation that fit)
        const bool fits = wo + nw <= wedge_cap;
        if (nw && !fits) atomicMin(wcount + 1, wo);
        if (nw && fits) {
            for (uint32_t h = hits4; h; h &= h - 1) {
                const int bit = __ffs(h) - 1;
                const uint64_t i = base + (uint64_t)(bit >> 3) * 256 + threadIdx.x;
                wedges[wo++] = (i << 32) | (uint32_t)(i + (bit & 7) + 1);
            }
        }
        if (nw && !fits) {
            uint32_t firsts = 0;  // first edges with wedges, spilled to the long list
            for (int jj = 0; jj < kFilterItems; ++jj)
                if ((hits4 >> (8 * jj)) & 0xffu) firsts |= 1u << jj;
            const uint32_t o = atomicAdd(lcount, (uint32_t)__popc(firsts));
            uint32_t x = 0;
            for (uint32_t fbits = firsts; fbits; fbits &= fbits - 1)
                long_list[o + x++] = (uint32_t)(base + (uint64_t)(__ffs(fbits) - 1) * 256 + threadIdx.x);
        }
    }
}

// closing counts of wedge (i, j) in F: c[type * 2 + dk]; returns the cell
// base di * 4 + dj * 2 (cells type * 8 + base + dk)
__device__ __forceinline__ int wedge_counts(const PView& P, TimeArr FT, const uint32_t* __restrict__ FN,
                                            const uint32_t* __restrict__ FO, uint32_t i, uint32_t j,
                                            int64_t delta, int64_t t_last, uint32_t c[6]) {
    const uint32_t ni = FN[i], nj = FN[j];
    const int64_t ti = FT[i], tj = FT[j];
    closing_counts(P, ni & kNodeMask, nj & kNodeMask, sat_sub(tj, delta), sat_add(ti, delta), ti,
                   FO[i], tj, FO[j], t_last, c);
    return (int)((ni >> 31) * 4 + (nj >> 31) * 2);
}

// one wedge per thread
__global__ void __launch_bounds__(256, TM_WEDGE_MINB) tri_wedge_kernel(PView P, TimeArr FT,
                                                        const uint32_t* __restrict__ FN,
                                                        const uint32_t* __restrict__ FO,
                                                        int64_t delta, int64_t t_last,
                                                        const uint64_t* __restrict__ wedges,
                                                        uint64_t wedge_cap,
                                                        const unsigned long long* __restrict__ wcount,
                                                        const unsigned long long* __restrict__ wsum,
                                                        uint64_t gend_min, unsigned long long* queue,
                                                        uint64_t* out, uint64_t* stats) {
    __shared__ unsigned long long cells[48];
    if (!P.gend || *wsum < gend_min) P.gend = nullptr;  // group ends not built
    zero_cells(cells, 24);
    __syncthreads();
    WarpCells wc;
    uint64_t cnt = wcount[0] < wedge_cap ? wcount[0] : wedge_cap;
    if (wcount[1] < cnt) cnt = wcount[1];
    if (blockIdx.x == 0 && threadIdx.x == 0 && stats) stats[2] = cnt;
    // Warp-uniform trip count (the cells are reduced across the warp).  When
    // the long windows are many (the group-end gate) closing groups are long
    // and wedge costs heavy-tailed: 32 wedges per warp from the queue;
    // otherwise a fixed grid-stride share (measured: the queue costs ~0.5 %
    // at config 1 delta 3600 and saves 8-10 % at delta 86400).
    const bool dyn = P.gend != nullptr;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t base = dyn ? warp_take(queue, 32) : (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
    for (; base < cnt; base = dyn ? warp_take(queue, 32) : base + stride) {
        const uint64_t idx = base + (threadIdx.x & 31);
        uint32_t c[6] = {0, 0, 0, 0, 0, 0};
        int cb = 0;
        if (idx < cnt) {
            const uint64_t w = wedges[idx];
            cb = wedge_counts(P, FT, FN, FO, (uint32_t)(w >> 32), (uint32_t)w, delta, t_last, c);
        }
        wc.add6(idx < cnt, cb, c, cells, 24);
    }
    wc.flush(cells, 24, 24);
    __syncthreads();
    flush_cells(cells, 24, out, kAccCarry);
}

// first edges with long windows: one warp per first edge, lanes stride the
// in-window records (the HARE intra-node split, per first edge).
//
// The window of a long first edge i (neighbour v) holds records to few
// distinct neighbours w -- the long windows are those of high-degree centers,
// whose forward neighbours are the hubs above them -- so every (v, w) closing
// group is met many times.  Each warp keeps a direct-mapped cache of its
// current first edge's groups (keyed by w): the group [kb, ke), the
// boundaries that depend on e_i only (k2 = first record at or after e_i, k4 =
// first record past t_i + delta) and the last k1 / k3 found.  A hit costs two
// short gallops (k1 and k3 only grow with t_j) instead of the block search,
// the group end and four window searches.
struct GroupCacheEntry {
    uint32_t w, k1, k2, k3, k4, d2, d4, pad;  // d2, d4: direction prefix at k2, k4
};

// first k in [from, end) with t >= x, galloping up from `from`
__device__ __forceinline__ uint32_t p_gallop_tlower(const PView& P, uint32_t from, uint32_t end, int64_t x) {
    return p_gallop_t(P, from, end, P.t.key_below(x));
}

// the v-w group [kb, ke) (empty when no v-w record: kb == ke)
__device__ __forceinline__ void locate_group(const PView& P, uint32_t v, uint32_t w, uint32_t& kb, uint32_t& ke) {
    const bool vlow = ranks_below(P.cls, v, w);
    const uint32_t a = vlow ? v : w, b = vlow ? w : v;
    const uint32_t blk_end = P.pofs[a + 1];
    kb = p_max_lower(P, P.pofs[a], blk_end, b);
    if (kb >= blk_end || P.max[kb] != b) {
        kb = ke = 0;
        return;
    }
    ke = P.gend ? p_group_end(P, kb) : p_max_upper(P, kb, blk_end, b);
}

// Two instantiations share the long list: kCache = false takes the first
// edges whose window holds at most kGroupCacheMinWindow records (one closing
// count per wedge, full occupancy), kCache = true the longer ones (the group
// cache's shared memory costs a resident block per SM).
template <bool kCache>
__global__ void __launch_bounds__(256, kCache ? TM_CACHE_MINB : TM_LONG_MINB) tri_long_kernel(PView P, TimeArr FT,
                                                       const uint32_t* __restrict__ FN,
                                                       const uint32_t* __restrict__ FO,
                                                       const uint32_t* __restrict__ Fnode,
                                                       const uint32_t* __restrict__ Foff,
                                                       int64_t delta, int64_t t_last,
                                                       const uint32_t* __restrict__ list, uint32_t long_cap,
                                                       const uint32_t* __restrict__ lcount,
                                                       const unsigned long long* __restrict__ pt_wsum,
                                                       uint64_t pt_min_wedges, uint64_t gend_min,
                                                       unsigned long long* queue, uint64_t* out,
                                                       uint64_t* stats) {
    __shared__ unsigned long long cells[48];
    extern __shared__ __align__(16) unsigned char gcache_raw[];  // kCache: 8 warps x kGroupCache entries
    zero_cells(cells, 24);
    __syncthreads();
    WarpCells wc;
    // the plain instantiation takes the long list (front), the cached one the
    // very-long list (back of the buffer)
    const uint32_t cnt = lcount[kCache ? 1 : 0];
    if (blockIdx.x == 0 && threadIdx.x == 0 && stats) atomicAdd((unsigned long long*)&stats[3], (unsigned long long)cnt);
    if (!P.gend || *pt_wsum < gend_min) P.gend = nullptr;  // group ends not built
    uint32_t my_wedges = 0;
    const int lane = threadIdx.x & 31;
    GroupCacheEntry* gc = reinterpret_cast<GroupCacheEntry*>(gcache_raw) + (size_t)(threadIdx.x >> 5) * kGroupCache;
    for (;;) {  // one first edge per warp from the queue
        const uint64_t idx = warp_take(queue, 1);
        if (idx >= cnt) break;
        const uint32_t i = kCache ? list[long_cap - 1 - idx] : list[idx];
        const uint32_t end = Foff[Fnode[i] + 1];
        const uint32_t ni = FN[i];
        const uint32_t v = ni & kNodeMask;
        const int64_t ti = FT[i];
        const uint32_t oi = FO[i];
        const int64_t lim = sat_add(ti, delta);
        const TimeKey limk = FT.key_upto(lim);  // in-window: t_j <= t_i + delta
        const RecKey ki = P.t.rec_key(ti, oi);
        // a window of at most kGroupCacheMinWindow records: one closing count
        // per wedge; a longer one goes through the group cache
        const bool longwin = kCache;
        bool more = longwin;
        uint32_t j0 = i + 1;
        for (; !longwin && j0 < end; j0 += 32) {
            const uint32_t j = j0 + lane;
            const bool in = j < end && FT.below(j, limk);
            const bool wedge = in && (FN[j] & kNodeMask) != v;
            uint32_t c[6] = {0, 0, 0, 0, 0, 0};
            int cb = 0;
            if (wedge) {
                cb = wedge_counts(P, FT, FN, FO, i, j, delta, t_last, c);
                ++my_wedges;
            }
            wc.add6(wedge, cb, c, cells, 24);
            if (!__all_sync(0xffffffffu, in)) {
                more = false;
                break;
            }
        }
        if (!more || j0 >= end) continue;
        for (int x = lane; x < kGroupCache; x += 32) gc[x].w = 0xFFFFFFFFu;
        __syncwarp();
        uint32_t misses = 0;
#ifdef TM_TRI_STATS
        uint32_t empties = 0, miss_iters = 0, iters = 0;
#endif
        for (; j0 < end; j0 += 32) {
#ifdef TM_TRI_STATS
            int miss_flag = 0;
#endif
            const uint32_t j = j0 + lane;
            const bool in = j < end && FT.below(j, limk);
            const uint32_t nj = in ? FN[j] : 0u;
            const uint32_t w = nj & kNodeMask;
            const bool wedge = in && w != v;
            uint32_t c[6] = {0, 0, 0, 0, 0, 0};
            int cb = 0;
            const uint32_t slot = (w * 0x9E3779B1u) >> (32 - TM_GCACHE_BITS);
            GroupCacheEntry e;
            if (wedge) {
                const int64_t tj = FT[j];
                const uint32_t oj = FO[j];
                e = gc[slot];
                if (e.w != w) {  // miss: the group and its e_i boundaries
                    ++misses;
#ifdef TM_TRI_STATS
                    miss_flag = 1;
#endif
                    e.w = w;
                    uint32_t kb, ke;
                    locate_group(P, v, w, kb, ke);
#ifdef TM_TRI_STATS
                    if (kb == ke) ++empties;
#endif
                    e.k1 = p_t_lower(P, kb, ke, sat_sub(tj, delta));
                    e.k2 = p_gallop_rec(P, e.k1, ke, ki);
                    e.k4 = p_t_upper(P, e.k2, ke, lim);
                    e.k3 = e.k2;
                    e.d2 = p_dir_before(P, e.k2);
                    e.d4 = p_dir_before(P, e.k4);
                }
                // the window's lower end t_j - delta and e_j only move forward with j
                const uint32_t k1 = p_gallop_tlower(P, e.k1, e.k2, sat_sub(tj, delta));
                const uint32_t k3 = p_gallop_rec(P, e.k3 > e.k2 ? e.k3 : e.k2, e.k4, P.t.rec_key(tj, oj));
                e.k1 = k1;
                e.k3 = k3;
                const uint32_t flip = ranks_below(P.cls, v, w) ? 0u : 1u;
                uint32_t k2e = e.k2;
                if (t_last != INT64_MAX) {
                    uint32_t l = k1, r = e.k2;
                    while (l < r) {
                        const uint32_t mid = (l + r) >> 1;
                        if (P.t[mid] <= t_last) l = mid + 1; else r = mid;
                    }
                    k2e = l;
                }
                // direction split of each type range from the P direction
                // prefix (at k2 and k4 cached per group)
                auto add_range = [&](int type, uint32_t x0, uint32_t d0, uint32_t x1, uint32_t d1) {
                    if (x1 <= x0) return;
                    const uint32_t n1 = d1 - d0;
                    const uint32_t n0 = (x1 - x0) - n1;
                    c[type * 2] += flip ? n1 : n0;  // static cell indices: c[] stays in registers
                    c[type * 2 + 1] += flip ? n0 : n1;
                };
                const uint32_t d1 = p_dir_before(P, k1), d3 = p_dir_before(P, k3);
                add_range(0, k1, d1, k2e, k2e == e.k2 ? e.d2 : p_dir_before(P, k2e));
                if (ti <= t_last) {
                    add_range(1, e.k2, e.d2, k3, d3);
                    add_range(2, k3, d3, e.k4, e.d4);
                }
                cb = (int)((ni >> 31) * 4 + (nj >> 31) * 2);
                ++my_wedges;
            }
            // one writer per cache slot: the highest wedge lane that maps there
            const unsigned peers = __match_any_sync(0xffffffffu, wedge ? slot : 0xFFFFFFFFu);
            if (wedge && (peers >> lane) == 1u) gc[slot] = e;
            __syncwarp();
            wc.add6(wedge, cb, c, cells, 24);
#ifdef TM_TRI_STATS
            ++iters;
            if (__any_sync(0xffffffffu, miss_flag)) ++miss_iters;
#endif
            if (!__all_sync(0xffffffffu, in)) break;
        }
#ifdef TM_TRI_STATS
        empties = warp_sum(empties);
        if (lane == 0 && stats) {
            atomicAdd((unsigned long long*)&stats[6], (unsigned long long)empties);
            atomicAdd((unsigned long long*)&stats[7], ((unsigned long long)miss_iters << 32) | iters);
        }
#endif
        misses = warp_sum(misses);
        if (lane == 0 && misses && stats) atomicAdd((unsigned long long*)&stats[5], (unsigned long long)misses);
    }
    wc.flush(cells, 24, 24);
    my_wedges = warp_sum(my_wedges);
    if (lane == 0 && my_wedges && stats) atomicAdd((unsigned long long*)&stats[4], (unsigned long long)my_wedges);
    __syncthreads();
    flush_cells(cells, 24, out, kAccCarry);
}

// ---- long windows of at most kGroupCacheMinWindow records: flattened ------
//
// tri_long_kernel<false> strides one window with the warp's lanes, so a
// window of 9..31 records leaves most lanes idle (ncu: 14.5 of 32 threads
// active per instruction at config 4, delta 3600).  tri_mid_kernel takes 32
// first edges per warp (one per lane: its window length by a short binary
// search), scans the lengths and walks the concatenated wedge space 32 wedges
// per step -- every lane holds a wedge until the warp's last step; a wedge's
// owner is found by a five-step shuffle search over the scanned lengths.
#ifndef TM_MID_FLAT
#define TM_MID_FLAT 1
#endif
__global__ void __launch_bounds__(256, TM_LONG_MINB) tri_mid_kernel(PView P, TimeArr FT,
                                                       const uint32_t* __restrict__ FN,
                                                       const uint32_t* __restrict__ FO,
                                                       const uint32_t* __restrict__ Fnode,
                                                       const uint32_t* __restrict__ Foff,
                                                       int64_t delta, int64_t t_last,
                                                       const uint32_t* __restrict__ list,
                                                       const uint32_t* __restrict__ lcount,
                                                       const unsigned long long* __restrict__ pt_wsum,
                                                       uint64_t gend_min, unsigned long long* queue,
                                                       uint64_t* out, uint64_t* stats) {
    __shared__ unsigned long long cells[48];
    zero_cells(cells, 24);
    __syncthreads();
    WarpCells wc;
    const uint32_t cnt = lcount[0];  // the long list (front of the buffer)
    if (blockIdx.x == 0 && threadIdx.x == 0 && stats) atomicAdd((unsigned long long*)&stats[3], (unsigned long long)cnt);
    if (!P.gend || *pt_wsum < gend_min) P.gend = nullptr;  // group ends not built
    P.pt_keys = nullptr;
    uint32_t my_wedges = 0;
    const int lane = threadIdx.x & 31;
    // first edges per take: 32, fewer when the list would not reach every warp
    // (config 1 at delta 3600: a few thousand long first edges)
    uint32_t take = 32;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    while (take > 1 && take * warps > cnt) take >>= 1;
    for (;;) {  // `take` first edges per warp from the queue
        const uint64_t base = warp_take(queue, take);
        if (base >= cnt) break;
        uint32_t i = 0, len = 0;
        if ((uint32_t)lane < take && base + lane < cnt) {
            i = list[base + lane];
            const uint32_t end = Foff[Fnode[i] + 1];
            const TimeKey limk = FT.key_upto(sat_add(FT[i], delta));  // in-window: t_j <= t_i + delta
            // first record past the window (the filter saw it end within
            // kGroupCacheMinWindow records; searched on if it does not)
            uint32_t lo = i + 1, hi = end - lo > kGroupCacheMinWindow ? lo + kGroupCacheMinWindow : end;
            const uint32_t cap = hi;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (FT.below(mid, limk)) lo = mid + 1; else hi = mid;
            }
            if (lo == cap && cap < end) {
                hi = end;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (FT.below(mid, limk)) lo = mid + 1; else hi = mid;
                }
            }
            len = lo - (i + 1);
        }
        const uint32_t incl = warp_inclusive_scan(len);
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - len;
        for (uint32_t x0 = 0; x0 < total; x0 += 32) {
            const uint32_t x = x0 + lane;
            int o = 0;  // the first lane whose scanned length exceeds x
#pragma unroll
            for (int step = 16; step; step >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, incl, o + step - 1);
                if (v <= x) o += step;
            }
            const uint32_t io = __shfl_sync(0xffffffffu, i, o);
            const uint32_t so = __shfl_sync(0xffffffffu, excl, o);
            uint32_t c[6] = {0, 0, 0, 0, 0, 0};
            int cb = 0;
            bool wedge = false;
            if (x < total) {
                const uint32_t j = io + 1 + (x - so);
                if ((FN[io] & kNodeMask) != (FN[j] & kNodeMask)) {
                    wedge = true;
                    cb = wedge_counts(P, FT, FN, FO, io, j, delta, t_last, c);
                    ++my_wedges;
                }
            }
            wc.add6(wedge, cb, c, cells, 24);
        }
    }
    wc.flush(cells, 24, 24);
    my_wedges = warp_sum(my_wedges);
    if (lane == 0 && my_wedges && stats) atomicAdd((unsigned long long*)&stats[4], (unsigned long long)my_wedges);
    __syncthreads();
    flush_cells(cells, 24, out, kAccCarry);
}

// ---- very long windows: resolve-then-count -------------------------------
//
// tri_long_kernel<true> looks a group up the first time a lane meets it, so in
// nearly every 32-record step a few lanes run the whole lookup (block search,
// group end, four window searches) while the others wait.  tri_window_kernel
// splits each window segment in two passes over the same records (they stay
// in L1):
//   A. collect the neighbours w the warp's table does not hold yet -- one
//      claim per distinct w, appended to a pending list -- and resolve the
//      pending groups 32 at a time, one per lane, so lookups run with every
//      lane busy;
//   B. count: every wedge finds its group in the table (linear probing, a
//      handful of slots) and pays two short gallops for k1 / k3, which only
//      grow with j; a group with no record inside [t_j - delta, t_i + delta]
//      is skipped on its cached bounds.
// The table lives for one first edge (k2, k4 and the direction prefixes there
// depend on e_i only) and is cleared between segments once half full; a
// neighbour that finds no free slot within kGcProbes falls back to the
// one-off closing count.
#ifndef TM_LONG_SEG
#define TM_LONG_SEG 128
#endif
constexpr uint32_t kGcEmpty = 0xFFFFFFFFu;
constexpr int kGcProbes = 4;
constexpr uint32_t kLongSeg = TM_LONG_SEG;  // window records per resolve / count segment
static_assert(kLongSeg % 32 == 0, "segments are whole 32-record steps");

// slot of w in the warp's table (found), else the first empty slot on its
// probe path (found = false), else -1 (no room within kGcProbes)
__device__ __forceinline__ int gc_probe(const GroupCacheEntry* gc, uint32_t w, bool& found) {
    const uint32_t h = (w * 0x9E3779B1u) >> (32 - TM_GCACHE_BITS);
    found = false;
#pragma unroll
    for (int p = 0; p < kGcProbes; ++p) {
        const uint32_t s = (h + p) & (kGroupCache - 1);
        const uint32_t tag = gc[s].w;
        if (tag == w) {
            found = true;
            return (int)s;
        }
        if (tag == kGcEmpty) return (int)s;
    }
    return -1;
}

// fill the claimed entry of neighbour w, first met at window record j
__device__ __forceinline__ void gc_resolve(const PView& P, const TimeArr& FT, GroupCacheEntry* gc, uint32_t v,
                                           uint32_t w, uint32_t j, int64_t delta, const RecKey& ki, int64_t lim) {
    GroupCacheEntry e;
    e.w = w;
    uint32_t kb, ke;
    locate_group(P, v, w, kb, ke);
    e.k1 = p_t_lower(P, kb, ke, sat_sub(FT[j], delta));
    e.k2 = p_gallop_rec(P, e.k1, ke, ki);
    e.k4 = p_t_upper(P, e.k2, ke, lim);
    e.k3 = e.k2;
    e.d2 = p_dir_before(P, e.k2);
    e.d4 = p_dir_before(P, e.k4);
    e.pad = ranks_below(P.cls, v, w) ? 0u : 1u;  // dir_rel_lower -> dir relative to v
    bool found;
    const int slot = gc_probe(gc, w, found);  // the slot claimed for w
    gc[slot] = e;
}

__global__ void __launch_bounds__(256, TM_CACHE_MINB) tri_window_kernel(PView P, TimeArr FT,
                                                       const uint32_t* __restrict__ FN,
                                                       const uint32_t* __restrict__ FO,
                                                       const uint32_t* __restrict__ Fnode,
                                                       const uint32_t* __restrict__ Foff,
                                                       int64_t delta, int64_t t_last,
                                                       const uint32_t* __restrict__ list, uint32_t long_cap,
                                                       const uint32_t* __restrict__ lcount,
                                                       const unsigned long long* __restrict__ pt_wsum,
                                                       uint64_t gend_min, unsigned long long* queue,
                                                       uint64_t* out, uint64_t* stats) {
    __shared__ unsigned long long cells[48];
    __shared__ uint2 pend_all[8][64];  // per warp: (w, first window record) awaiting a lookup
    extern __shared__ __align__(16) unsigned char gcache_raw[];  // 8 warps x kGroupCache entries
    zero_cells(cells, 24);
    __syncthreads();
    WarpCells wc;
    const uint32_t cnt = lcount[1];  // the very-long list (back of the buffer)
    if (blockIdx.x == 0 && threadIdx.x == 0 && stats) atomicAdd((unsigned long long*)&stats[3], (unsigned long long)cnt);
    if (!P.gend || *pt_wsum < gend_min) P.gend = nullptr;  // group ends not built
    P.pt_keys = nullptr;
    uint32_t my_wedges = 0, lookups = 0;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    GroupCacheEntry* gc = reinterpret_cast<GroupCacheEntry*>(gcache_raw) + (size_t)(threadIdx.x >> 5) * kGroupCache;
    uint2* pend = pend_all[threadIdx.x >> 5];
    for (;;) {  // one first edge per warp from the queue
        const uint64_t idx = warp_take(queue, 1);
        if (idx >= cnt) break;
        const uint32_t i = list[long_cap - 1 - idx];
        const uint32_t end = Foff[Fnode[i] + 1];
        const uint32_t ni = FN[i];
        const uint32_t v = ni & kNodeMask;
        const int64_t ti = FT[i];
        const uint32_t oi = FO[i];
        const int64_t lim = sat_add(ti, delta);
        const TimeKey limk = FT.key_upto(lim);  // in-window: t_j <= t_i + delta
        const RecKey ki = P.t.rec_key(ti, oi);
        for (int x = lane; x < kGroupCache; x += 32) gc[x].w = kGcEmpty;
        __syncwarp();
        uint32_t used = 0;  // claimed entries (warp-uniform)
        bool done = false;
        for (uint32_t s0 = i + 1; s0 < end && !done; s0 += kLongSeg) {
            const uint32_t s1 = end - s0 > kLongSeg ? s0 + kLongSeg : end;
            if (used > (uint32_t)kGroupCache / 2) {
                for (int x = lane; x < kGroupCache; x += 32) gc[x].w = kGcEmpty;
                used = 0;
                __syncwarp();
            }
            // ---- pass A: claim and resolve the groups the table lacks
            uint32_t npend = 0;
            for (uint32_t j0 = s0; j0 < s1; j0 += 32) {
                const uint32_t j = j0 + lane;
                const bool in = j < s1 && FT.below(j, limk);
                const uint32_t w = in ? FN[j] & kNodeMask : v;
                bool found = false;
                int slot = -1;
                if (w != v) slot = gc_probe(gc, w, found);
                const bool need = w != v && !found && slot >= 0;
                // one candidate per distinct w: its earliest record (lowest lane)
                const unsigned same_w = __match_any_sync(0xffffffffu, need ? w : (0x80000000u | (uint32_t)lane));
                bool cand = need && (__ffs(same_w) - 1) == lane;
                while (__any_sync(0xffffffffu, cand)) {
                    // two neighbours may want the same empty slot: the lower lane takes it
                    const unsigned same_s =
                        __match_any_sync(0xffffffffu, cand ? (uint32_t)slot : (0x80000000u | (uint32_t)lane));
                    const bool win = cand && (__ffs(same_s) - 1) == lane;
                    if (win) gc[slot].w = w;
                    const unsigned wm = __ballot_sync(0xffffffffu, win);
                    if (win) pend[npend + __popc(wm & lt_mask)] = make_uint2(w, j);
                    npend += __popc(wm);
                    used += __popc(wm);
                    __syncwarp();
                    if (npend >= 32) {  // a full batch: one lookup per lane
                        const uint2 pe = pend[lane];
                        const uint2 rest = pend[32 + lane];
                        gc_resolve(P, FT, gc, v, pe.x, pe.y, delta, ki, lim);
                        lookups += 1;
                        __syncwarp();
                        pend[lane] = rest;
                        npend -= 32;
                        __syncwarp();
                    }
                    const bool lose = cand && !win;
                    cand = false;
                    if (lose) {
                        slot = gc_probe(gc, w, found);
                        cand = slot >= 0;  // (w itself cannot have appeared: one candidate per w)
                    }
                }
                if (!__all_sync(0xffffffffu, in)) break;
            }
            if (npend) {  // the rest of the segment's claims
                if ((uint32_t)lane < npend) {
                    const uint2 pe = pend[lane];
                    gc_resolve(P, FT, gc, v, pe.x, pe.y, delta, ki, lim);
                    lookups += 1;
                }
            }
            __syncwarp();
            // ---- pass B: count
            for (uint32_t j0 = s0; j0 < s1; j0 += 32) {
                const uint32_t j = j0 + lane;
                const bool in = j < s1 && FT.below(j, limk);
                const uint32_t nj = in ? FN[j] : 0u;
                const uint32_t w = nj & kNodeMask;
                const bool wedge = in && w != v;
                uint32_t c[6] = {0, 0, 0, 0, 0, 0};
                int cb = 0;
                bool upd = false;
                int slot = -1;
                uint32_t k1 = 0, k3 = 0;
                if (wedge) {
                    ++my_wedges;
                    cb = (int)((ni >> 31) * 4 + (nj >> 31) * 2);
                    bool found;
                    slot = gc_probe(gc, w, found);
                    if (!found) {  // no room in the table: the one-off closing count
                        wedge_counts(P, FT, FN, FO, i, j, delta, t_last, c);
                        lookups += 1;
                    } else {
                        const GroupCacheEntry e = gc[slot];
                        if (e.k4 > e.k1) {  // records left inside [t_j - delta, t_i + delta]
                            const int64_t tj = FT[j];
                            // the window's lower end t_j - delta and e_j only move forward with j
                            k1 = p_gallop_tlower(P, e.k1, e.k2, sat_sub(tj, delta));
                            k3 = p_gallop_rec(P, e.k3, e.k4, P.t.rec_key(tj, FO[j]));
                            upd = true;
                            const uint32_t flip = e.pad;
                            uint32_t k2e = e.k2;
                            if (t_last != INT64_MAX) {
                                uint32_t l = k1, r = e.k2;
                                while (l < r) {
                                    const uint32_t mid = (l + r) >> 1;
                                    if (P.t[mid] <= t_last) l = mid + 1; else r = mid;
                                }
                                k2e = l;
                            }
                            auto add_range = [&](int type, uint32_t x0, uint32_t d0, uint32_t x1, uint32_t d1) {
                                if (x1 <= x0) return;
                                const uint32_t n1 = d1 - d0;
                                const uint32_t n0 = (x1 - x0) - n1;
                                c[type * 2] += flip ? n1 : n0;  // static cell indices: c[] stays in registers
                                c[type * 2 + 1] += flip ? n0 : n1;
                            };
                            if (k1 < k2e) add_range(0, k1, p_dir_before(P, k1), k2e, k2e == e.k2 ? e.d2 : p_dir_before(P, k2e));
                            if (ti <= t_last) {
                                const uint32_t d3 = (k3 == e.k2) ? e.d2 : (k3 == e.k4) ? e.d4 : p_dir_before(P, k3);
                                add_range(1, e.k2, e.d2, k3, d3);
                                add_range(2, k3, d3, e.k4, e.d4);
                            }
                        }
                    }
                }
                // one writer per group: the highest lane that advanced it
                const unsigned peers = __match_any_sync(0xffffffffu, upd ? w : (0x80000000u | (uint32_t)lane));
                if (upd && (peers >> lane) == 1u) {
                    gc[slot].k1 = k1;
                    gc[slot].k3 = k3;
                }
                __syncwarp();
                wc.add6(wedge, cb, c, cells, 24);
                if (!__all_sync(0xffffffffu, in)) {
                    done = true;
                    break;
                }
            }
        }
    }
    wc.flush(cells, 24, 24);
    my_wedges = warp_sum(my_wedges);
    lookups = warp_sum(lookups);
    if (lane == 0 && stats) {
        if (my_wedges) atomicAdd((unsigned long long*)&stats[4], (unsigned long long)my_wedges);
        if (lookups) atomicAdd((unsigned long long*)&stats[5], (unsigned long long)lookups);
    }
    __syncthreads();
    flush_cells(cells, 24, out, kAccCarry);
}

__device__ __forceinline__ uint32_t find_item(const uint64_t* __restrict__ item_off, uint64_t n_items,
                                              uint64_t idx) {
    uint64_t lo = 0, hi = n_items;
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (item_off[mid] <= idx) lo = mid; else hi = mid;
    }
    return (uint32_t)lo;
}

__global__ void __launch_bounds__(256) tri_items_kernel(SView S, PView P, int64_t delta,
                                                        uint64_t n_items,
                                                        const uint32_t* __restrict__ nodes,
                                                        const uint64_t* __restrict__ begin,
                                                        const uint64_t* __restrict__ item_off,
                                                        uint64_t total,
                                                        const uint8_t* __restrict__ live,
                                                        uint64_t* __restrict__ out) {
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t it = find_item(item_off, n_items, idx);
        const uint32_t u = nodes[it];
        const uint32_t start = S.off[u], end = S.off[u + 1];
        const uint32_t i = start + (uint32_t)begin[it] + (uint32_t)(idx - item_off[it]);
        wedges_from(P, S.t, S.nbr, S.ord, i, end, delta, live,
                    GlobalSink{(unsigned long long*)out + (uint64_t)it * 48, 24});
    }
}

// Pair table for the long windows, built only when their wedges are many
// (decided on the device from long_window_sum_kernel's bound: no host sync):
// clear, one insert per P group (its first record), then the group lengths
// (its last record).
// upper bound of the long-window wedges: the in-window records after every
// long first edge (one gallop per first edge, warp-aggregated sum)
__global__ void long_window_sum_kernel(TimeArr FT, const uint32_t* __restrict__ Fnode,
                                       const uint32_t* __restrict__ Foff, int64_t delta,
                                       const uint32_t* __restrict__ list, uint32_t long_cap,
                                       const uint32_t* __restrict__ lcount,
                                       unsigned long long* __restrict__ sum) {
    const uint32_t n0 = lcount[0], cnt = n0 + lcount[1];
    unsigned long long acc = 0;
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < cnt;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = idx < n0 ? list[idx] : list[long_cap - 1 - (idx - n0)];
        const uint32_t end = Foff[Fnode[i] + 1];
        const int64_t lim = sat_add(FT[i], delta);
        uint32_t lo = i + 1, hi = end, span = 8;
        while (true) {  // gallop: windows are long here
            const uint64_t probe = (uint64_t)lo + span;
            if (probe >= hi) break;
            if (FT[probe] > lim) {
                hi = (uint32_t)probe;
                break;
            }
            lo = (uint32_t)probe + 1;
            span <<= 1;
        }
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (FT[mid] > lim) hi = mid; else lo = mid + 1;
        }
        acc += lo - i - 1;
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(sum, acc);
}

// gend[group index] = one past the group's last record, written by that
// record (only when the long windows are many enough: device-side gate)
__global__ void group_end_kernel(const uint32_t* __restrict__ P_w, const uint32_t* __restrict__ gmask,
                                 const uint32_t* __restrict__ gpref, uint64_t m, uint32_t* __restrict__ gend,
                                 const unsigned long long* __restrict__ wsum, uint64_t min_wedges) {
    if (*wsum < min_wedges) return;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (uint64_t)gridDim.x * blockDim.x) {
        if (!(__ldcs(P_w + k) & kPLast)) continue;
        const uint32_t x = (uint32_t)k;
        // inclusive count of group starts up to k, minus one
        gend[gpref[x >> 5] + __popc(gmask[x >> 5] & ((2u << (x & 31)) - 1u)) - 1] = x + 1;
    }
}

__device__ __forceinline__ bool pair_table_wanted(const unsigned long long* wsum, uint64_t min_wedges) {
    return *wsum >= min_wedges;
}

__global__ void pair_table_clear_kernel(unsigned long long* __restrict__ keys, uint64_t cap,
                                        const unsigned long long* __restrict__ wsum, uint64_t min_wedges) {
    if (!pair_table_wanted(wsum, min_wedges)) return;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < cap;
         x += (uint64_t)gridDim.x * blockDim.x)
        keys[x] = kPairEmpty;
}
__global__ void pair_table_insert_kernel(const uint32_t* __restrict__ P_min, const uint32_t* __restrict__ P_max,
                                         const uint32_t* __restrict__ P_w, uint64_t m,
                                         unsigned long long* __restrict__ keys, unsigned long long* __restrict__ vals,
                                         uint64_t mask, const unsigned long long* __restrict__ wsum,
                                         uint64_t min_wedges, int pass) {
    if (!pair_table_wanted(wsum, min_wedges)) return;
    const uint32_t flag = pass == 0 ? kPFirst : kPLast;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (uint64_t)gridDim.x * blockDim.x) {
        if (!(P_w[k] & flag)) continue;
        const uint32_t a = P_min[k], b = P_max[k];
        const unsigned long long key = ((unsigned long long)a << 32) | b;
        uint64_t slot = pair_slot(a, b) & mask;
        if (pass == 0) {  // each pair is one group: a free slot is always found
            while (atomicCAS(&keys[slot], kPairEmpty, key) != kPairEmpty) slot = (slot + 1) & mask;
            vals[slot] = (unsigned long long)k << 32;
        } else {
            while (keys[slot] != key) slot = (slot + 1) & mask;
            vals[slot] |= (uint32_t)(k + 1 - (uint32_t)(vals[slot] >> 32));
        }
    }
}

}  // namespace

void tri_filter_stage(const DeviceGraph& g, const Forward& f, int64_t delta, uint32_t f_begin, uint32_t f_end,
                      cudaStream_t st, TriStage& ts) {
    ts = TriStage{};
    ts.delta = delta;
    ts.f_begin = f_begin;
    ts.f_end = f_end;
    if (f_end <= f_begin) return;
    const uint64_t work = f_end - f_begin;
    const uint64_t cap = (uint64_t)sm_count() * 8;
    uint64_t grid = (work + 256 * kFilterItems - 1) / (256 * kFilterItems);
    if (grid > cap) grid = cap;
    ts.wedge_cap = work + 1024;  // overflow spills to the long list
    ts.wedges = dalloc<uint64_t>(ts.wedge_cap, st);
    // [0] wedge slots reserved (u64: up to kWedgeScan per record), [1] valid
    // end, then the u32 long-list fill
    ts.wbuf = dalloc<uint64_t>(3, st);
    unsigned long long* wcount = reinterpret_cast<unsigned long long*>(ts.wbuf);
    uint32_t* lcount = reinterpret_cast<uint32_t*>(ts.wbuf + 2);
    ts.long_list = dalloc<uint32_t>(work + 1, st);
    ts.long_cap = (uint32_t)(work + 1);
    TM_CUDA(cudaMemsetAsync(wcount, 0, sizeof(uint64_t), st));
    TM_CUDA(cudaMemsetAsync(wcount + 1, 0xFF, sizeof(uint64_t), st));
    TM_CUDA(cudaMemsetAsync(lcount, 0, 2 * sizeof(uint32_t), st));
    TM_LAUNCH("tri_filter", st, tri_filter_kernel, (unsigned)grid, 256, 0, f.t.view(g.tbase), f.nbr, f.node, delta,
              f_begin, f_end, ts.wedges, ts.wedge_cap, ts.long_list, (uint32_t)(work + 1), wcount, lcount);
    // the long windows' wedge bound gates the group ends (both counting
    // kernels) and the pair table (long windows) on the device: no host sync
    ts.wsum = dalloc<unsigned long long>(1, st);
    TM_CUDA(cudaMemsetAsync(ts.wsum, 0, sizeof(unsigned long long), st));
    TM_LAUNCH("tri_gate", st, long_window_sum_kernel, (unsigned)cap, 256, 0, f.t.view(g.tbase), f.node, f.off,
              delta, ts.long_list, (uint32_t)(work + 1), lcount, ts.wsum);
    ts.valid = true;
}

// The pair table is off by default since the fenced block search: at config
// 4, delta 86400 its build (clear + two CAS insert passes over 600M records,
// every insert a full 128-byte line) took 497 ms to save 155 ms of tri_long.
// TM_PAIR_TABLE=<k> builds it when the long windows hold >= k wedges per edge.
uint64_t pair_table_min_wedges(const DeviceGraph& g) {
    static const long long env = [] {
        const char* e = std::getenv("TM_PAIR_TABLE");
        return e ? std::atoll(e) : 0ll;
    }();
    if (env <= 0) return ~0ull;
    return (uint64_t)env * std::max<uint64_t>(g.m, 1024);
}

// long-window wedges (upper bound) at which the group ends pay for their
// pass over P: one per 16 edges (config 1 at delta 3600 has 0.003 per edge
// and would lose ~1 %, at 86400 2.6 per edge and gains 12 %).
// TM_GROUP_ENDS=0 disables them, 1 builds them always.
uint64_t group_end_min_wedges(const DeviceGraph& g) {
    static const long long env = [] {
        const char* e = std::getenv("TM_GROUP_ENDS");
        return e ? std::atoll(e) : -1ll;
    }();
    if (env == 0) return ~0ull;
    if (env == 1) return 0;
    return std::max<uint64_t>(g.m / 16, 1024);
}

void tri_work_stage(const DeviceGraph& g, const Forward& f, TriStage& ts, int64_t t_last, uint64_t* d_out,
                    uint64_t* d_stats) {
    if (!ts.valid) return;
    cudaStream_t st = g.stream;
    const uint64_t cap = (uint64_t)sm_count() * 8;
    unsigned long long* wcount = reinterpret_cast<unsigned long long*>(ts.wbuf);
    uint32_t* lcount = reinterpret_cast<uint32_t*>(ts.wbuf + 2);
    ts.queue = dalloc<unsigned long long>(3, st);
    TM_CUDA(cudaMemsetAsync(ts.queue, 0, 3 * sizeof(unsigned long long), st));
    PView pv = pview(g);
    const uint64_t gend_min = group_end_min_wedges(g);
    if (gend_min != ~0ull && g.m) {
        ts.gend = dalloc<uint32_t>(g.m, st);
        uint64_t grid = (g.m + 255) / 256;
        if (grid > cap) grid = cap;
        TM_LAUNCH("group_end", st, group_end_kernel, (unsigned)grid, 256, 0, g.P_w, g.P_gmask, g.P_gpref, g.m,
                  ts.gend, ts.wsum, gend_min);
        pv.gend = ts.gend;
    }
    TM_LAUNCH("tri_wedge", st, tri_wedge_kernel, (unsigned)cap, 256, 0, pv, f.t.view(g.tbase), f.nbr, f.ord,
              ts.delta, t_last, ts.wedges, ts.wedge_cap, wcount, ts.wsum, gend_min, ts.queue, d_out, d_stats);
    // pair table for the long windows when they hold many wedges: the
    // table costs ~one random insert per P group, and replaces the block
    // search of each long-window wedge
    const uint64_t min_wedges = pair_table_min_wedges(g);
    if (min_wedges != ~0ull && g.m) {
        uint64_t pc = 1024;
        while (pc < g.m + g.m / 4) pc <<= 1;
        ts.pt = dalloc<unsigned long long>(2 * pc, st);
        ts.pt_cap = pc;
        uint64_t grid = (pc + 255) / 256;
        if (grid > cap) grid = cap;
        TM_LAUNCH("pair_table", st, pair_table_clear_kernel, (unsigned)grid, 256, 0, ts.pt, pc, ts.wsum,
                  min_wedges);
        grid = (g.m + 255) / 256;
        if (grid > cap) grid = cap;
        for (int pass = 0; pass < 2; ++pass)
            TM_LAUNCH("pair_table", st, pair_table_insert_kernel, (unsigned)grid, 256, 0, g.P_min, g.P_max, g.P_w,
                      g.m, ts.pt, ts.pt + pc, pc - 1, ts.wsum, min_wedges, pass);
        pv.pt_keys = ts.pt;
        pv.pt_vals = ts.pt + pc;
        pv.pt_mask = pc - 1;
    }
#if TM_MID_FLAT
    TM_LAUNCH("tri_long", st, tri_mid_kernel, (unsigned)cap, 256, 0, pv, f.t.view(g.tbase), f.nbr, f.ord, f.node,
              f.off, ts.delta, t_last, ts.long_list, lcount, ts.wsum, gend_min, ts.queue + 1, d_out, d_stats);
#else
    TM_LAUNCH("tri_long", st, tri_long_kernel<false>, (unsigned)cap, 256, 0, pv, f.t.view(g.tbase), f.nbr, f.ord,
              f.node, f.off, ts.delta, t_last, ts.long_list, ts.long_cap, lcount, ts.wsum, min_wedges, gend_min,
              ts.queue + 1, d_out, d_stats);
#endif
    constexpr size_t kCacheBytes = 8 * (size_t)kGroupCache * sizeof(GroupCacheEntry);
    static const bool cache_attr = [] {
        TM_CUDA(cudaFuncSetAttribute(tri_long_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kCacheBytes));
        return true;
    }();
    (void)cache_attr;
#ifndef TM_TWO_PHASE
#define TM_TWO_PHASE 1
#endif
#if TM_TWO_PHASE
    static const bool window_attr = [] {
        TM_CUDA(cudaFuncSetAttribute(tri_window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kCacheBytes));
        return true;
    }();
    (void)window_attr;
    TM_LAUNCH("tri_long", st, tri_window_kernel, (unsigned)cap, 256, kCacheBytes, pv, f.t.view(g.tbase), f.nbr, f.ord,
              f.node, f.off, ts.delta, t_last, ts.long_list, ts.long_cap, lcount, ts.wsum, gend_min,
              ts.queue + 2, d_out, d_stats);
#else
    TM_LAUNCH("tri_long", st, tri_long_kernel<true>, (unsigned)cap, 256, kCacheBytes, pv, f.t.view(g.tbase), f.nbr, f.ord,
              f.node, f.off, ts.delta, t_last, ts.long_list, ts.long_cap, lcount, ts.wsum, min_wedges, gend_min,
              ts.queue + 2, d_out, d_stats);
#endif
    dfree(ts.pt, st);
    dfree(ts.gend, st);
    dfree(ts.queue, st);
    dfree(ts.wsum, st);
    dfree(ts.wedges, st);
    dfree(ts.long_list, st);
    dfree(ts.wbuf, st);
    ts.valid = false;
}

void tri_oriented(const DeviceGraph& g, const Forward& f, int64_t delta, uint32_t f_begin,
                  uint32_t f_end, int64_t t_last, uint64_t* d_out, uint64_t* d_stats) {
    TriStage ts;
    tri_filter_stage(g, f, delta, f_begin, f_end, g.stream, ts);
    tri_work_stage(g, f, ts, t_last, d_out, d_stats);
}

void tri_items(const DeviceGraph& g, int64_t delta, uint64_t n_items, const uint32_t* d_nodes,
               const uint64_t* d_begin, const uint64_t* d_item_off, uint64_t total,
               const uint8_t* d_live, uint64_t* d_out) {
    if (total == 0) return;
    const uint64_t cap = (uint64_t)sm_count() * 8;
    uint64_t grid = (total + 255) / 256;
    if (grid > cap) grid = cap;
    TM_LAUNCH("tri_items", g.stream, tri_items_kernel, (unsigned)grid, 256, 0, sview(g), pview(g),
              delta, n_items, d_nodes, d_begin, d_item_off, total, d_live, d_out);
}

}  // namespace tmb
