// tm_star.cu -- FAST-Star (Algorithm 1, star_engine.cpp:64-127) on B200.
//
// The reference walks, for every first edge a of S_u, all third edges c in the
// delta window and keeps per-neighbour tallies of the edges in between
// (m_in / m_out), i.e. O(|S_u| * d^delta) per center.  Every tally it reads is
// a count of same-neighbour records in a position interval, so the same cells
// can be written as sums over the *neighbour group* of one record only:
//
//   for first edge a (window W(a) = (a, e(a)), g = group of a):
//     Pair[d1,d2,d3]   += #{b<c in W, x_b = x_c = x_a}
//     A                 = #{b<c in W, x_b = x_a}           Star-III = A - Pair
//     B                 = #{b<c in W, x_c = x_a}           Star-II  = B - Pair
//   and, charged to the third edge c (lo(c) = first index with t >= t_c - d):
//     C                 = sum over b in g(c), lo(c) < b < c of
//                         #{a in [lo(c), b), dir_a = d1}   Star-I   = C - Pair
//
// A, B and Pair only need the same-neighbour records of a inside its window
// (walked in P, where the pair {u, x} is one contiguous time-ordered group
// shared by both endpoints) plus global prefix
// counts of outward records (S_pg); C walks the same-neighbour records of c
// backwards.  Each record is handled by one thread, so a hub needs no special
// treatment and there is no per-center state at all.  Work per record is
// O(log d^delta) for the window search plus the same-neighbour window length.
//
// Output: 32 raw u64 sums  [0..8) Pair, [8..16) C, [16..24) B, [24..32) A,
// each indexed d1*4 + d2*2 + d3; the host forms Star = raw - Pair
// (all arithmetic modulo 2^64, exact because every final cell is >= 0).
#include "tm_primitives.cuh"

namespace tmb {

namespace {

// first index in [beg, end) with T[idx] > lim (end if none); T ascending
__device__ __forceinline__ uint32_t gallop_upper(const TimeArr& T, uint32_t beg,
                                                 uint32_t end, int64_t lim) {
    uint32_t lo = beg, hi = end;
    uint32_t span = 1;
    while (true) {
        const uint64_t probe = (uint64_t)lo + span - 1;
        if (probe >= end) break;
        if (T[probe] > lim) {
            hi = (uint32_t)probe;
            break;
        }
        lo = (uint32_t)probe + 1;
        span <<= 1;
    }
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (T[mid] > lim) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// first index in [beg, from] with T[idx] >= lim, given T[from] >= lim
__device__ __forceinline__ uint32_t gallop_lower_back(const TimeArr& T, uint32_t beg,
                                                      uint32_t from, int64_t lim) {
    uint32_t hi = from, lo = beg;
    uint32_t span = 1;
    while (true) {
        if (hi < beg + span) break;
        const uint32_t probe = hi - span;
        if (T[probe] < lim) {
            lo = probe + 1;
            break;
        }
        hi = probe;
        span <<= 1;
    }
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (T[mid] >= lim) hi = mid; else lo = mid + 1;
    }
    return lo;
}

template <typename Sink>
__device__ __forceinline__ void add_d1(const Sink& sink, int base, uint32_t d1, const uint64_t x[4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) sink.add(base + (int)d1 * 4 + j, x[j]);
}

// Side of center u in the unordered pair {u, other}: 0 when u is the pair's
// lower endpoint in (degree class, id) order (P_min / dir_rel_min describe
// it), 1 when u is the upper one.
__device__ __forceinline__ uint32_t side_of(const PView& P, uint32_t u, uint32_t other) {
    return ranks_below(P.cls, u, other) ? 0u : 1u;
}

// (t, ordinal) strict order between S record p and (t, ord)
__device__ __forceinline__ bool s_before(const SView& S, uint32_t p, int64_t t, uint32_t ord) {
    const int64_t tp = S.t[p];
    return tp < t || (tp == t && (S.ord[p] & kNodeMask) < ord);
}

// first position in [lo, hi) not before (t, ord): the record itself when it
// lies in the range.  gallop_locate probes upward from lo, gallop_locate_back
// downward from hi (members of a group are met in order, close to the last).
__device__ __forceinline__ uint32_t gallop_locate(const SView& S, uint32_t lo, uint32_t hi, int64_t t,
                                                  uint32_t ord) {
    uint32_t a = lo, b = hi, span = 1;
    while (true) {
        const uint64_t probe = (uint64_t)a + span - 1;
        if (probe >= hi) break;
        if (!s_before(S, (uint32_t)probe, t, ord)) {
            b = (uint32_t)probe;
            break;
        }
        a = (uint32_t)probe + 1;
        span <<= 1;
    }
    while (a < b) {
        const uint32_t mid = (a + b) >> 1;
        if (s_before(S, mid, t, ord)) a = mid + 1; else b = mid;
    }
    return a;
}
__device__ __forceinline__ uint32_t gallop_locate_back(const SView& S, uint32_t lo, uint32_t hi,
                                                       int64_t t, uint32_t ord) {
    uint32_t a = lo, b = hi, span = 1;
    while (true) {
        if (b - lo < span) break;
        const uint32_t probe = b - span;
        if (s_before(S, probe, t, ord)) {
            a = probe + 1;
            break;
        }
        b = probe;
        span <<= 1;
    }
    while (a < b) {
        const uint32_t mid = (a + b) >> 1;
        if (s_before(S, mid, t, ord)) a = mid + 1; else b = mid;
    }
    return a;
}

// first-edge role of S position q = P record k seen from center u (side 0:
// u is the pair's smaller id), S range [start, end): Pair, A, B.
template <typename Sink>
__device__ __forceinline__ void first_role(const SView& S, const PView& P, uint32_t q, uint32_t k,
                                           uint32_t side, uint32_t start, uint32_t end,
                                           int64_t delta, const Sink& acc) {
    const int64_t ta = S.t[q];
    const uint32_t da = S.nbr[q] >> 31;
    const int64_t lim = sat_add(ta, delta);
    if (P.w[k] & kPLast) return;
    if (P.t[k + 1] > lim) return;  // no same-neighbour record in the window

    const uint32_t base = outward_before(S, start);
    const uint32_t e = gallop_upper(S.t, q + 1, end, lim);
    const uint64_t pe_o = outward_before(S, e) - base, pe_i = (uint64_t)(e - start) - pe_o;
    const uint64_t pa_o = (uint64_t)(outward_before(S, q) - base) + (da ? 0u : 1u);
    const uint64_t pa_i = (uint64_t)(q - start + 1) - pa_o;

    uint64_t n0 = 0, n1 = 0;
    uint64_t A00 = 0, A01 = 0, A10 = 0, A11 = 0;   // A[d2][d3]: sum [dir_b=d2] P_d3(b+1)
    uint64_t B00 = 0, B01 = 0, B10 = 0, B11 = 0;   // B[d3][d2]: sum [dir_c=d3] P_d2(c)
    uint64_t P00 = 0, P01 = 0, P10 = 0, P11 = 0;   // Pair[d2][d3]
    uint32_t qb = q;
    for (++k;; ++k) {
        const int64_t tb = P.t[k];
        if (tb > lim) break;
        const uint32_t w = P.w[k];
        qb = gallop_locate(S, qb + 1, e, tb, P.ord[k]);  // member's place in S_u
        const uint64_t pos = qb - start;
        const uint64_t pb_o = outward_before(S, qb) - base;
        const uint64_t pb_i = pos - pb_o;
        if ((w >> 31) ^ side) {  // inward relative to u
            A10 += pb_o;
            A11 += pos + 1 - pb_o;
            B10 += pb_o;
            B11 += pb_i;
            P01 += n0;
            P11 += n1;
            ++n1;
        } else {
            A00 += pb_o + 1;
            A01 += pos - pb_o;
            B00 += pb_o;
            B01 += pb_i;
            P00 += n0;
            P10 += n1;
            ++n0;
        }
        if (w & kPLast) break;
    }
    uint64_t pair[4] = {P00, P01, P10, P11};
    // A(d2,d3) = n[d2] * P_d3(e) - Aacc[d2][d3]
    uint64_t a[4] = {n0 * pe_o - A00, n0 * pe_i - A01, n1 * pe_o - A10, n1 * pe_i - A11};
    // B(d2,d3) = Bacc[d3][d2] - n[d3] * P_d2(a+1)
    uint64_t b[4] = {B00 - n0 * pa_o, B10 - n1 * pa_o, B01 - n0 * pa_i, B11 - n1 * pa_i};
    add_d1(acc, 0, da, pair);
    add_d1(acc, 24, da, a);
    add_d1(acc, 16, da, b);
}

// third-edge role of S position q = P record k seen from center u: the
// Star-I pair term C.  rb/re: first-edge range (local), clipped; the full run
// passes rb = 0, re = s.
template <typename Sink>
__device__ __forceinline__ void third_role(const SView& S, const PView& P, uint32_t q, uint32_t k,
                                           uint32_t side, uint32_t start, int64_t delta,
                                           uint32_t rb, uint32_t re, const Sink& acc) {
    if (P.w[k] & kPFirst) return;
    const int64_t tc = S.t[q];
    const int64_t lo_lim = sat_sub(tc, delta);
    // quick reject: previous same-neighbour record already before the window
    if (P.t[k - 1] < lo_lim) return;
    const uint32_t dc = S.nbr[q] >> 31;
    const uint32_t lo = gallop_lower_back(S.t, start, q, lo_lim);
    const uint32_t L = max(lo, start + rb);
    if (L >= q) return;
    const uint32_t pl = outward_before(S, L);
    const int64_t tL = S.t[L];
    const uint32_t oL = S.ord[L] & kNodeMask;
    const uint32_t hiq = start + re;
    uint64_t x0 = 0, x1 = 0, y0 = 0, y1 = 0;  // x: d1 = out, y: d1 = in ; index d2
    uint32_t qb = q;
    for (--k;; --k) {
        const int64_t tb = P.t[k];
        const uint32_t ob = P.ord[k];
        if (tb < tL || (tb == tL && ob <= oL)) break;  // member at or before position L
        const uint32_t w = P.w[k];
        qb = gallop_locate_back(S, L + 1, qb, tb, ob);
        const uint32_t mhi = min(qb, hiq);
        if (mhi > L) {
            const uint64_t x = (uint64_t)(outward_before(S, mhi) - pl);
            const uint64_t y = (uint64_t)(mhi - L) - x;
            if ((w >> 31) ^ side) { x1 += x; y1 += y; } else { x0 += x; y0 += y; }
        }
        if (w & kPFirst) break;
    }
    // cells C[d1][d2][dc]
    acc.add(8 + 0 + 0 + dc, x0);
    acc.add(8 + 0 + 2 + dc, x1);
    acc.add(8 + 4 + 0 + dc, y0);
    acc.add(8 + 4 + 2 + dc, y1);
}

// Filter: one coalesced pass over P.  A record can contribute as a first
// edge only if the next record of its pair group is inside its window, and as
// a third edge only if the previous one is (otherwise every term of
// first_role / third_role is zero).  Both endpoints share the group order, so
// a surviving record yields a candidate at each of its centers inside the
// center partition [cb, ce); entries are 2k + side.
constexpr int kFilterItems = 4;  // edges per thread per block iteration (one reservation)
__global__ void __launch_bounds__(256) star_filter_kernel(PView P, int64_t delta, uint64_t m,
                                                          uint32_t cb, uint32_t ce,
                                                          uint32_t* __restrict__ first_list,
                                                          uint32_t* __restrict__ third_list,
                                                          uint32_t* __restrict__ counters) {
    constexpr uint64_t kStep = 256 * kFilterItems;
    for (uint64_t base = (uint64_t)blockIdx.x * kStep; base < m; base += (uint64_t)gridDim.x * kStep) {
        // bit 2j + side: edge j's entry for that center is a first / third candidate
        uint32_t fbits = 0, tbits = 0;
#pragma unroll
        for (int j = 0; j < kFilterItems; ++j) {
            const uint64_t k = base + (uint64_t)j * 256 + threadIdx.x;
            if (k < m) {
                const uint32_t w = P.w[k];
                const int64_t t = P.t[k];
                const bool f = !(w & kPLast) && P.t[k + 1] <= sat_add(t, delta);
                const bool th = !(w & kPFirst) && P.t[k - 1] >= sat_sub(t, delta);
                if (f || th) {
                    const uint32_t a = P.min[k], b = P.max[k];
                    const uint32_t in = (a >= cb && a < ce ? 1u : 0u) | (b >= cb && b < ce ? 2u : 0u);
                    if (f) fbits |= in << (2 * j);
                    if (th) tbits |= in << (2 * j);
                }
            }
        }
        uint32_t of, ot;
        block_reserve2<8, uint32_t>((uint32_t)__popc(fbits), (uint32_t)__popc(tbits), counters, counters + 1,
                                    of, ot);
        while (fbits) {
            const int b = __ffs(fbits) - 1;
            fbits &= fbits - 1;
            const uint64_t k = base + (uint64_t)(b >> 1) * 256 + threadIdx.x;
            first_list[of++] = (uint32_t)(2 * k + (b & 1));
        }
        while (tbits) {
            const int b = __ffs(tbits) - 1;
            tbits &= tbits - 1;
            const uint64_t k = base + (uint64_t)(b >> 1) * 256 + threadIdx.x;
            third_list[ot++] = (uint32_t)(2 * k + (b & 1));
        }
    }
}

// ---- full pass: the candidates' S positions first, then the sums --------
//
// Every member of a candidate's window is itself a candidate: a record after
// first edge a inside its window has its predecessor within delta (so it is a
// third-edge candidate), and a record before third edge c inside c's window
// has its successor within delta (a first-edge candidate).  star_locate
// therefore finds the S position q (and the outward count before it) of every
// candidate once -- a fenced search in its center's sequence -- into the
// P-indexed planes PS[side][k]; star_work then walks each window's members
// through PS (contiguous 8-byte reads) instead of locating every member in
// S_u again, which cost a gallop of scattered 128-byte lines per member.

// S position of the first record after q with t > lim (end if none): a
// short gallop (the window is usually a few lines), then the fenced search
__device__ __forceinline__ uint32_t s_window_end(const SView& S, uint32_t q, uint32_t end, int64_t lim) {
    uint32_t lo = q + 1;
    const TProbe<false> pr(S.t, S.t32, S.t1k, lim);
    for (uint32_t span = 1; span <= 32; span <<= 1) {
        const uint64_t probe = (uint64_t)lo + span - 1;
        if (probe >= end) return fenced_lower_bound(lo, end, pr);
        if (!pr.below0((uint32_t)probe)) return fenced_lower_bound(lo, (uint32_t)probe, pr);
        lo = (uint32_t)probe + 1;
    }
    return fenced_lower_bound(lo, end, pr);
}
// first S position in [start, q] with t >= lim (q itself when none before)
__device__ __forceinline__ uint32_t s_window_begin(const SView& S, uint32_t start, uint32_t q, int64_t lim) {
    uint32_t hi = q;
    const TProbe<true> pr(S.t, S.t32, S.t1k, lim);
    for (uint32_t span = 1; span <= 32; span <<= 1) {
        if (hi - start < span) return fenced_lower_bound(start, hi, pr);
        const uint32_t probe = hi - span;
        if (pr.below0(probe)) return fenced_lower_bound(probe + 1, hi, pr);
        hi = probe;
    }
    return fenced_lower_bound(start, hi, pr);
}

__global__ void __launch_bounds__(256) star_locate_kernel(SView S, PView P, uint64_t m,
                                                          const uint32_t* __restrict__ first_list,
                                                          const uint32_t* __restrict__ third_list,
                                                          const uint32_t* __restrict__ counters,
                                                          uint2* __restrict__ PS) {
    const uint32_t nf = counters[0], nt = counters[1];
    const uint64_t total = (uint64_t)nf + nt;
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e = idx < nf ? first_list[idx] : third_list[idx - nf];
        const uint32_t k = e >> 1, side = e & 1u;
        const uint32_t u = side ? P.max[k] : P.min[k];
        const uint32_t q = s_locate_fenced(S, S.off[u], S.off[u + 1], P.t[k], P.ord[k]);
        PS[(uint64_t)side * m + k] = make_uint2(q, outward_before(S, q));
    }
}

// first-edge role of candidate k at center u (side), S position q = PS: Pair, A, B
__device__ __forceinline__ void first_role_ps(const SView& S, const PView& P, const uint2* __restrict__ PSs,
                                              uint32_t q, uint32_t ob_q, uint32_t k, uint32_t side,
                                              uint32_t start, uint32_t end, int64_t delta, uint64_t pair[4],
                                              uint64_t a[4], uint64_t b[4], uint32_t& da) {
    const uint32_t wa = P.w[k];
    const int64_t ta = P.t[k];
    da = (wa >> 31) ^ side;  // 0: outward from u
    const int64_t lim = sat_add(ta, delta);
    const TimeKey limk = P.t.key_upto(lim);
    if ((wa & kPLast) || !P.t.below(k + 1, limk)) return;  // no same-neighbour record in the window
    const uint32_t base = outward_before(S, start);
    const uint32_t e = s_window_end(S, q, end, lim);
    const uint64_t pe_o = outward_before(S, e) - base, pe_i = (uint64_t)(e - start) - pe_o;
    const uint64_t pa_o = (uint64_t)(ob_q - base) + (da ? 0u : 1u);
    const uint64_t pa_i = (uint64_t)(q - start + 1) - pa_o;
    uint64_t n0 = 0, n1 = 0;
    uint64_t A00 = 0, A01 = 0, A10 = 0, A11 = 0;   // A[d2][d3]: sum [dir_b=d2] P_d3(b+1)
    uint64_t B00 = 0, B01 = 0, B10 = 0, B11 = 0;   // B[d3][d2]: sum [dir_c=d3] P_d2(c)
    uint64_t P00 = 0, P01 = 0, P10 = 0, P11 = 0;   // Pair[d2][d3]
    for (uint32_t j = k + 1;; ++j) {
        if (!P.t.below(j, limk)) break;
        const uint32_t w = P.w[j];
        const uint2 ps = PSs[j];
        const uint64_t pos = ps.x - start;
        const uint64_t pb_o = ps.y - base;
        const uint64_t pb_i = pos - pb_o;
        if ((w >> 31) ^ side) {  // inward relative to u
            A10 += pb_o;
            A11 += pos + 1 - pb_o;
            B10 += pb_o;
            B11 += pb_i;
            P01 += n0;
            P11 += n1;
            ++n1;
        } else {
            A00 += pb_o + 1;
            A01 += pos - pb_o;
            B00 += pb_o;
            B01 += pb_i;
            P00 += n0;
            P10 += n1;
            ++n0;
        }
        if (w & kPLast) break;
    }
    pair[0] = P00; pair[1] = P01; pair[2] = P10; pair[3] = P11;
    // A(d2,d3) = n[d2] * P_d3(e) - Aacc[d2][d3]
    a[0] = n0 * pe_o - A00; a[1] = n0 * pe_i - A01; a[2] = n1 * pe_o - A10; a[3] = n1 * pe_i - A11;
    // B(d2,d3) = Bacc[d3][d2] - n[d3] * P_d2(a+1)
    b[0] = B00 - n0 * pa_o; b[1] = B10 - n1 * pa_o; b[2] = B01 - n0 * pa_i; b[3] = B11 - n1 * pa_i;
}

// third-edge role of candidate k at center u (side), S position q = PS: the
// Star-I pair term C, x[d1*2 + d2]; first edges restricted to the local
// prefix [0, re) of S_u (time slices), dc = the third edge's direction
__device__ __forceinline__ void third_role_ps(const SView& S, const PView& P, const uint2* __restrict__ PSs,
                                              uint32_t q, uint32_t k, uint32_t side, uint32_t start,
                                              int64_t delta, uint32_t re, uint64_t x[4], uint32_t& dc) {
    const uint32_t wc = P.w[k];
    dc = (wc >> 31) ^ side;
    if (wc & kPFirst) return;
    const int64_t lo_lim = sat_sub(P.t[k], delta);
    const TimeKey lok = P.t.key_below(lo_lim);
    if (P.t.below(k - 1, lok)) return;  // previous same-neighbour record already before the window
    const uint32_t lo = s_window_begin(S, start, q, lo_lim);
    if (lo >= q) return;
    const uint32_t pl = outward_before(S, lo);
    const uint32_t hiq = start + re;
    const uint32_t o_hiq = hiq < q ? outward_before(S, hiq) : 0u;
    for (uint32_t j = k - 1;; --j) {
        // a record before the window is no candidate (its PS entry is not
        // written): stop on its time first; in-window members are candidates
        if (P.t.below(j, lok)) break;
        const uint2 ps = PSs[j];
        if (ps.x <= lo) break;  // the member at the window start itself
        const uint32_t w = P.w[j];
        const uint32_t mhi = min(ps.x, hiq);
        if (mhi > lo) {
            const uint64_t xo = (uint64_t)((mhi == ps.x ? ps.y : o_hiq) - pl);
            const uint64_t yi = (uint64_t)(mhi - lo) - xo;
            const int d2 = (int)(((w >> 31) ^ side));
            x[d2] += xo;      // d1 = out
            x[2 + d2] += yi;  // d1 = in
        }
        if (w & kPFirst) break;
    }
}

// exact warp sum of a u64 (three 22-bit chunks through redux.sync): the
// total as a 128-bit (lo, hi) pair
__device__ __forceinline__ void warp_sum_u64(uint64_t v, uint64_t& lo, uint32_t& hi) {
    const uint32_t a = __reduce_add_sync(0xffffffffu, (uint32_t)v & 0x3fffffu);
    const uint32_t b = __reduce_add_sync(0xffffffffu, (uint32_t)(v >> 22) & 0x3fffffu);
    const uint32_t c = __reduce_add_sync(0xffffffffu, (uint32_t)(v >> 44));
    const unsigned __int128 t = (unsigned __int128)a + ((unsigned __int128)b << 22) + ((unsigned __int128)c << 44);
    lo = (uint64_t)t;
    hi = (uint32_t)(t >> 64);
}

// lane L holds star raw cell L (32 cells) with its wrap count
struct StarLaneCell {
    uint64_t mine = 0;
    uint32_t wraps = 0;
    // warp-wide: add v (per lane) into cell `cell` (per lane; -1 = none)
    __device__ __forceinline__ void add(int cell, uint64_t v, int c0, int c1) {
        // the lanes' cells are one of {c0, c1} (or none): one exact sum each
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = h ? c1 : c0;
            if (!__any_sync(0xffffffffu, cell == c && v)) continue;
            uint64_t lo;
            uint32_t hi;
            warp_sum_u64(cell == c ? v : 0ull, lo, hi);
            if ((int)(threadIdx.x & 31) == c) {
                const uint64_t nm = mine + lo;
                wraps += hi + (nm < mine ? 1u : 0u);
                mine = nm;
            }
        }
    }
};

__global__ void __launch_bounds__(256, 4) star_work_kernel(SView S, PView P, int64_t delta, int64_t t_last,
                                                        uint64_t m, const uint2* __restrict__ PS,
                                                        const uint32_t* __restrict__ first_list,
                                                        const uint32_t* __restrict__ third_list,
                                                        const uint32_t* __restrict__ counters,
                                                        unsigned long long* __restrict__ queue,
                                                        uint64_t* __restrict__ out,
                                                        uint64_t* __restrict__ stats) {
    __shared__ unsigned long long cells[64];
    zero_cells(cells, 32);
    if (blockIdx.x == 0 && threadIdx.x == 0 && stats) {
        stats[0] = counters[0];
        stats[1] = counters[1];
    }
    __syncthreads();
    StarLaneCell lc;
    const uint32_t nf = counters[0], nt = counters[1];
    const uint64_t total = (uint64_t)nf + nt;
    for (;;) {  // 32 items per warp from the queue (hub items are heavy-tailed)
        const uint64_t base = warp_take(queue, 32);
        if (base >= total) break;
        const uint64_t idx = base + (threadIdx.x & 31);
        uint64_t pr[4] = {0, 0, 0, 0}, av[4] = {0, 0, 0, 0}, bv[4] = {0, 0, 0, 0}, xv[4] = {0, 0, 0, 0};
        uint32_t d1 = 0, dc = 0;
        bool is_first = false, is_third = false;
        if (idx < total) {
            const bool first = idx < nf;
            const uint32_t e = first ? first_list[idx] : third_list[idx - nf];
            const uint32_t k = e >> 1, side = e & 1u;
            const uint32_t u = side ? P.max[k] : P.min[k];
            const uint32_t start = S.off[u], end = S.off[u + 1];
            const uint2* PSs = PS + (uint64_t)side * m;
            const uint2 me = PSs[k];
            if (first) {
                if (P.t[k] <= t_last) {  // else: the instance's first edge is outside the time slice
                    first_role_ps(S, P, PSs, me.x, me.y, k, side, start, end, delta, pr, av, bv, d1);
                    is_first = true;
                }
            } else {
                // first edges restricted to t <= t_last: a prefix of S_u
                const uint32_t re = t_last == INT64_MAX ? end - start : s_t_upper(S, start, end, t_last) - start;
                third_role_ps(S, P, PSs, me.x, k, side, start, delta, re, xv, dc);
                is_third = true;
            }
        }
        // warp reductions into the lane-held cells: Pair [0,8), C [8,16), B [16,24), A [24,32)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = is_first ? (int)d1 * 4 + j : -1;
            lc.add(c, pr[j], j, 4 + j);
            lc.add(c < 0 ? -1 : 24 + c, av[j], 24 + j, 28 + j);
            lc.add(c < 0 ? -1 : 16 + c, bv[j], 16 + j, 20 + j);
        }
#pragma unroll
        for (int x = 0; x < 4; ++x) {  // C[d1][d2][dc]: x = d1 * 2 + d2
            const int c = is_third ? 8 + x * 2 + (int)dc : -1;
            lc.add(c, xv[x], 8 + x * 2, 9 + x * 2);
        }
    }
    const int lane = threadIdx.x & 31;
    cell_add(&cells[lane], 32, lc.mine);
    if (lc.wraps) atomicAdd(&cells[lane + 32], (unsigned long long)lc.wraps);
    __syncthreads();
    flush_cells(cells, 32, out, kAccCarry);
}

__device__ __forceinline__ uint32_t find_item(const uint64_t* __restrict__ item_off, uint64_t n_items,
                                              uint64_t idx) {
    uint64_t lo = 0, hi = n_items;  // last item with item_off[it] <= idx
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (item_off[mid] <= idx) lo = mid; else hi = mid;
    }
    return (uint32_t)lo;
}

// per-item star/pair: first-edge positions [rb, min(re, s)), third positions (rb, s)
__global__ void __launch_bounds__(256) star_items_kernel(
    SView S, PView P, int64_t delta, uint64_t n_items, const uint32_t* __restrict__ nodes,
    const uint64_t* __restrict__ begin, const uint64_t* __restrict__ endr,
    const uint64_t* __restrict__ first_off, uint64_t total_first,
    const uint64_t* __restrict__ third_off, uint64_t total_third, uint64_t* __restrict__ out) {
    const uint64_t total = total_first + total_third;
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t it;
        if (idx < total_first) {
            it = find_item(first_off, n_items, idx);
            const uint32_t u = nodes[it];
            const uint32_t start = S.off[u], end = S.off[u + 1];
            const uint32_t q = start + (uint32_t)begin[it] + (uint32_t)(idx - first_off[it]);
            first_role(S, P, q, S.pidx[q], side_of(P, u, S.nbr[q] & kNodeMask), start, end, delta,
                       GlobalSink{(unsigned long long*)out + (uint64_t)it * 64, 32});
        } else {
            const uint64_t j = idx - total_first;
            it = find_item(third_off, n_items, j);
            const uint32_t u = nodes[it];
            const uint32_t start = S.off[u], end = S.off[u + 1];
            const uint32_t s = end - start;
            const uint32_t rb = (uint32_t)begin[it];
            const uint32_t re = (uint32_t)(endr[it] < (uint64_t)s ? endr[it] : (uint64_t)s);
            const uint32_t q = start + rb + 1 + (uint32_t)(j - third_off[it]);
            third_role(S, P, q, S.pidx[q], side_of(P, u, S.nbr[q] & kNodeMask), start, delta, rb, re,
                       GlobalSink{(unsigned long long*)out + (uint64_t)it * 64, 32});
        }
    }
}

}  // namespace

void star_full(const DeviceGraph& g, int64_t delta, uint32_t c_begin, uint32_t c_end, int64_t t_last,
               uint64_t* d_out, uint64_t* d_stats, cudaStream_t st) {
    if (c_end <= c_begin || g.m == 0) return;
    const uint64_t cap = (uint64_t)sm_count() * 8;
    uint64_t grid = (g.m + 256 * kFilterItems - 1) / (256 * kFilterItems);
    if (grid > cap) grid = cap;
    const uint64_t work = 2 * g.m;
    uint32_t* lists = dalloc<uint32_t>(2 * work + 4, st);
    uint32_t* counters = lists + 2 * work;  // 2 list fills, then (8-byte aligned) the work queue
    unsigned long long* queue = reinterpret_cast<unsigned long long*>(lists + 2 * work + 2);
    TM_CUDA(cudaMemsetAsync(counters, 0, 4 * sizeof(uint32_t), st));
    TM_LAUNCH("star_filter", st, star_filter_kernel, (unsigned)grid, 256, 0, pview(g), delta, g.m,
              c_begin, c_end, lists, lists + work, counters);
    // candidates' S positions (P-indexed planes, one per side; only candidate
    // entries are written), then the sums
    uint2* PS = dalloc<uint2>(2 * g.m, st);
    TM_LAUNCH("star_locate", st, star_locate_kernel, (unsigned)cap, 256, 0, sview(g), pview(g), g.m, lists,
              lists + work, counters, PS);
    TM_LAUNCH("star_work", st, star_work_kernel, (unsigned)cap, 256, 0, sview(g), pview(g), delta, t_last, g.m,
              PS, lists, lists + work, counters, queue, d_out, d_stats);
    dfree(PS, st);
    dfree(lists, st);
}

void star_items(const DeviceGraph& g, int64_t delta, uint64_t n_items, const uint32_t* d_nodes,
                const uint64_t* d_begin, const uint64_t* d_end, const uint64_t* d_first_off,
                uint64_t total_first, uint64_t total_third, const uint64_t* d_third_off,
                uint64_t* d_out) {
    const uint64_t total = total_first + total_third;
    if (total == 0) return;
    const uint64_t cap = (uint64_t)sm_count() * 8;
    uint64_t grid = (total + 255) / 256;
    if (grid > cap) grid = cap;
    TM_LAUNCH("star_items", g.stream, star_items_kernel, (unsigned)grid, 256, 0, sview(g), pview(g),
              delta, n_items, d_nodes, d_begin, d_end, d_first_off, total_first, d_third_off,
              total_third, d_out);
}

}  // namespace tmb
