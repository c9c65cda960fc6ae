// tm_graph.cu -- GPU construction of the temporal adjacency.
//
// Replaces TemporalGraph::build (graph.cpp:13-44), NodeSequenceIndex
// (indexes.cpp:7-26) and PairEdgeIndex (indexes.cpp:28-58):
//   1. validate endpoints, find t range, detect already-sorted input;
//   2. stable radix sort of edges by t (skipped when already sorted), so the
//      edge order is the reference's (t, ordinal) total order;
//   3. stable radix sort of the 2m incident records (emitted in that order)
//      by node -> S, the per-node time-ordered sequences;
//   4. P, the per-pair time-sorted edge lists (PairEdgeIndex), which are also
//      each endpoint's same-neighbour runs: the max-side records of S are
//      already in (max, t, ordinal) order, so a stable sort of them by the min
//      endpoint alone yields (min, max, t, ordinal) -- nb key bits instead of
//      2 nb.  Keys carry their payload in the low bits (keys-only sorts).
#include <vector>

#include "tm_primitives.cuh"

namespace tmb {

namespace {

using BuildStats = BuildVerdict;

// packed (t - tmin) << kbits | k  when it fits 64 bits, else key = t - tmin, val = k
__global__ void time_keys_kernel(const int64_t* __restrict__ t, uint64_t m, int64_t tmin, int kbits,
                                 bool packed, uint64_t* __restrict__ keys,
                                 uint32_t* __restrict__ vals) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t rel = (uint64_t)t[k] - (uint64_t)tmin;
        if (packed) {
            keys[k] = (rel << kbits) | k;
        } else {
            keys[k] = rel;
            vals[k] = (uint32_t)k;
        }
    }
}

// Edge records in input order (indexed by ordinal), read by random gathers in
// gather_s and gather_p.  Wide (16 B): any int64 timestamps.  Narrow (8 B): t - t_min
// as u32 and src ^ dst with "src is the smaller endpoint" in the top bit (node
// ids are < 2^31), used whenever the time span fits 32 bits -- half the bytes
// per gather, and the whole array (80 MB at 10M edges) mostly stays in L2.
struct WideEdge {
    int64_t t;
    uint32_t src;
    uint32_t dst;
};
struct NarrowEdge {
    uint32_t trel;
    uint32_t x;
};
template <bool kNarrow>
struct EdgeCodec;
template <>
struct EdgeCodec<false> {
    using Rec = WideEdge;
    __device__ static Rec make(int64_t t, uint32_t a, uint32_t b, int64_t) { return Rec{t, a, b}; }
    __device__ static int64_t time(const Rec& e, int64_t) { return e.t; }
    __device__ static uint32_t rel(const Rec&) { return 0u; }
    __device__ static uint32_t other(const Rec& e, uint32_t u) { return e.src ^ e.dst ^ u; }
    __device__ static uint32_t dir_from_min(const Rec& e, uint32_t mn) { return e.src == mn ? 0u : 1u; }
};
template <>
struct EdgeCodec<true> {
    using Rec = NarrowEdge;
    __device__ static Rec make(int64_t t, uint32_t a, uint32_t b, int64_t tmin) {
        return Rec{(uint32_t)((uint64_t)t - (uint64_t)tmin), (a ^ b) | (a < b ? 0x80000000u : 0u)};
    }
    __device__ static int64_t time(const Rec& e, int64_t tmin) { return tmin + (int64_t)e.trel; }
    __device__ static uint32_t rel(const Rec& e) { return e.trel; }
    __device__ static uint32_t other(const Rec& e, uint32_t u) { return (e.x & kNodeMask) ^ u; }
    __device__ static uint32_t dir_from_min(const Rec& e, uint32_t) { return (e.x >> 31) ? 0u : 1u; }
};

// record r = 2k + side of the p-th edge in (t, ordinal) order, k its input
// index: key node << 32 | r.  The stable node sort keeps (t, ordinal) order
// inside each node because the keys are emitted in that order; the payload
// names the input edge, so the edge records E are indexed by input position
// (written coalesced here) and S / P read their ordinals straight from the key.
// One block per radix-sort tile (kSortTile keys = kSortTile / 2 edges): the
// tile's histogram of the first digit (node & dmask0, the node sort's first
// digit width: radix_digit_width) is written digit-major like
// radix_upsweep's, so the node sort skips its first counting pass.
constexpr int kPackBlock = 256;
constexpr int kPackEdges = kSortTile / 2;
// With `st` set (first pass over the caller's arrays, no permutation) the
// kernel also validates the edges (endpoint range, self loops), reduces the
// t range, detects time-unordered input, and -- packing narrow records
// relative to t[0] -- flags spans that do not fit; the host reads `st` once
// and re-packs in the rare cases (unordered input, wide span).  The (t,
// ordinal) order of unordered input comes as perm[p] or as the low kmask bits
// of the time sort's packed keys tkeys[p].  Endpoints are clamped into range
// in every pass: a speculatively replayed build of input the verdict later
// rejects stays in bounds.
// kScan: validate, reduce and count only -- nothing is written: the node
// sort's first pass then reads the caller's arrays itself (RawEdgeLoad).
template <bool kNarrow, bool kPermuted, bool kScan = false>
__global__ void __launch_bounds__(kPackBlock) pack_edges_kernel(
    const uint32_t* __restrict__ perm, const uint64_t* __restrict__ tkeys, uint64_t kmask,
    const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst, const int64_t* __restrict__ t,
    uint64_t m, uint64_t n, int64_t tmin, typename EdgeCodec<kNarrow>::Rec* __restrict__ E,
    uint64_t* __restrict__ keys, uint64_t* __restrict__ vals, uint32_t* __restrict__ counts, uint32_t ntiles,
    BuildStats* __restrict__ st) {
    constexpr int NW = kPackBlock / 32;
    __shared__ uint32_t hist[NW][kRadix];
    const int w = threadIdx.x >> 5;
    int nbits = 1;
    while (nbits < 32 && ((n > 1 ? n - 1 : 1) >> nbits)) ++nbits;
    const uint32_t dmask0 = (1u << radix_digit_width(nbits, radix_passes(nbits))) - 1u;
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    unsigned bad = 0, uns = 0;
    if (st) tmin = t[0];
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int i = threadIdx.x; i < NW * kRadix; i += kPackBlock) (&hist[0][0])[i] = 0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kPackEdges / kPackBlock; ++j) {
            const uint64_t p = (uint64_t)tile * kPackEdges + j * kPackBlock + threadIdx.x;
            if (p < m) {
                const uint32_t k = !kPermuted ? (uint32_t)p : perm ? perm[p] : (uint32_t)(tkeys[p] & kmask);
                uint32_t a = src[k], b = dst[k];
                const int64_t tp = t[p];
                if (st) {
                    bad |= (a == b) | (a >= n) | (b >= n);
                    lo = min(lo, (long long)tp);
                    hi = max(hi, (long long)tp);
                    if (p + 1 < m) uns |= (t[p + 1] < tp);
                }
                a = a < n ? a : 0u;
                b = b < n ? b : 0u;
                uint32_t ea = a, eb = b;  // edge p in input order
                if (kPermuted) {
                    ea = src[p];
                    eb = dst[p];
                    ea = ea < n ? ea : 0u;
                    eb = eb < n ? eb : 0u;
                }
                if (!kScan && !(kNarrow && vals)) E[p] = EdgeCodec<kNarrow>::make(tp, ea, eb, tmin);  // gathered (wide only)
                if (!kScan)
                    reinterpret_cast<ulonglong2*>(keys)[p] =
                        make_ulonglong2(((uint64_t)a << 32) | (2 * k), ((uint64_t)b << 32) | (2 * k + 1));
                if (!kScan && kNarrow && vals) {  // the gathers' payload travels with the node sort
                    const uint64_t rel = (uint64_t)(kPermuted ? t[k] : tp) - (uint64_t)tmin;
                    reinterpret_cast<ulonglong2*>(vals)[p] =
                        make_ulonglong2((rel << 32) | b, (rel << 32) | a | kDirBit);
                }
                atomicAdd(&hist[w][a & dmask0], 1u);
                atomicAdd(&hist[w][b & dmask0], 1u);
            }
        }
        __syncthreads();
        for (int d = threadIdx.x; d <= (int)dmask0; d += kPackBlock) {
            uint32_t c = 0;
#pragma unroll
            for (int ww = 0; ww < NW; ++ww) c += hist[ww][d];
            counts[(uint64_t)d * ntiles + tile] = c;
        }
        __syncthreads();
    }
    if (st) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
            bad |= __shfl_xor_sync(0xffffffffu, bad, o);
            uns |= __shfl_xor_sync(0xffffffffu, uns, o);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&st->tmin, lo);
            atomicMax(&st->tmax, hi);
            if (bad) atomicOr(&st->bad, 1u);
            if (uns) atomicOr(&st->unsorted, 1u);
        }
    }
}

template <bool kNarrow>
__global__ void gather_s_kernel(const typename EdgeCodec<kNarrow>::Rec* __restrict__ E, int64_t tmin,
                                const uint64_t* __restrict__ skeys, uint64_t R, uint64_t n,
                                uint32_t* __restrict__ off,
                                int64_t* __restrict__ S_tw, uint32_t* __restrict__ S_tn,
                                uint32_t* __restrict__ S_nbr,
                                uint32_t* __restrict__ S_ord, uint32_t* __restrict__ S_node,
                                uint32_t* __restrict__ omask,
                                int64_t* __restrict__ t32w, uint32_t* __restrict__ t32n,
                                int64_t* __restrict__ t1kw, uint32_t* __restrict__ t1kn) {
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < R;
         base += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t q = base + threadIdx.x;
        uint32_t out = 0;
        if (q < R) {
            const uint64_t key = __ldcs(skeys + q);  // streamed: leave L2 to the edge records
            const uint32_t r = (uint32_t)key;
            const uint32_t p = r >> 1, side = r & 1u;
            using Codec = EdgeCodec<kNarrow>;
            const typename Codec::Rec e = E[p];
            const uint32_t u = (uint32_t)(key >> 32), x = Codec::other(e, u);
            // CSR offsets from the node boundaries of the sorted keys
            const int64_t prev = q ? (int64_t)(skeys[q - 1] >> 32) : -1;
            for (int64_t y = prev + 1; y <= (int64_t)u; ++y) off[y] = (uint32_t)q;
            if (q == R - 1)
                for (int64_t y = (int64_t)u + 1; y <= (int64_t)n; ++y) off[y] = (uint32_t)R;
            out = side ^ 1u;
            if (kNarrow) __stcs(S_tn + q, Codec::rel(e));
            else __stcs(S_tw + q, Codec::time(e, tmin));
            if ((q & 31) == 0) {  // the fences (tm_internal.cuh fenced_lower_bound)
                if (kNarrow) t32n[q >> 5] = Codec::rel(e);
                else t32w[q >> 5] = Codec::time(e, tmin);
                if ((q & 1023) == 0) {
                    if (kNarrow) t1kn[q >> 10] = Codec::rel(e);
                    else t1kw[q >> 10] = Codec::time(e, tmin);
                }
            }
            __stcs(S_ord + q, p);
            __stcs(S_node + q, u);
            __stcs(S_nbr + q, x | (side << 31));
        }
        const unsigned ob = __ballot_sync(0xffffffffu, out);
        if ((threadIdx.x & 31) == 0 && q < R) omask[q >> 5] = ob;
    }
}

// The node sort's first pass over time-ordered input with a narrow time span:
// a tile's kSortTile / 2 edges come straight from the caller's src / dst / t
// (three TMA copies into the tile's key area, 8 bytes per record instead of
// the 16 of packed keys + payloads) and each thread forms its records' keys
// node << 32 | 2k + side and payloads (t - tmin) << 32 | other | side << 31 in
// registers, exactly as pack_edges would have written them.  Needs 16-byte
// aligned arrays (the tile starts are multiples of 6 KB).
struct RawEdgeLoad {
    static constexpr bool kOn = true;
    static constexpr uint32_t kEdges = kSortTile / 2;
    const uint32_t* src;
    const uint32_t* dst;
    const int64_t* t;
    uint64_t m, n;
    int64_t tmin;
    __device__ __forceinline__ void issue(unsigned char* stage, uint32_t tile, uint64_t* bar) const {
        const uint64_t e0 = (uint64_t)tile * kEdges;
        const uint32_t cnt = (uint32_t)(m - e0 < kEdges ? m - e0 : kEdges);
        uint32_t* ss = reinterpret_cast<uint32_t*>(stage);
        uint32_t* sd = ss + kEdges;
        int64_t* st = reinterpret_cast<int64_t*>(stage + kEdges * 8);
        const uint32_t b4 = (cnt * 4u) & ~15u, b8 = (cnt * 8u) & ~15u;
        mbar_expect_tx(bar, 2 * b4 + b8);
        if (b4) {
            tma_load_1d(ss, src + e0, b4, bar);
            tma_load_1d(sd, dst + e0, b4, bar);
        }
        if (b8) tma_load_1d(st, t + e0, b8, bar);
        // the last tile's tail (under 16 bytes per array) by plain loads
        for (uint32_t i = b4 / 4; i < cnt; ++i) {
            ss[i] = src[e0 + i];
            sd[i] = dst[e0 + i];
        }
        for (uint32_t i = b8 / 8; i < cnt; ++i) st[i] = t[e0 + i];
    }
    __device__ __forceinline__ void fetch(const unsigned char* stage, uint32_t tile, uint32_t i, uint64_t& key,
                                          uint64_t& val) const {
        const uint32_t* ss = reinterpret_cast<const uint32_t*>(stage);
        const uint32_t e = i >> 1, side = i & 1u;
        uint32_t a = ss[e], b = ss[kEdges + e];
        a = a < n ? a : 0u;  // clamped like pack_edges: a rejected batch stays in bounds
        b = b < n ? b : 0u;
        const uint64_t rel = (uint64_t)reinterpret_cast<const int64_t*>(stage + kEdges * 8)[e] - (uint64_t)tmin;
        const uint32_t r = 2u * (tile * kEdges + e) + side;
        key = ((uint64_t)(side ? b : a) << 32) | r;
        val = (rel << 32) | (side ? (a | kDirBit) : b);
    }
};

// S for narrow records: the payload (t - tmin) << 32 | other | side << 31
// travelled with the node sort's keys (node << 32 | 2k + side), and the sort's
// LAST downsweep pass hands each (position, key, payload) to this emitter,
// which writes the S arrays and the S_t fences in place of the sorted keys and
// payloads -- no gather of the edge records (a random 8-byte read costs a whole
// 128-byte line from HBM on B200, profiles/gatherbench.cu) and no separate
// pass over the sorted data either (gather_s: 38 GB of traffic at config 4).
struct SEmit {
    static constexpr bool kOn = true;
    uint32_t* S_tn;
    uint32_t* S_nbr;
    uint32_t* S_ord;
    uint32_t* S_node;
    uint32_t* t32n;
    uint32_t* t1kn;
    __device__ __forceinline__ void operator()(uint32_t q, uint64_t key, uint64_t val) const {
        const uint32_t r = (uint32_t)key, trel = (uint32_t)(val >> 32);
        // plain stores: a digit run ends inside a sector that the neighbouring
        // tile's run completes, so the lines should stay in L2 until then
        S_tn[q] = trel;
        S_ord[q] = r >> 1;
        S_node[q] = (uint32_t)(key >> 32);
        S_nbr[q] = ((uint32_t)val & kNodeMask) | ((r & 1u) << 31);
        if ((q & 31) == 0) {  // the fences (tm_internal.cuh fenced_lower_bound)
            t32n[q >> 5] = trel;
            if ((q & 1023) == 0) t1kn[q >> 10] = trel;
        }
    }
};

// CSR offsets from the node boundaries of S_node (the emitter's output):
// four records per thread (one 16-byte load)
__global__ void s_offsets_kernel(const uint32_t* __restrict__ S_node, uint64_t R, uint64_t n,
                                 uint32_t* __restrict__ off) {
    const uint64_t quads = (R + 3) / 4;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < quads; x += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t q0 = x * 4;
        uint32_t u[4];
        if (q0 + 4 <= R) {
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(S_node) + x);
            u[0] = v.x; u[1] = v.y; u[2] = v.z; u[3] = v.w;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) u[k] = q0 + k < R ? S_node[q0 + k] : 0u;
        }
        // node ids are below 2^31, so 0xFFFFFFFF stands for "before node 0";
        // most records repeat their predecessor's node (one compare each)
        uint32_t prev = q0 ? S_node[q0 - 1] : 0xFFFFFFFFu;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint64_t q = q0 + k;
            if (q < R && u[k] != prev) {
                for (uint32_t y = prev + 1u;; ++y) {  // S_node ascends: prev + 1 .. u[k]
                    off[y] = (uint32_t)q;
                    if (y == u[k]) break;
                }
                prev = u[k];
            }
        }
        if (q0 + 4 >= R)  // the quad with the last record closes the remaining nodes
            for (uint64_t y = (uint64_t)prev + 1; y <= n; ++y) off[y] = (uint32_t)R;
    }
}

// pair keys from the upper-side records of S (in (upper, t, ordinal) order):
// lower << 32 | p, compacted by the xmask prefix
// Degree class for the triangle pass's orientation: the degree itself below
// 8, else 3 mantissa bits under the leading bit (~12 % steps) -- monotone in
// the degree, so (class, id) is a strict total order that still puts hubs
// last.  One byte per node (50 MB at 50M nodes) stays in L2 under pair_keys'
// random neighbour reads, where the 4-byte CSR offsets (two per read, 200 MB)
// missed: config 4 pair_keys read 81 GB from HBM for 19 GB of keys and S.
__device__ __forceinline__ uint8_t degree_class(uint32_t d) {
    if (d < 8) return (uint8_t)d;
    const int e = 31 - __clz(d);
    return (uint8_t)(8 + (e - 3) * 8 + ((d >> (e - 3)) & 7u));
}
__global__ void degree_class_kernel(const uint32_t* __restrict__ off, uint64_t n, uint8_t* __restrict__ cls) {
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (uint64_t)gridDim.x * blockDim.x)
        cls[u] = degree_class(off[u + 1] - off[u]);
}

// Orientation of every incident record by (degree class, id): forward
// (fmask: the neighbour ranks above the center -- the degree orientation of
// the triangle pass) or backward (xmask: the center is the pair's upper
// endpoint).  P is keyed by each pair's LOWER endpoint in this order, so a
// pair lookup searches the lower endpoint's block, which holds only its
// records to nodes ranked above it: a low-degree node's block is short, and a
// hub's block holds only its records to the few hubs above it.
__global__ void orient_kernel(const uint32_t* __restrict__ S_node, const uint32_t* __restrict__ S_nbr,
                              const uint8_t* __restrict__ cls, uint64_t R, uint32_t* __restrict__ xmask,
                              uint32_t* __restrict__ fmask, uint32_t* __restrict__ omask) {
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < R; base += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t q = base + threadIdx.x;
        uint32_t fwd = 0, bwd = 0, out = 0;
        if (q < R) {
            const uint32_t u = __ldcs(S_node + q), nbr = __ldcs(S_nbr + q), x = nbr & kNodeMask;
            const uint32_t du = cls[u], dx = cls[x];
            fwd = (dx > du || (dx == du && x > u)) ? 1u : 0u;
            bwd = fwd ^ 1u;
            out = (nbr >> 31) ^ 1u;  // the outward records (the star pass's P_o prefix)
        }
        const unsigned fb = __ballot_sync(0xffffffffu, fwd), bb = __ballot_sync(0xffffffffu, bwd);
        const unsigned ob = __ballot_sync(0xffffffffu, out);
        if ((threadIdx.x & 31) == 0 && q < R) {
            fmask[q >> 5] = fb;
            xmask[q >> 5] = bb;
            omask[q >> 5] = ob;
        }
    }
}

// (narrow records: also the payload (t - tmin) << 32 | max | dir_rel_min << 31
// for gather_p_pay, read from S_t / S_nbr)
__global__ void pair_keys_kernel(const uint32_t* __restrict__ S_node, const uint32_t* __restrict__ S_ord,
                                 const uint32_t* __restrict__ S_nbr, const uint32_t* __restrict__ S_tn,
                                 const uint32_t* __restrict__ xmask, const uint32_t* __restrict__ xpref,
                                 uint64_t R, uint64_t* __restrict__ pkeys, uint64_t* __restrict__ pvals) {
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < R; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t word = xmask[q >> 5], bit = 1u << (q & 31);
        if (!(word & bit)) continue;
        const uint32_t nbr = __ldcs(S_nbr + q);
        const uint32_t u = __ldcs(S_node + q), x = nbr & kNodeMask;
        const uint32_t j = xpref[q >> 5] + __popc(word & (bit - 1u));
        pkeys[j] = ((uint64_t)x << 32) | __ldcs(S_ord + q);
        // u is the upper endpoint; the lower one x is the source iff u's record is inward
        if (pvals) pvals[j] = ((uint64_t)__ldcs(S_tn + q) << 32) | u | ((~nbr) & kDirBit);
    }
}

// P records from the sorted pair keys (min << 32 | p): the max endpoint is
// the edge's other one; group first/last flags compare (min, max) with the
// neighbours, staged through shared memory (block-edge neighbours re-read).
template <bool kNarrow>
__device__ __forceinline__ void pair_of(const uint64_t* __restrict__ pkeys,
                                        const typename EdgeCodec<kNarrow>::Rec* __restrict__ E, uint64_t k,
                                        uint32_t& a, uint32_t& b) {
    const uint64_t key = pkeys[k];
    a = (uint32_t)(key >> 32);
    b = EdgeCodec<kNarrow>::other(E[(uint32_t)key], a);
}

template <bool kNarrow>
__global__ void __launch_bounds__(256) gather_p_kernel(const uint64_t* __restrict__ pkeys, uint64_t m,
                                                       const typename EdgeCodec<kNarrow>::Rec* __restrict__ E,
                                                       int64_t tmin,
                                                       int64_t* __restrict__ P_tw,
                                                       uint32_t* __restrict__ P_tn,
                                                       uint32_t* __restrict__ P_ord,
                                                       uint32_t* __restrict__ P_min,
                                                       uint32_t* __restrict__ P_max,
                                                       uint32_t* __restrict__ P_w, uint64_t n,
                                                       uint32_t* __restrict__ pofs,
                                                       uint32_t* __restrict__ dmask,
                                                       uint32_t* __restrict__ gmask,
                                                       uint32_t* __restrict__ max32, uint32_t* __restrict__ max1k,
                                                       int64_t* __restrict__ t32w, uint32_t* __restrict__ t32n,
                                                       int64_t* __restrict__ t1kw, uint32_t* __restrict__ t1kn) {
    using Codec = EdgeCodec<kNarrow>;
    __shared__ uint32_t s_a[258], s_b[258];
    const int tid = threadIdx.x;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < m;
         base += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = base + tid;
        uint32_t a = 0, b = 0, p = 0;
        bool first = false;
        typename Codec::Rec ed{};
        if (k < m) {
            const uint64_t key = __ldcs(pkeys + k);
            p = (uint32_t)key;
            ed = E[p];
            a = (uint32_t)(key >> 32);
            b = Codec::other(ed, a);
            s_a[tid + 1] = a;
            s_b[tid + 1] = b;
        }
        if (tid == 0 && k > 0 && k - 1 < m) pair_of<kNarrow>(pkeys, E, k - 1, s_a[0], s_b[0]);
        if (tid == (int)blockDim.x - 1 && k + 1 < m)
            pair_of<kNarrow>(pkeys, E, k + 1, s_a[tid + 2], s_b[tid + 2]);
        __syncthreads();
        if (k < m) {
            first = k == 0 || s_a[tid] != a || s_b[tid] != b;
            const bool last = k + 1 == m || s_a[tid + 2] != a || s_b[tid + 2] != b;
            const uint32_t dir_min = Codec::dir_from_min(ed, a);  // 0: min -> max
            if (kNarrow) __stcs(P_tn + k, Codec::rel(ed));
            else __stcs(P_tw + k, Codec::time(ed, tmin));
            __stcs(P_ord + k, p);
            __stcs(P_min + k, a);
            __stcs(P_max + k, b);
            __stcs(P_w + k, (dir_min << 31) | (first ? kPFirst : 0u) | (last ? kPLast : 0u));
            if ((k & 31) == 0) {  // the fences (tm_internal.cuh fenced_lower_bound)
                max32[k >> 5] = b;
                if (kNarrow) t32n[k >> 5] = Codec::rel(ed);
                else t32w[k >> 5] = Codec::time(ed, tmin);
                if ((k & 1023) == 0) {
                    max1k[k >> 10] = b;
                    if (kNarrow) t1kn[k >> 10] = Codec::rel(ed);
                    else t1kw[k >> 10] = Codec::time(ed, tmin);
                }
            }
            // pofs[x] = first P position whose min endpoint is x (block boundaries)
            const int64_t prev = k == 0 ? -1 : (int64_t)s_a[tid];
            for (int64_t x = prev + 1; x <= (int64_t)a; ++x) pofs[x] = (uint32_t)k;
            if (k + 1 == m)
                for (int64_t x = (int64_t)a + 1; x <= (int64_t)n; ++x) pofs[x] = (uint32_t)m;
        }
        const unsigned db = __ballot_sync(0xffffffffu, k < m && Codec::dir_from_min(ed, a));
        const unsigned gb = __ballot_sync(0xffffffffu, first);
        if ((tid & 31) == 0 && k < m) {
            dmask[k >> 5] = db;
            gmask[k >> 5] = gb;
        }
        __syncthreads();
    }
}

// P for narrow records: the pair sort's last pass hands (position, key =
// min << 32 | p, payload = (t - tmin) << 32 | max | dir_rel_min << 31) to this
// emitter, which writes the P columns, the direction bit of P_w and the P
// fences; p_flags_kernel then adds what needs a record's neighbours (group
// first / last flags, pofs, the direction and group-first bitmasks) from
// P_min / P_max / P_w -- 16 bytes per edge instead of gather_p's 36.
struct PEmit {
    static constexpr bool kOn = true;
    uint32_t* P_tn;
    uint32_t* P_ord;
    uint32_t* P_min;
    uint32_t* P_max;
    uint32_t* P_w;
    uint32_t* max32;
    uint32_t* max1k;
    uint32_t* t32n;
    uint32_t* t1kn;
    __device__ __forceinline__ void operator()(uint32_t k, uint64_t key, uint64_t val) const {
        const uint32_t trel = (uint32_t)(val >> 32), b = (uint32_t)val & kNodeMask;
        P_tn[k] = trel;
        P_ord[k] = (uint32_t)key;
        P_min[k] = (uint32_t)(key >> 32);  // re-read by p_flags_kernel
        P_max[k] = b;
        P_w[k] = (uint32_t)val & kDirBit;
        if ((k & 31) == 0) {
            max32[k >> 5] = b;
            t32n[k >> 5] = trel;
            if ((k & 1023) == 0) {
                max1k[k >> 10] = b;
                t1kn[k >> 10] = trel;
            }
        }
    }
};

__global__ void __launch_bounds__(256) p_flags_kernel(const uint32_t* __restrict__ P_min,
                                                      const uint32_t* __restrict__ P_max, uint64_t m, uint64_t n,
                                                      uint32_t* __restrict__ P_w, uint32_t* __restrict__ pofs,
                                                      uint32_t* __restrict__ dmask, uint32_t* __restrict__ gmask) {
    // four records per thread (16-byte loads); the records either side of the
    // quad come from the neighbouring threads' lines (cache hits); eight lanes
    // assemble one word of each bitmask
    const uint64_t quads = (m + 3) / 4, span = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t rounds = (quads + span - 1) / span;  // whole warps stay in the loop (shuffles)
    const int lane = threadIdx.x & 31;
    for (uint64_t r = 0; r < rounds; ++r) {
        const uint64_t x = r * span + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
        const uint64_t k0 = x * 4;
        uint32_t a[6], b[6], w[4];  // [0] = record k0 - 1, [5] = record k0 + 4
        uint32_t dn = 0, gn = 0;
        if (k0 < m) {
            if (k0 + 4 <= m) {
                const uint4 va = *(reinterpret_cast<const uint4*>(P_min) + x), vb = *(reinterpret_cast<const uint4*>(P_max) + x);
                const uint4 vw = *(reinterpret_cast<const uint4*>(P_w) + x);
                a[1] = va.x; a[2] = va.y; a[3] = va.z; a[4] = va.w;
                b[1] = vb.x; b[2] = vb.y; b[3] = vb.z; b[4] = vb.w;
                w[0] = vw.x; w[1] = vw.y; w[2] = vw.z; w[3] = vw.w;
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const bool in = k0 + i < m;
                    a[1 + i] = in ? P_min[k0 + i] : 0u;
                    b[1 + i] = in ? P_max[k0 + i] : 0u;
                    w[i] = in ? P_w[k0 + i] : 0u;
                }
            }
            a[0] = k0 ? P_min[k0 - 1] : 0u;
            b[0] = k0 ? P_max[k0 - 1] : 0u;
            a[5] = k0 + 4 < m ? P_min[k0 + 4] : 0u;
            b[5] = k0 + 4 < m ? P_max[k0 + 4] : 0u;
            uint32_t wo[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint64_t k = k0 + i;
                wo[i] = 0;
                if (k < m) {
                    const bool first = k == 0 || a[i] != a[1 + i] || b[i] != b[1 + i];
                    const bool last = k + 1 == m || a[2 + i] != a[1 + i] || b[2 + i] != b[1 + i];
                    const uint32_t dir = w[i] >> 31;
                    wo[i] = (dir << 31) | (first ? kPFirst : 0u) | (last ? kPLast : 0u);
                    dn |= dir << i;
                    gn |= (first ? 1u : 0u) << i;
                    const int64_t prev = k == 0 ? -1 : (int64_t)a[i];
                    for (int64_t y = prev + 1; y <= (int64_t)a[1 + i]; ++y) pofs[y] = (uint32_t)k;
                    if (k + 1 == m)
                        for (int64_t y = (int64_t)a[1 + i] + 1; y <= (int64_t)n; ++y) pofs[y] = (uint32_t)m;
                }
            }
            if (k0 + 4 <= m) {
                __stcs(reinterpret_cast<uint4*>(P_w) + x, make_uint4(wo[0], wo[1], wo[2], wo[3]));
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (k0 + i < m) P_w[k0 + i] = wo[i];
            }
        }
        dn <<= 4 * (lane & 7);
        gn <<= 4 * (lane & 7);
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            dn |= __shfl_xor_sync(0xffffffffu, dn, o);
            gn |= __shfl_xor_sync(0xffffffffu, gn, o);
        }
        if ((lane & 7) == 0 && k0 < m) {
            dmask[k0 >> 5] = dn;
            gmask[k0 >> 5] = gn;
        }
    }
}

// S -> P index for the per-center items API: each P record finds its two S
// positions by binary search of (t, ordinal) in its endpoints' sequences.
__device__ __forceinline__ uint32_t s_locate(const TimeArr& S_t,
                                             const uint32_t* __restrict__ S_ord, uint32_t lo,
                                             uint32_t hi, int64_t t, uint32_t ord) {
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const int64_t tm = S_t[mid];
        if (tm < t || (tm == t && (S_ord[mid] & kNodeMask) < ord)) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void s_pidx_kernel(TimeArr P_t, const uint32_t* __restrict__ P_ord,
                              const uint32_t* __restrict__ P_min, const uint32_t* __restrict__ P_max,
                              TimeArr S_t, const uint32_t* __restrict__ S_ord,
                              const uint32_t* __restrict__ off, uint64_t m,
                              uint32_t* __restrict__ S_pidx) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t t = P_t[k];
        const uint32_t o = P_ord[k], a = P_min[k], b = P_max[k];
        S_pidx[s_locate(S_t, S_ord, off[a], off[a + 1], t, o)] = (uint32_t)k;
        S_pidx[s_locate(S_t, S_ord, off[b], off[b + 1], t, o)] = (uint32_t)k;
    }
}

// two word-popcount prefixes in one scan: low / high 32 bits of a u64
struct PopcLoad2 {
    const uint32_t* a;
    const uint32_t* b;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
        return (uint64_t)__popc(a[i]) | ((uint64_t)__popc(b[i]) << 32);
    }
};
struct SplitStore2 {
    uint32_t* a;
    uint32_t* b;
    __device__ __forceinline__ void operator()(uint64_t i, uint64_t v) const {
        a[i] = (uint32_t)v;
        b[i] = (uint32_t)(v >> 32);
    }
};
struct PopcLoad {
    const uint32_t* mask;
    __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return __popc(mask[i]); }
};
// forward(u -> x) bitmask for the node-index orientation (removal mode); the
// degree orientation's mask is written by gather_s
__global__ void index_forward_mask_kernel(const uint32_t* __restrict__ node,
                                          const uint32_t* __restrict__ nbr, uint64_t R,
                                          uint32_t* __restrict__ fmask) {
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < R;
         base += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t q = base + threadIdx.x;
        const uint32_t f = q < R && (nbr[q] & kNodeMask) > node[q] ? 1u : 0u;
        const unsigned b = __ballot_sync(0xffffffffu, f);
        if ((threadIdx.x & 31) == 0 && q < R) fmask[q >> 5] = b;
    }
}

// F position of forward record q = fpref[q/32] + popc(fmask[q/32] & below)
__global__ void forward_scatter_kernel(const uint32_t* __restrict__ fmask,
                                       const uint32_t* __restrict__ fpref, uint64_t R,
                                       const int64_t* __restrict__ S_tw,
                                       const uint32_t* __restrict__ S_tn,
                                       const uint32_t* __restrict__ S_nbr,
                                       const uint32_t* __restrict__ S_ord,
                                       const uint32_t* __restrict__ S_node, int64_t* __restrict__ F_tw,
                                       uint32_t* __restrict__ F_tn,
                                       uint32_t* __restrict__ F_nbr, uint32_t* __restrict__ F_ord,
                                       uint32_t* __restrict__ F_node) {
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < R;
         q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t word = fmask[q >> 5], bit = 1u << (q & 31);
        if (word & bit) {
            const uint32_t j = fpref[q >> 5] + __popc(word & (bit - 1u));
            if (S_tn) F_tn[j] = S_tn[q];
            else F_tw[j] = S_tw[q];
            F_nbr[j] = S_nbr[q];
            F_ord[j] = S_ord[q] & kNodeMask;
            F_node[j] = S_node[q];
        }
    }
}

__global__ void forward_off_kernel(const uint32_t* __restrict__ off, const uint32_t* __restrict__ fmask,
                                   const uint32_t* __restrict__ fpref, uint64_t n,
                                   uint32_t* __restrict__ F_off) {
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u <= n;
         u += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = off[u];
        F_off[u] = fpref[q >> 5] + __popc(fmask[q >> 5] & ((1u << (q & 31)) - 1u));
    }
}

// time-slice partition: keep edges with t in [lo, hi) (ingestion order kept)
// keep lo <= t <= hi (both inclusive: an open end is INT64_MIN / INT64_MAX
// and keeps every timestamp)
__global__ void slice_mask_kernel(const int64_t* __restrict__ t, uint64_t m, int64_t lo, int64_t hi,
                                  uint32_t* __restrict__ mask) {
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < m;
         base += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = base + threadIdx.x;
        const uint32_t keep = k < m && t[k] >= lo && t[k] <= hi ? 1u : 0u;
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        if ((threadIdx.x & 31) == 0 && k < m) mask[k >> 5] = b;
    }
}

__global__ void slice_scatter_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                     const int64_t* __restrict__ t, uint64_t m,
                                     const uint32_t* __restrict__ mask, const uint32_t* __restrict__ pref,
                                     uint32_t* __restrict__ osrc, uint32_t* __restrict__ odst,
                                     int64_t* __restrict__ ot) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t word = mask[k >> 5], bit = 1u << (k & 31);
        if (word & bit) {
            const uint32_t j = pref[k >> 5] + __popc(word & (bit - 1u));
            osrc[j] = src[k];
            odst[j] = dst[k];
            ot[j] = t[k];
        }
    }
}

unsigned grid_for(uint64_t work, int block = 256) {
    const uint64_t cap = (uint64_t)sm_count() * 8;
    uint64_t g = (work + block - 1) / block;
    if (g < 1) g = 1;
    return (unsigned)(g < cap ? g : cap);
}

// Side streams and events, recycled per host thread (creating and
// destroying them per graph costs tens of microseconds of host time).
struct SideSet {
    cudaStream_t aux[2];
    cudaEvent_t ev[3];
};
struct SidePool {
    std::vector<SideSet> free_sets;
    ~SidePool() {
        for (auto& x : free_sets) {
            for (auto a : x.aux) cudaStreamDestroy(a);
            for (auto e : x.ev) cudaEventDestroy(e);
        }
    }
};
thread_local SidePool g_side_pool;

void acquire_side(DeviceGraph& g) {
    SideSet x;
    if (!g_side_pool.free_sets.empty()) {
        x = g_side_pool.free_sets.back();
        g_side_pool.free_sets.pop_back();
    } else {
        for (auto& a : x.aux) TM_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
        for (auto& e : x.ev) TM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    g.aux[0] = x.aux[0];
    g.aux[1] = x.aux[1];
    g.ev_fork = x.ev[0];
    g.ev_join = x.ev[1];
    g.fwd_ready = x.ev[2];
}

void release_side(DeviceGraph& g) {
    g_side_pool.free_sets.push_back(SideSet{{g.aux[0], g.aux[1]}, {g.ev_fork, g.ev_join, g.fwd_ready}});
    g.aux[0] = g.aux[1] = nullptr;
    g.ev_fork = g.ev_join = g.fwd_ready = nullptr;
}

}  // namespace

static bool raw_first_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TM_RAW_FIRST");
        return !(e && e[0] == '0');
    }();
    return on;
}

BuildPlan build_prepare(DeviceGraph& g, const uint32_t* d_src, const uint32_t* d_dst, const int64_t* d_t,
                        uint64_t m, uint64_t n, BuildWorkspace* ws, BuildVerdict* h_async) {
    cudaStream_t s = g.stream;
    if (2 * m > 0xFFFFFFF0ull) throw tm_error(9, "graph too large: 2m must fit 32-bit positions");
    if (!g.aux[0]) acquire_side(g);
    if (n > kNodeMask) throw tm_error(9, "graph too large: node ids must fit 31 bits");
    g.n = n;
    g.m = m;
    g.R = 2 * m;
    const uint64_t R = g.R;

    // 1. pack + validate in one pass, assuming time-ordered input and a time
    //    span that fits narrow records; one 4-word read-back decides whether
    //    to re-pack (time sort first / wide records)
    BuildPlan pl;
    pl.ntiles = (uint32_t)((R + kSortTile - 1) / kSortTile);
    pl.owned = ws == nullptr;
    BuildStats* d_st;
    if (ws) {  // persistent buffers (graph replay): sized for wide records
        if (!ws->nk0) {
            ws->nk0 = dalloc<uint64_t>(R + kSortPad, s);
            ws->nk1 = dalloc<uint64_t>(R + kSortPad, s);
            ws->nv0 = dalloc<uint64_t>(R + kSortPad, s);
            ws->nv1 = dalloc<uint64_t>(R + kSortPad, s);
            ws->c0 = dalloc<uint32_t>((uint64_t)kRadix * pl.ntiles, s);
            ws->E = dalloc<uint8_t>(m * sizeof(WideEdge), s);
            ws->st = dalloc<uint8_t>(sizeof(BuildStats), s);
        }
        pl.nk0 = ws->nk0;
        pl.nk1 = ws->nk1;
        pl.nv0 = ws->nv0;
        pl.nv1 = ws->nv1;
        pl.c0 = ws->c0;
        pl.E = ws->E;
        pl.E_bytes = m * sizeof(WideEdge);
        d_st = reinterpret_cast<BuildStats*>(ws->st);
    } else {
        pl.nk0 = dalloc<uint64_t>(R + kSortPad, s);
        pl.nk1 = dalloc<uint64_t>(R + kSortPad, s);
        pl.nv0 = dalloc<uint64_t>(R + kSortPad, s);
        pl.nv1 = dalloc<uint64_t>(R + kSortPad, s);
        pl.c0 = dalloc<uint32_t>((uint64_t)kRadix * pl.ntiles, s);
        pl.E = dalloc<uint8_t>(m * sizeof(NarrowEdge), s);
        pl.E_bytes = m * sizeof(NarrowEdge);
        d_st = dalloc<BuildStats>(1, s);
    }
    BuildStats h_st{LLONG_MAX, LLONG_MIN, 0, 0, 0, 0};
    BuildStats* hv = h_async ? h_async : &h_st;
    *hv = h_st;
    TM_CUDA(cudaMemcpyAsync(d_st, hv, sizeof(h_st), cudaMemcpyHostToDevice, s));
    if (m) {
        // scan only when the node sort can read the arrays itself (RawEdgeLoad)
        pl.raw_first = raw_first_enabled() && ((reinterpret_cast<uintptr_t>(d_src) | reinterpret_cast<uintptr_t>(d_dst) |
                                                reinterpret_cast<uintptr_t>(d_t)) & 15u) == 0;
        if (pl.raw_first)
            TM_LAUNCH("pack_edges", s, (pack_edges_kernel<true, false, true>), grid_for(m, kPackEdges), kPackBlock, 0,
                      nullptr, nullptr, 0ull, d_src, d_dst, d_t, m, n, (int64_t)0,
                      reinterpret_cast<NarrowEdge*>(pl.E), pl.nk0, pl.nv0, pl.c0, pl.ntiles, d_st);
        else
            TM_LAUNCH("pack_edges", s, (pack_edges_kernel<true, false>), grid_for(m, kPackEdges), kPackBlock, 0,
                      nullptr, nullptr, 0ull, d_src, d_dst, d_t, m, n, (int64_t)0,
                      reinterpret_cast<NarrowEdge*>(pl.E), pl.nk0, pl.nv0, pl.c0, pl.ntiles, d_st);
    }
    TM_CUDA(cudaMemcpyAsync(hv, d_st, sizeof(h_st), cudaMemcpyDeviceToHost, s));
    if (h_async) return pl;  // verdict read later (plan_from_verdict)
    TM_CUDA(cudaStreamSynchronize(s));
    if (!ws) dfree(d_st, s);
    plan_from_verdict(g, pl, h_st);
    return pl;
}

void plan_from_verdict(DeviceGraph& g, BuildPlan& pl, const BuildVerdict& v) {
    if (v.bad) {
        release_plan(g, pl);
        throw tm_error(1, "self-loop or out-of-range endpoint in edge list");
    }
    // narrow 8-byte edge records when the time span fits 32 bits
    // (offsets stay <= 0xFFFFFFFE: TimeKey's u32 threshold 0xFFFFFFFF means "every record")
    pl.narrow = (uint64_t)v.tmax - (uint64_t)v.tmin < 0xFFFFFFFFull;
    pl.unsorted = v.unsorted != 0;
    pl.tmin = v.tmin;
    pl.tmax = v.tmax;
}

void release_plan(DeviceGraph& g, BuildPlan& pl) {
    if (!pl.owned) return;
    cudaStream_t s = g.stream;
    dfree(pl.nk0, s); dfree(pl.nk1, s); dfree(pl.nv0, s); dfree(pl.nv1, s); dfree(pl.c0, s); dfree(pl.E, s);
}

void build_graph(DeviceGraph& g, const uint32_t* d_src, const uint32_t* d_dst, const int64_t* d_t,
                 uint64_t m, uint64_t n, const RunHint* hint) {
    BuildPlan pl = build_prepare(g, d_src, d_dst, d_t, m, n, nullptr, nullptr);
    build_finish(g, pl, d_src, d_dst, d_t, hint);
}

template <bool kNarrow, bool kPermuted>
void launch_repack(const uint32_t* perm, const uint64_t* tkeys, uint64_t kmask, const uint32_t* d_src,
                   const uint32_t* d_dst, const int64_t* d_t, uint64_t m, uint64_t n, int64_t tmin, uint8_t* E,
                   uint64_t* keys, uint64_t* vals, uint32_t* counts, uint32_t ntiles, cudaStream_t s) {
    TM_LAUNCH("pack_edges", s, (pack_edges_kernel<kNarrow, kPermuted>), grid_for(m, kPackEdges), kPackBlock, 0, perm,
              tkeys, kmask, d_src, d_dst, d_t, m, n, tmin,
              reinterpret_cast<typename EdgeCodec<kNarrow>::Rec*>(E), keys, vals, counts, ntiles, nullptr);
}

void build_finish(DeviceGraph& g, BuildPlan& pl, const uint32_t* d_src, const uint32_t* d_dst,
                  const int64_t* d_t, const RunHint* hint) {
    cudaStream_t s = g.stream;
    const uint64_t m = g.m, n = g.n, R = g.R;
    const bool narrow = pl.narrow;
    const int64_t tmin = pl.tmin;
    const bool repack = m && (pl.unsorted || !narrow);
    BuildStats h_st{pl.tmin, pl.tmax, 0, pl.unsorted ? 1u : 0u, 0, 0};
    uint64_t* nk0 = pl.nk0;
    uint64_t* nk1 = pl.nk1;
    uint64_t* nv0 = pl.nv0;
    uint64_t* nv1 = pl.nv1;
    uint32_t* c0 = pl.c0;
    uint8_t* E = pl.E;
    const uint32_t ntiles = pl.ntiles;

    g.off = dalloc<uint32_t>(n + 1, s);
    g.pofs = dalloc<uint32_t>(n + 1, s);
    g.tbase = narrow ? tmin : 0;
    if (narrow) g.S_t.n = dalloc<uint32_t>(R, s);
    else g.S_t.w = dalloc<int64_t>(R, s);
    if (narrow) {
        g.S_t32.n = dalloc<uint32_t>(R / 32 + 1, s);
        g.S_t1k.n = dalloc<uint32_t>(R / 1024 + 1, s);
    } else {
        g.S_t32.w = dalloc<int64_t>(R / 32 + 1, s);
        g.S_t1k.w = dalloc<int64_t>(R / 1024 + 1, s);
    }
    g.S_nbr = dalloc<uint32_t>(R, s);
    g.S_ord = dalloc<uint32_t>(R, s);
    g.S_node = dalloc<uint32_t>(R, s);
    const uint64_t nw = R / 32 + 1;  // mask words (+1: a zero word past the end)
    g.S_omask = dalloc<uint32_t>(nw, s);
    g.S_opref = dalloc<uint32_t>(nw + 1, s);
    g.S_fmask = dalloc<uint32_t>(nw, s);
    if (narrow) g.P_t.n = dalloc<uint32_t>(m, s);
    else g.P_t.w = dalloc<int64_t>(m, s);
    g.P_ord = dalloc<uint32_t>(m, s);
    g.P_max = dalloc<uint32_t>(m, s);
    g.P_w = dalloc<uint32_t>(m, s);
    g.P_min = dalloc<uint32_t>(m, s);
    g.P_dmask = dalloc<uint32_t>(m / 32 + 1, s);
    g.P_dpref = dalloc<uint32_t>(m / 32 + 2, s);
    g.P_gmask = dalloc<uint32_t>(m / 32 + 1, s);
    g.P_gpref = dalloc<uint32_t>(m / 32 + 2, s);
    g.P_max32 = dalloc<uint32_t>(m / 32 + 1, s);
    g.P_max1k = dalloc<uint32_t>(m / 1024 + 1, s);
    if (narrow) {
        g.P_t32.n = dalloc<uint32_t>(m / 32 + 1, s);
        g.P_t1k.n = dalloc<uint32_t>(m / 1024 + 1, s);
    } else {
        g.P_t32.w = dalloc<int64_t>(m / 32 + 1, s);
        g.P_t1k.w = dalloc<int64_t>(m / 1024 + 1, s);
    }
    TM_CUDA(cudaMemsetAsync(g.P_dmask + m / 32, 0, sizeof(uint32_t), s));
    TM_CUDA(cudaMemsetAsync(g.P_gmask + m / 32, 0, sizeof(uint32_t), s));

    if (m == 0) {
        release_plan(g, pl);
        TM_CUDA(cudaMemsetAsync(g.off, 0, (n + 1) * sizeof(uint32_t), s));
        TM_CUDA(cudaMemsetAsync(g.pofs, 0, (n + 1) * sizeof(uint32_t), s));
        g.cls = dalloc<uint8_t>(n + 1, s);
        TM_CUDA(cudaMemsetAsync(g.cls, 0, n + 1, s));
        TM_CUDA(cudaMemsetAsync(g.S_omask, 0, nw * sizeof(uint32_t), s));
        TM_CUDA(cudaMemsetAsync(g.S_opref, 0, (nw + 1) * sizeof(uint32_t), s));
        g.max_degree = 0;
        return;
    }
    uint32_t* nullv = nullptr;
    uint32_t* nullv2 = nullptr;

    // 1. (t, ordinal) order of the edges (skipped for time-ordered input):
    //    input indices in the low kbits of the sorted packed keys, or the
    //    sorted values when (t - tmin, index) does not fit 64 bits
    uint32_t* perm = nullptr;
    uint64_t* tkeys = nullptr;
    uint64_t kmask = 0;
    if (h_st.unsorted) {
        const int tbits = bit_width_u64((uint64_t)h_st.tmax - (uint64_t)h_st.tmin);
        const int kbits = bit_width_u64(m - 1 ? m - 1 : 1);
        const bool packed = tbits + kbits <= 64;
        uint64_t* k0 = dalloc<uint64_t>(m + kSortPad, s);
        uint64_t* k1 = dalloc<uint64_t>(m + kSortPad, s);
        uint32_t* v0 = packed ? nullptr : dalloc<uint32_t>(m + kSortPad, s);
        uint32_t* v1 = packed ? nullptr : dalloc<uint32_t>(m + kSortPad, s);
        TM_LAUNCH("time_keys", s, time_keys_kernel, grid_for(m), 256, 0, d_t, m, (int64_t)h_st.tmin,
                  kbits, packed, k0, v0);
        if (packed) {
            radix_sort<uint64_t>(k0, nullv, k1, nullv2, m, kbits, kbits + tbits, s);
            tkeys = k0;
            kmask = (1ull << kbits) - 1;
            dfree(k1, s);
        } else {
            radix_sort<uint64_t>(k0, v0, k1, v1, m, 0, tbits, s);
            perm = v0;
            dfree(v1, s);
            dfree(k0, s);
            dfree(k1, s);
        }
    }

    // 2. S: stable sort of the incident records by node (key node << 32 | r)
    const int nb = bit_width_u64(n > 1 ? n - 1 : 1);
    {
        if (repack) {
            if (!narrow && pl.E_bytes < m * sizeof(WideEdge)) {
                dfree(E, s);
                E = dalloc<uint8_t>(m * sizeof(WideEdge), s);
                pl.E = E;
                pl.E_bytes = m * sizeof(WideEdge);
            }
            const bool permuted = perm || tkeys;
            if (narrow && permuted) launch_repack<true, true>(perm, tkeys, kmask, d_src, d_dst, d_t, m, n, tmin, E, nk0, nv0, c0, ntiles, s);
            else if (narrow) launch_repack<true, false>(perm, tkeys, kmask, d_src, d_dst, d_t, m, n, tmin, E, nk0, nv0, c0, ntiles, s);
            else if (permuted) launch_repack<false, true>(perm, tkeys, kmask, d_src, d_dst, d_t, m, n, tmin, E, nk0, nullptr, c0, ntiles, s);
            else launch_repack<false, false>(perm, tkeys, kmask, d_src, d_dst, d_t, m, n, tmin, E, nk0, nullptr, c0, ntiles, s);
            // the gathers read ordinals from the keys: the order is no longer needed
            if (perm) dfree(perm, s);
            if (tkeys) dfree(tkeys, s);
        }
        auto EW = reinterpret_cast<WideEdge*>(E);
        // narrow records: the S payload travels with the keys (no gather)
        const SEmit semit{g.S_t.n, g.S_nbr, g.S_ord, g.S_node, g.S_t32.n, g.S_t1k.n};
        if (narrow && !repack && pl.raw_first)
            radix_sort<uint64_t, uint64_t, SEmit, RawEdgeLoad>(nk0, nv0, nk1, nv1, R, 32, 32 + nb, s, c0, semit,
                                                               RawEdgeLoad{d_src, d_dst, d_t, m, n, tmin});
        else if (narrow)
            radix_sort<uint64_t, uint64_t, SEmit>(nk0, nv0, nk1, nv1, R, 32, 32 + nb, s, c0, semit);
        else radix_sort<uint64_t>(nk0, nullv, nk1, nullv2, R, 32, 32 + nb, s, c0);
        if (pl.owned) dfree(c0, s);
        TM_CUDA(cudaMemsetAsync(g.S_omask + (nw - 1), 0, sizeof(uint32_t), s));
        TM_CUDA(cudaMemsetAsync(g.S_fmask + (nw - 1), 0, sizeof(uint32_t), s));
        uint32_t* xmask = dalloc<uint32_t>(nw, s);
        uint32_t* xpref = dalloc<uint32_t>(nw + 1, s);
        TM_CUDA(cudaMemsetAsync(xmask + (nw - 1), 0, sizeof(uint32_t), s));
        g.cls = dalloc<uint8_t>(n + 1, s);  // kept: the pair lookups pick a pair's lower endpoint by it
        if (narrow)  // the sort's last pass wrote S; the CSR offsets from its node column
            TM_LAUNCH("s_offsets", s, s_offsets_kernel, grid_for((R + 3) / 4), 256, 0, g.S_node, R, n, g.off);
        else
            TM_LAUNCH("gather_s", s, gather_s_kernel<false>, grid_for(R), 256, 0, EW, tmin, nk0, R, n, g.off,
                      g.S_t.w, g.S_t.n, g.S_nbr, g.S_ord, g.S_node, g.S_omask, g.S_t32.w, g.S_t32.n,
                      g.S_t1k.w, g.S_t1k.n);
        // orientation by (degree class, id): forward mask (triangle pass) and
        // upper-side mask (pair keys)
        TM_LAUNCH("degree_class", s, degree_class_kernel, grid_for(n), 256, 0, g.off, n, g.cls);
        TM_LAUNCH("orient", s, orient_kernel, grid_for(R), 256, 0, g.S_node, g.S_nbr, g.cls, R, xmask, g.S_fmask,
                  g.S_omask);
        // outward prefix (stars) and upper-side prefix (pair keys) in one scan
        exclusive_scan_to<uint64_t>(PopcLoad2{g.S_omask, xmask}, nw, SplitStore2{g.S_opref, xpref}, s);

        // 3. P: the max-side records (one per edge, (max, t, ordinal) order)
        //    stably sorted by the min endpoint
        uint64_t* pk0 = dalloc<uint64_t>(m + kSortPad, s);
        uint64_t* pk0_alloc = pk0;
        uint64_t* pk1 = nk1;  // R + pad >= m + pad
        uint64_t* spare = nk1;  // the node sort's second buffer (plan-owned)
        nk1 = nullptr;
        uint64_t* pv0 = narrow ? dalloc<uint64_t>(m + kSortPad, s) : nullptr;
        uint64_t* pv0_alloc = pv0;
        uint64_t* pv1 = nv1;  // the node sort's second value buffer
        TM_LAUNCH("pair_keys", s, pair_keys_kernel, grid_for(R), 256, 0, g.S_node, g.S_ord, g.S_nbr, g.S_t.n, xmask, xpref, R,
                  pk0,
                  pv0);

        // the forward sequences (degree orientation) only need S and the
        // forward mask: build them on a side stream while the pair index sorts
        stream_after(g, g.aux[0], s);
        build_forward(g, 0, g.aux[0]);
        if (hint && hint->early_tri)  // the one-shot count's triangle filter needs F only
            tri_filter_stage(g, g.fwd[0], hint->delta, 0, (uint32_t)g.fwd[0].len, g.aux[0], g.pre_tri);
        TM_CUDA(cudaEventRecord(g.fwd_ready, g.aux[0]));
        g.fwd_pending = true;
        if (pl.owned) {
            dfree(nk0, s);
            dfree(nv0, s);
        }
        dfree(xmask, s);
        dfree(xpref, s);
        if (narrow) {
            radix_sort<uint64_t, uint64_t, PEmit>(pk0, pv0, pk1, pv1, m, 32, 32 + nb, s, nullptr,
                                                  PEmit{g.P_t.n, g.P_ord, g.P_min, g.P_max, g.P_w, g.P_max32,
                                                        g.P_max1k, g.P_t32.n, g.P_t1k.n});
            TM_LAUNCH("p_flags", s, p_flags_kernel, grid_for((m + 3) / 4), 256, 0, g.P_min, g.P_max, m, n, g.P_w, g.pofs,
                      g.P_dmask, g.P_gmask);
        } else {
            radix_sort<uint64_t>(pk0, nullv, pk1, nullv2, m, 32, 32 + nb, s);
            TM_LAUNCH("gather_p", s, gather_p_kernel<false>, grid_for(m), 256, 0, pk0, m, EW, tmin, g.P_t.w, g.P_t.n,
                      g.P_ord, g.P_min, g.P_max, g.P_w, n, g.pofs, g.P_dmask, g.P_gmask, g.P_max32, g.P_max1k,
                      g.P_t32.w, g.P_t32.n, g.P_t1k.w, g.P_t1k.n);
        }
        dfree(pk0_alloc, s);
        dfree(pv0_alloc, s);
        // direction prefix and group-first prefix in one scan
        exclusive_scan_to<uint64_t>(PopcLoad2{g.P_dmask, g.P_gmask}, m / 32 + 1, SplitStore2{g.P_dpref, g.P_gpref},
                                    s);
        if (pl.owned) {
            dfree(spare, s);
            dfree(nv1, s);
            dfree(E, s);
        }
    }
    g.max_degree = 0;  // not needed by the layout (positions are global 32-bit)
}

void stream_after(DeviceGraph& g, cudaStream_t st, cudaStream_t from) {
    if (st == from) return;
    for (int i = 0; i < 2; ++i)
        if (st == g.aux[i]) g.aux_used[i] = true;
    TM_CUDA(cudaEventRecord(g.ev_fork, from));
    TM_CUDA(cudaStreamWaitEvent(st, g.ev_fork, 0));
}

void build_forward(DeviceGraph& g, int mode, cudaStream_t s) {
    Forward& f = g.fwd[mode];
    if (f.valid) {
        if (mode == 0 && g.fwd_pending) TM_CUDA(cudaStreamWaitEvent(s, g.fwd_ready, 0));
        return;
    }
    const uint64_t R = g.R;
    f.mode = mode;
    f.len = g.m;  // every edge is forward from exactly one endpoint
    if (g.S_t.n) f.t.n = dalloc<uint32_t>(g.m, s);
    else f.t.w = dalloc<int64_t>(g.m, s);
    f.nbr = dalloc<uint32_t>(g.m, s);
    f.ord = dalloc<uint32_t>(g.m, s);
    f.node = dalloc<uint32_t>(g.m, s);
    f.off = dalloc<uint32_t>(g.n + 1, s);
    const uint64_t nw = R / 32 + 1;
    uint32_t* fmask = g.S_fmask;
    uint32_t* imask = nullptr;
    if (mode == 1) {
        imask = dalloc<uint32_t>(nw, s);
        TM_CUDA(cudaMemsetAsync(imask + (nw - 1), 0, sizeof(uint32_t), s));
        if (R) {
            TM_LAUNCH("forward_mask", s, index_forward_mask_kernel, grid_for(R), 256, 0, g.S_node, g.S_nbr,
                      R, imask);
        }
        fmask = imask;
    }
    uint32_t* fpref = dalloc<uint32_t>(nw + 1, s);
    exclusive_scan<uint32_t>(PopcLoad{fmask}, nw, fpref, s);
    if (R) {
        TM_LAUNCH("forward_scatter", s, forward_scatter_kernel, grid_for(R), 256, 0, fmask, fpref, R, g.S_t.w,
                  g.S_t.n, g.S_nbr, g.S_ord, g.S_node, f.t.w, f.t.n, f.nbr, f.ord, f.node);
    }
    TM_LAUNCH("forward_off", s, forward_off_kernel, grid_for(g.n + 1), 256, 0, g.off, fmask, fpref, g.n,
              f.off);
    dfree(fpref, s);
    dfree(imask, s);
    f.valid = true;
}

uint64_t slice_edges(const uint32_t* d_src, const uint32_t* d_dst, const int64_t* d_t, uint64_t m,
                     int64_t lo, int64_t hi, uint32_t** o_src, uint32_t** o_dst, int64_t** o_t,
                     cudaStream_t s) {
    const uint64_t nw = m / 32 + 1;
    uint32_t* mask = dalloc<uint32_t>(nw, s);
    uint32_t* pref = dalloc<uint32_t>(nw + 1, s);
    TM_CUDA(cudaMemsetAsync(mask + (nw - 1), 0, sizeof(uint32_t), s));
    if (m) {
        TM_LAUNCH("slice_mask", s, slice_mask_kernel, grid_for(m), 256, 0, d_t, m, lo, hi, mask);
    }
    exclusive_scan<uint32_t>(PopcLoad{mask}, nw, pref, s);
    uint32_t cnt = 0;
    TM_CUDA(cudaMemcpyAsync(&cnt, pref + nw, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    *o_src = dalloc<uint32_t>(cnt, s);
    *o_dst = dalloc<uint32_t>(cnt, s);
    *o_t = dalloc<int64_t>(cnt, s);
    if (m && cnt) {
        TM_LAUNCH("slice_scatter", s, slice_scatter_kernel, grid_for(m), 256, 0, d_src, d_dst, d_t, m, mask,
                  pref, *o_src, *o_dst, *o_t);
    }
    dfree(mask, s);
    dfree(pref, s);
    return cnt;
}

void build_s_pidx(DeviceGraph& g) {
    if (g.S_pidx || g.m == 0) {
        if (!g.S_pidx) g.S_pidx = dalloc<uint32_t>(1, g.stream);
        return;
    }
    g.S_pidx = dalloc<uint32_t>(g.R, g.stream);
    TM_LAUNCH("s_pidx", g.stream, s_pidx_kernel, grid_for(g.m), 256, 0, g.P_t.view(g.tbase), g.P_ord, g.P_min,
              g.P_max, g.S_t.view(g.tbase), g.S_ord, g.off, g.m, g.S_pidx);
}

void free_graph(DeviceGraph& g) {
    cudaStream_t s = g.stream;
    if (g.aux[0]) {
        // the frees below are ordered after everything the side streams did
        // (only streams that were forked: joining an unused one would tie a
        // captured stream to uncaptured work)
        for (int i = 0; i < 2; ++i)
            if (g.aux_used[i]) stream_after(g, s, g.aux[i]);
        g.aux_used[0] = g.aux_used[1] = false;
        release_side(g);
    }
    g.fwd_pending = false;
    dfree(g.S_t.w, s); dfree(g.S_t.n, s); dfree(g.S_nbr, s); dfree(g.S_ord, s); dfree(g.S_node, s);
    dfree(g.S_omask, s); dfree(g.S_opref, s); dfree(g.S_fmask, s); dfree(g.S_pidx, s);
    dfree(g.off, s);
    dfree(g.cls, s);
    dfree(g.S_t32.w, s); dfree(g.S_t32.n, s); dfree(g.S_t1k.w, s); dfree(g.S_t1k.n, s);
    dfree(g.P_t.w, s); dfree(g.P_t.n, s); dfree(g.P_ord, s); dfree(g.P_max, s); dfree(g.P_w, s);
    dfree(g.P_min, s); dfree(g.pofs, s); dfree(g.P_dmask, s); dfree(g.P_dpref, s);
    dfree(g.P_gmask, s); dfree(g.P_gpref, s);
    dfree(g.P_max32, s); dfree(g.P_max1k, s); dfree(g.P_t32.w, s); dfree(g.P_t32.n, s); dfree(g.P_t1k.w, s);
    dfree(g.P_t1k.n, s);
    dfree(g.pre_tri.wedges, s); dfree(g.pre_tri.long_list, s); dfree(g.pre_tri.wbuf, s);
    g.pre_tri.valid = false;
    for (auto& f : g.fwd) {
        dfree(f.t.w, s); dfree(f.t.n, s); dfree(f.nbr, s); dfree(f.ord, s); dfree(f.node, s); dfree(f.off, s);
        f.valid = false;
    }
    dfree(g.d_acc, s);
}

}  // namespace tmb
