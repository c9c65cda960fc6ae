// tm_primitives.cuh -- own-written device-wide scan and stable LSD radix sort.
//
// The radix sort orders the incident records by (node, t, ordinal) exactly as
// the reference's std::sort with the (t, ordinal) comparator followed by the
// CSR fill does (graph.cpp:37-41, indexes.cpp:7-26): keys are stable-sorted,
// and records enter the sort in (t, ordinal) order, so ties keep input order.
//
// Scan: chunked reduce-then-scan (one contiguous chunk per block, no
// inter-block waiting).  Sort: LSD, 8-bit digits, 2048-key tiles; per pass an
// upsweep (per-tile digit counts), a row scan (one block per digit) and a
// persistent downsweep that streams the next tile into shared memory with TMA
// (cp.async.bulk + mbarrier) while it ranks the current one (peer masks from
// __match_any_sync for one of the eight rounds and a ballot multi-split for the
// rest, so the ADU and ALU pipes share the work; per-warp running counts keep
// input order), reorders it in place in shared memory and writes each digit
// run as one burst.  Ranking, not HBM, bounds a pass (profiles/sortbench.cu,
// profiles/rankbench.cu).  Keys carry their payload in the low bits when it
// fits, so most sorts are keys-only.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <string>

#include "tm_internal.cuh"

#ifndef TM_RANK_MATCH_ROUNDS
#define TM_RANK_MATCH_ROUNDS 1  // of the 8 ranking rounds per tile, how many use match.any
#endif

namespace tmb {

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// exclusive scan across a block of NW warps; *total (shared) gets the sum
template <typename T, int NW>
__device__ __forceinline__ T block_exclusive_scan(T v, T* total) {
    __shared__ T warp_tot[NW];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T inc = warp_inclusive_scan(v);
    if (lane == 31) warp_tot[w] = inc;
    __syncthreads();
    if (w == 0) {
        T x = lane < NW ? warp_tot[lane] : T(0);
        T xi = warp_inclusive_scan(x);
        if (lane < NW) warp_tot[lane] = xi - x;
        if (lane == NW - 1 && total) *total = xi;
    }
    __syncthreads();
    T r = warp_tot[w] + inc - v;
    __syncthreads();
    return r;
}

// Block-wide reservation in two lists at once: each thread asks for `a` slots
// of list A and `b` of list B and gets its first slot in each; one global
// atomic per list per block call (all threads of the block call).  The counts
// travel packed 16/16 through one u32 scan, so a block's total per list must
// stay below 65536.  No trailing barrier is needed: the shared words are only
// rewritten after every warp has passed the next call's first barrier.
template <int NW, typename CA>
__device__ __forceinline__ void block_reserve2(uint32_t a, uint32_t b, CA* ca, uint32_t* cb,
                                               CA& oa, uint32_t& ob) {
    __shared__ uint32_t s_w[NW];
    __shared__ CA s_base_a;
    __shared__ uint32_t s_base_b;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t v = (b << 16) | a;
    const uint32_t inc = warp_inclusive_scan(v);
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    if (w == 0) {
        const uint32_t x = lane < NW ? s_w[lane] : 0u;
        const uint32_t xi = warp_inclusive_scan(x);
        if (lane < NW) s_w[lane] = xi - x;
        if (lane == NW - 1) {
            const uint32_t ta = xi & 0xffffu, tb = xi >> 16;
            s_base_a = ta ? atomicAdd(ca, (CA)ta) : (CA)0;
            s_base_b = tb ? atomicAdd(cb, tb) : 0u;
        }
    }
    __syncthreads();
    const uint32_t ex = s_w[w] + inc - v;
    oa = s_base_a + (ex & 0xffffu);
    ob = s_base_b + (ex >> 16);
}

// Dynamic work queue: the warp's next `n` items (lane 0 takes them, all
// lanes get the base).  Work kernels with heavy-tailed items (hub windows,
// long same-neighbour walks) pull chunks instead of striding a fixed share,
// so no warp idles while another still holds a long tail.
__device__ __forceinline__ unsigned long long warp_take(unsigned long long* queue, unsigned n) {
    unsigned long long b = 0;
    if ((threadIdx.x & 31) == 0) b = atomicAdd(queue, (unsigned long long)n);
    return __shfl_sync(0xffffffffu, b, 0);
}

// warp-aggregated append of `value` to list when pred holds (whole warp calls)
__device__ __forceinline__ void warp_append(bool pred, uint32_t value, uint32_t* list,
                                            uint32_t* counter) {
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    if (!mask) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(counter, (uint32_t)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (pred) list[base + __popc(mask & ((1u << lane) - 1u))] = value;
}

__device__ __forceinline__ void warp_append64(bool pred, uint64_t value, uint64_t* list,
                                              uint32_t* counter) {
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    if (!mask) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(counter, (uint32_t)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (pred) list[base + __popc(mask & ((1u << lane) - 1u))] = value;
}

// Counter cells are exact to 128 bits: every u64 cell has a wrap counter
// `cstride` words after it, bumped whenever an add wraps the cell, so the host
// sees the true total and raises CounterOverflowError exactly when the
// reference's checked_increment would (types.hpp:65-70) -- including for
// cells formed by a difference of two raw sums (Star = raw - Pair).
__device__ __forceinline__ void cell_add(unsigned long long* cell, int cstride, uint64_t v) {
    if (!v) return;
    const unsigned long long old = atomicAdd(cell, (unsigned long long)v);
    if (old + v < old) atomicAdd(cell + cstride, 1ull);
}

// Count sinks: rare per-item contributions go straight to shared (per block)
// or global (per work item) u64 cells, so no kernel keeps a register array.
struct SmemSink {
    unsigned long long* cells;
    int cstride;  // wrap counter of cells[i] at cells[i + cstride]
    __device__ __forceinline__ void add(int i, uint64_t v) const { cell_add(&cells[i], cstride, v); }
};
using GlobalSink = SmemSink;

// Warp-held cells: lane L keeps the warp's running sum of cell L (up to 32
// cells).  A u64 shared-memory atomicAdd compiles to a CAS loop that
// serialises every lane of a warp adding to the same cell, so hot cells are
// summed across the warp with __reduce_add_sync (32-bit) instead.
//   add6(): six per-lane counts bound for cells ty * 8 + base + dk (c[ty * 2 +
//   dk], base in {0, 2, 4, 6}) -- the triangle kernels, whose long-window lanes
//   share the first edge; one reduction per value and distinct base present.
// A warp whose counts reach 2^27 (32 of them could wrap) takes the per-lane
// atomics instead.  `wraps` counts wraps of the lane's u64 (exactness).
struct WarpCells {
    uint64_t mine = 0;
    uint32_t wraps = 0;
    __device__ __forceinline__ void fold(uint64_t sum) {
        const uint64_t nm = mine + sum;
        wraps += nm < mine ? 1u : 0u;
        mine = nm;
    }
    __device__ __forceinline__ void add6(bool active, int base, const uint32_t c[6],
                                         unsigned long long* cells, int cstride) {
        uint32_t big = 0, nz = 0;
#pragma unroll
        for (int x = 0; x < 6; ++x) {
            const uint32_t v = active ? c[x] : 0u;
            big |= v >> 27;
            nz |= v;
        }
        if (__any_sync(0xffffffffu, big)) {
            if (active)
#pragma unroll
                for (int x = 0; x < 6; ++x) cell_add(&cells[(x >> 1) * 8 + base + (x & 1)], cstride, c[x]);
            return;
        }
        const uint32_t present = __reduce_or_sync(0xffffffffu, nz ? 1u << (base >> 1) : 0u);
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (!((present >> q) & 1u)) continue;  // warp-uniform
            const bool mine_q = active && base == 2 * q;
#pragma unroll
            for (int x = 0; x < 6; ++x) {
                const uint32_t sum = __reduce_add_sync(0xffffffffu, mine_q ? c[x] : 0u);
                if (lane == (x >> 1) * 8 + 2 * q + (x & 1)) fold(sum);
            }
        }
    }
    // each lane's cell into the block's shared cells (whole warp, before the block flush)
    __device__ __forceinline__ void flush(unsigned long long* cells, int ncells, int cstride) const {
        const int lane = threadIdx.x & 31;
        if (lane < ncells) {
            cell_add(&cells[lane], cstride, mine);
            if (wraps) atomicAdd(&cells[lane + cstride], (unsigned long long)wraps);
        }
    }
};

// zero `count` shared cells and their wrap counters (2 * count words); call
// before use, followed by __syncthreads
__device__ __forceinline__ void zero_cells(unsigned long long* cells, int count) {
    for (int i = threadIdx.x; i < 2 * count; i += blockDim.x) cells[i] = 0;
}
// add block cells (wrap counters at cells[i + count]) to global out (wrap
// counters at out[i + ostride]), after __syncthreads
__device__ __forceinline__ void flush_cells(const unsigned long long* cells, int count, uint64_t* out,
                                            int ostride) {
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        const unsigned long long v = cells[i];
        unsigned long long c = cells[i + count];
        if (v) {
            const unsigned long long old = atomicAdd((unsigned long long*)&out[i], v);
            if (old + v < old) ++c;
        }
        if (c) atomicAdd((unsigned long long*)&out[i + ostride], c);
    }
}

// last u with off[u] <= k (the node owning record k); off has n+1 entries
__device__ __forceinline__ uint32_t owner_of(const uint32_t* __restrict__ off, uint64_t n,
                                             uint32_t k) {
    uint64_t lo = 0, hi = n + 1;  // upper_bound(off, k) - 1
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (off[mid] <= k) lo = mid + 1; else hi = mid;
    }
    return (uint32_t)(lo - 1);
}

template <typename T>
struct ArrayLoad {
    const T* p;
    __device__ __forceinline__ T operator()(uint64_t i) const { return p[i]; }
};

// Chunked reduce-then-scan: G blocks each own one contiguous chunk; phase 1
// reduces it, phase 2 scans the G partials, phase 3 re-reads the chunk in
// 4096-element tiles (coalesced loads staged through shared memory) and writes
// the exclusive prefix with a running in-block carry.  No inter-block waiting.
constexpr int kScanBlock = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanBlock * kScanItems;  // 4096

template <typename T, typename Load>
__global__ void __launch_bounds__(kScanBlock) scan_chunk_reduce(Load load, uint64_t n, uint64_t chunk,
                                                                T* partials) {
    const uint64_t b0 = (uint64_t)blockIdx.x * chunk;
    const uint64_t b1 = b0 + chunk < n ? b0 + chunk : n;
    T acc = 0;
    for (uint64_t base = b0; base < b1; base += kScanTile) {
        T x[kScanItems];
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint64_t i = base + (uint64_t)k * kScanBlock + threadIdx.x;
            x[k] = i < b1 ? load(i) : T(0);
        }
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) acc += x[k];
    }
    acc = warp_sum(acc);
    __shared__ T ws[kScanBlock / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        T t = 0;
        for (int w = 0; w < kScanBlock / 32; ++w) t += ws[w];
        partials[blockIdx.x] = t;
    }
}

template <typename T>
struct ArrayStore {
    T* p;
    __device__ __forceinline__ void operator()(uint64_t i, T v) const { p[i] = v; }
};

template <typename T, typename Load, typename Store>
__global__ void __launch_bounds__(kScanBlock) scan_chunk_down(Load load, uint64_t n, uint64_t chunk,
                                                              const T* __restrict__ partials, Store out) {
    __shared__ T stage[kScanTile + kScanTile / 32];
    __shared__ T s_tot;
    const uint64_t b0 = (uint64_t)blockIdx.x * chunk;
    const uint64_t b1 = b0 + chunk < n ? b0 + chunk : n;
    // this chunk's offset: the sum of the chunk totals before it (<= 1024 of
    // them, reduced in-block instead of a separate scan launch)
    T carry = 0;
    {
        T p = 0;
        for (uint32_t c = threadIdx.x; c < blockIdx.x; c += kScanBlock) p += partials[c];
        p = warp_sum(p);
        __shared__ T ws[kScanBlock / 32];
        if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = p;
        __syncthreads();
#pragma unroll
        for (int w = 0; w < kScanBlock / 32; ++w) carry += ws[w];
    }
    for (uint64_t base = b0; base < b1; base += kScanTile) {
        {
            T x[kScanItems];
#pragma unroll
            for (int k = 0; k < kScanItems; ++k) {
                const uint64_t i = base + (uint64_t)k * kScanBlock + threadIdx.x;
                x[k] = i < b1 ? load(i) : T(0);
            }
#pragma unroll
            for (int k = 0; k < kScanItems; ++k) {
                const uint32_t j = k * kScanBlock + threadIdx.x;
                stage[j + (j >> 5)] = x[k];
            }
        }
        __syncthreads();
        T v[kScanItems];
        T ts = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint32_t j = threadIdx.x * kScanItems + k;
            v[k] = stage[j + (j >> 5)];
            ts += v[k];
        }
        T run = block_exclusive_scan<T, kScanBlock / 32>(ts, &s_tot) + carry;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint32_t j = threadIdx.x * kScanItems + k;
            stage[j + (j >> 5)] = run;
            run += v[k];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint64_t i = base + (uint64_t)k * kScanBlock + threadIdx.x;
            const uint32_t j = k * kScanBlock + threadIdx.x;
            if (i < b1) out(i, stage[j + (j >> 5)]);
        }
        carry += s_tot;
        __syncthreads();
    }
    if (b1 == n && b0 < b1 && threadIdx.x == 0) out(n, carry);
}

// out(i, exclusive prefix of load(0..i-1)) for i in [0, n]; out(n, .) = total.
template <typename T, typename Load, typename Store>
void exclusive_scan_to(Load load, uint64_t n, Store out, cudaStream_t s) {
    uint64_t g = (uint64_t)sm_count() * 4;
    if (g > 1024) g = 1024;
    uint64_t chunk = (n + g - 1) / g;
    chunk = (chunk + kScanTile - 1) / kScanTile * kScanTile;
    g = (n + chunk - 1) / chunk;
    T* partials = dalloc<T>(g, s);
    TM_LAUNCH("scan", s, (scan_chunk_reduce<T, Load>), (unsigned)g, kScanBlock, 0, load, n, chunk,
              partials);
    TM_LAUNCH("scan", s, (scan_chunk_down<T, Load, Store>), (unsigned)g, kScanBlock, 0, load, n, chunk,
              partials, out);
    dfree(partials, s);
}

// out[0..n] = exclusive prefix of load(0..n-1); out[n] = total.
template <typename T, typename Load>
void exclusive_scan(Load load, uint64_t n, T* out, cudaStream_t s) {
    if (n == 0) {
        TM_CUDA(cudaMemsetAsync(out, 0, sizeof(T), s));
        return;
    }
    exclusive_scan_to<T>(load, n, ArrayStore<T>{out}, s);
}

// digit passes for `bits` key bits, and the width of the next digit with
// `bits_left` bits over `passes_left` passes: the bits are spread evenly
// (20 bits: 7 + 7 + 6 rather than 8 + 8 + 4) -- fewer ballot rounds per
// ranking and longer digit runs per tile in the wide passes (sortbench:
// 20M node keys' downsweep -3 %, 200M keys of 26 bits -8 %)
#ifndef TM_RADIX_MAX_BITS
#define TM_RADIX_MAX_BITS 8  // digit bits per pass at most (9-bit digits measured slower: 512-row passes)
#endif
__host__ __device__ inline int radix_passes(int bits) { return (bits + TM_RADIX_MAX_BITS - 1) / TM_RADIX_MAX_BITS; }
__host__ __device__ inline int radix_digit_width(int bits_left, int passes_left) {
    return (bits_left + passes_left - 1) / passes_left;
}

// ---------------------------------------------------------------------------
// stable LSD radix sort of (key, u32 value) pairs, 8-bit digits, reduce-then-
// scan per pass: upsweep (per-tile digit counts) -> scan of the digit-major
// count matrix -> downsweep (rank the tile with per-warp __match_any_sync,
// keeping input order; reorder in shared memory; write each digit run as one
// burst).  All tile loads are issued before any ranking (ILP).
constexpr int kRadix = 1 << TM_RADIX_MAX_BITS;  // digit rows a count matrix / histogram may need

template <typename K, int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK) radix_upsweep(const K* __restrict__ keys, uint64_t n,
                                                       int shift, uint32_t dmask,
                                                       uint32_t* __restrict__ counts, uint32_t ntiles) {
    constexpr int NW = BLOCK / 32;
    constexpr int TILE = BLOCK * ITEMS;
    __shared__ uint32_t hist[NW][kRadix];
    for (int i = threadIdx.x; i < NW * kRadix; i += BLOCK) (&hist[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t base = (uint64_t)blockIdx.x * TILE + (uint64_t)w * (ITEMS * 32);
    K k[ITEMS];
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        const uint64_t i = base + r * 32 + lane;
        k[r] = i < n ? keys[i] : K(0);
    }
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        const uint64_t i = base + r * 32 + lane;
        if (i < n) atomicAdd(&hist[w][(uint32_t)(k[r] >> shift) & dmask], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d <= (int)dmask; d += BLOCK) {  // rows of this pass's digits only
        uint32_t s = 0;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) s += hist[ww][d];
        counts[(uint64_t)d * ntiles + blockIdx.x] = s;
    }
}

constexpr int kRowBlock = 512, kRowItems = 16, kRowChunk = kRowBlock * kRowItems;
// offs[d][t] = sum_{t' < t} counts[d][t'] (row-local), totals[d] = row sum;
// the downsweep adds the exclusive scan of totals.  One block per digit row,
// kRowChunk counts per step: loaded coalesced into
// shared memory, each thread scans its 16 contiguous counts, the block scans
// the thread sums, results go back through shared memory to coalesced stores.
static __global__ void __launch_bounds__(kRowBlock) radix_scan_counts(const uint32_t* __restrict__ counts,
                                                                      uint32_t ntiles,
                                                                      uint32_t* __restrict__ offs,
                                                                      uint32_t* __restrict__ totals) {
    const uint32_t d = blockIdx.x;
    __shared__ uint32_t s_row[kRowChunk + kRowChunk / 32];  // +1 word per 32: no bank conflicts
    __shared__ uint32_t s_tot;
    auto at = [](uint32_t i) { return i + (i >> 5); };
    uint32_t carry = 0;
    const uint32_t* row = counts + (uint64_t)d * ntiles;
    uint32_t* orow = offs + (uint64_t)d * ntiles;
    for (uint32_t base = 0; base < ntiles; base += kRowChunk) {
#pragma unroll
        for (int k = 0; k < kRowItems; ++k) {
            const uint32_t i = k * kRowBlock + threadIdx.x;
            s_row[at(i)] = base + i < ntiles ? __ldcs(row + base + i) : 0u;
        }
        __syncthreads();
        uint32_t v[kRowItems];
        uint32_t ts = 0;
#pragma unroll
        for (int k = 0; k < kRowItems; ++k) {
            v[k] = s_row[at(threadIdx.x * kRowItems + k)];
            ts += v[k];
        }
        uint32_t run = block_exclusive_scan<uint32_t, kRowBlock / 32>(ts, &s_tot) + carry;
#pragma unroll
        for (int k = 0; k < kRowItems; ++k) {
            s_row[at(threadIdx.x * kRowItems + k)] = run;
            run += v[k];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kRowItems; ++k) {
            const uint32_t i = k * kRowBlock + threadIdx.x;
            if (base + i < ntiles) orow[base + i] = s_row[at(i)];
        }
        carry += s_tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) totals[d] = carry;
}

// ---- TMA-pipelined persistent downsweep ----------------------------------
// Each block loops over tiles blockIdx.x, +gridDim.x, ...; one elected thread
// streams tile i+1 into the other shared-memory stage with cp.async.bulk
// (mbarrier completion) while the block ranks and scatters tile i.  Keys are
// re-read from shared memory instead of being held in registers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

// one digit bit of the ballot multi-split: the lanes whose bit equals ours
// (and-test with predicate out, vote, select, xor: four instructions)
__device__ __forceinline__ uint32_t wlms_bit(uint32_t d, uint32_t bit) {
    uint32_t r;
    asm("{\n\t.reg .pred p;\n\t.reg .b32 v, s, a;\n\t"
        "and.b32 a, %1, %2;\n\t"
        "setp.ne.u32 p, a, 0;\n\t"
        "vote.sync.ballot.b32 v, p, 0xffffffff;\n\t"
        "selp.b32 s, 0, -1, p;\n\t"
        "xor.b32 %0, v, s;\n\t}"
        : "=r"(r)
        : "r"(d), "r"(bit));
    return r;
}

#ifndef TM_RANK_MATCH_ROUNDS_NARROW
#define TM_RANK_MATCH_ROUNDS_NARROW 1  // the same for passes of <= 4 digit bits
#endif

// Last-pass output policy: NoEmit writes the sorted keys (and values); an
// emitter with kOn = true receives (sorted position, key, value) instead and
// writes its consumer's arrays directly -- the pass that would re-read the
// sorted keys + values only to split them into those arrays disappears.
struct NoEmit {
    static constexpr bool kOn = false;
    __device__ __forceinline__ void operator()(uint32_t, uint64_t, uint64_t) const {}
};

// First-pass input policy: NoLoad streams the key (and value) arrays; a loader
// with kOn = true fills a tile's stage from the producer's own data instead
// (issue: the TMA copies of tile `tile` into `stage`, completing on `bar`) and
// forms each element's (key, value) in registers (fetch) -- the pass that
// would write the keys + values only for this pass to read them disappears.
struct NoLoad {
    static constexpr bool kOn = false;
    __device__ __forceinline__ void issue(unsigned char*, uint32_t, uint64_t*) const {}
    __device__ __forceinline__ void fetch(const unsigned char*, uint32_t, uint32_t, uint64_t&, uint64_t&) const {}
};

// NBITS: digit bits of this pass (8, or 4 for a short last pass); digits are
// (key >> shift) & dmask with dmask < 2^NBITS
template <typename K, typename V, bool kVals, int BLOCK, int ITEMS, int MINB, int NBITS, typename Emit = NoEmit,
          typename Load = NoLoad>
__global__ void __launch_bounds__(BLOCK, MINB) radix_downsweep_tma(const K* __restrict__ kin,
                                                                   const V* __restrict__ vin,
                                                                   K* __restrict__ kout,
                                                                   V* __restrict__ vout, uint64_t n,
                                                                   int shift, uint32_t dmask,
                                                                   const uint32_t* __restrict__ tile_offsets,
                                                                   uint32_t ntiles,
                                                                   const uint32_t* __restrict__ totals,
                                                                   Emit emit, Load load) {
    constexpr int NW = BLOCK / 32, TILE = BLOCK * ITEMS;
    constexpr int kMatchRounds = NBITS >= 8 ? TM_RANK_MATCH_ROUNDS : TM_RANK_MATCH_ROUNDS_NARROW;
    constexpr int RADIX = 1 << NBITS;
    constexpr uint32_t kNone = RADIX;  // digit of a lane past the tile end
    constexpr int DPT = (RADIX + BLOCK - 1) / BLOCK;  // digits per thread (consecutive)
    constexpr uint32_t STAGE_BYTES = TILE * (sizeof(K) + (kVals ? sizeof(V) : 0));
    extern __shared__ __align__(128) unsigned char tma_smem[];
    // [stage0][stage1]: each TILE keys (+ TILE vals); a tile is reordered in
    // place in its own stage (its keys are in registers by then)
    auto stage_keys = [&](int s) { return reinterpret_cast<K*>(tma_smem + s * STAGE_BYTES); };
    auto stage_vals = [&](int s) {
        return reinterpret_cast<V*>(tma_smem + s * STAGE_BYTES + TILE * sizeof(K));
    };
    __shared__ __align__(16) uint16_t wcnt[NW][RADIX];  // per-warp digit counts, then (warp, digit) run starts
    __shared__ uint32_t dglob[RADIX];
    __shared__ __align__(8) uint64_t bar[2];

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](uint32_t tile, int s) {
        const uint64_t base = (uint64_t)tile * TILE;
        const uint64_t cnt = (n - base) < (uint64_t)TILE ? (n - base) : (uint64_t)TILE;
        const uint32_t kbytes = (uint32_t)((cnt * sizeof(K) + 15) & ~uint64_t(15));
        const uint32_t vbytes = kVals ? (uint32_t)((cnt * sizeof(V) + 15) & ~uint64_t(15)) : 0u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if constexpr (Load::kOn) {
            load.issue(tma_smem + s * STAGE_BYTES, tile, &bar[s]);
        } else {
            mbar_expect_tx(&bar[s], kbytes + vbytes);
            tma_load_1d(stage_keys(s), kin + base, kbytes, &bar[s]);
            if (kVals) tma_load_1d(stage_vals(s), vin + base, vbytes, &bar[s]);
        }
    };
    // count rows exist for this pass's digits only (<= dmask)
    // global base of each of this thread's digits (digits tid * DPT + k)
    uint32_t dbase[DPT];
    {
        uint32_t tot[DPT], tsum = 0;
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
            const int d = tid * DPT + k;
            tot[k] = d <= (int)dmask ? totals[d] : 0u;
            tsum += tot[k];
        }
        uint32_t run = block_exclusive_scan<uint32_t, NW>(tsum, nullptr);
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
            dbase[k] = run;
            run += tot[k];
        }
    }
    uint32_t tile = blockIdx.x;
    if (tid == 0 && tile < ntiles) issue(tile, 0);
    for (uint32_t it = 0; tile < ntiles; ++it, tile += gridDim.x) {
        const int s = it & 1;
        const uint32_t next = tile + gridDim.x;
        if (tid == 0 && next < ntiles) issue(next, s ^ 1);
        for (int i = tid; i < NW * RADIX / 8; i += BLOCK) reinterpret_cast<uint4*>(&wcnt[0][0])[i] = make_uint4(0, 0, 0, 0);
        const uint64_t tbase = (uint64_t)tile * TILE;
        const uint32_t tile_n = (uint32_t)((n - tbase) < (uint64_t)TILE ? (n - tbase) : (uint64_t)TILE);
        // the tile's digit offsets, loaded now and used after the ranking
        // (keeps the global-load latency off the critical path)
        uint32_t toff[DPT];
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
            const int d = tid * DPT + k;
            toff[k] = d <= (int)dmask ? __ldg(tile_offsets + (uint64_t)d * ntiles + tile) : 0u;
        }
        mbar_wait(&bar[s], (it >> 1) & 1);
        __syncthreads();
        K* sk = stage_keys(s);
        V* sv = stage_vals(s);
        // digits and match masks of all rounds first (independent, overlapped),
        // then the warp's sequential per-digit running counts
        K key[ITEMS];
        V val[kVals ? ITEMS : 1];
        uint32_t dig[ITEMS], rank[ITEMS];
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
            const uint32_t i = w * (ITEMS * 32) + r * 32 + lane;
            if constexpr (Load::kOn) {
                uint64_t lk = 0, lv = 0;
                load.fetch(tma_smem + s * STAGE_BYTES, tile, i, lk, lv);
                key[r] = (K)lk;
                if (kVals) val[r] = (V)lv;
            } else {
                key[r] = sk[i];
                if (kVals) val[r] = sv[i];
            }
            dig[r] = i < tile_n ? ((uint32_t)(key[r] >> shift) & dmask) : kNone;
        }
        // Peer masks (lanes holding the same digit).  match.any costs ~60 clocks
        // per warp-instruction per SM on 8-bit random digits (ADU pipe,
        // profiles/rankbench.cu); a ballot multi-split costs ~4 ALU
        // instructions per digit bit.  The first kMatchRounds rounds use
        // match.any and the rest ballots, so the two pipes share the ranking.
        const bool full_tile = tile_n == (uint32_t)TILE;
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
            if (r < kMatchRounds) {
                rank[r] = __match_any_sync(0xffffffffu, dig[r]);
            } else {
                uint32_t peers = full_tile ? 0xffffffffu : __ballot_sync(0xffffffffu, dig[r] < kNone);
                if (dig[r] >= kNone) peers = ~peers;
#pragma unroll
                for (int b = 0; b < NBITS; ++b) peers &= wlms_bit(dig[r], 1u << b);
                rank[r] = peers;
            }
        }
        // running per-warp digit counts, one load -> store step per round
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
            const bool valid = dig[r] < kNone;
            const unsigned peers = rank[r];
            const uint32_t prev = valid ? wcnt[w][dig[r]] : 0u;
            rank[r] = prev + __popc(peers & lt);
            __syncwarp();
            if (valid && (peers & lt) == 0) wcnt[w][dig[r]] = (uint16_t)(prev + __popc(peers));
            __syncwarp();
        }
        __syncthreads();
        uint32_t cnt[DPT], csum = 0;
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
            const int d = tid * DPT + k;
            cnt[k] = 0;
            if (d < RADIX) {
#pragma unroll
                for (int ww = 0; ww < NW; ++ww) cnt[k] += wcnt[ww][d];
            }
            csum += cnt[k];
        }
        uint32_t ex = block_exclusive_scan<uint32_t, NW>(csum, nullptr);
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
            const int d = tid * DPT + k;
            if (d < RADIX) {
                // tile position of each (warp, digit) run; global minus tile start per digit
                uint32_t run = ex;
#pragma unroll
                for (int ww = 0; ww < NW; ++ww) {
                    const uint32_t c = wcnt[ww][d];
                    wcnt[ww][d] = (uint16_t)run;
                    run += c;
                }
                dglob[d] = toff[k] + dbase[k] - ex;
            }
            ex += cnt[k];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
            if (dig[r] < kNone) {
                const uint32_t q = wcnt[w][dig[r]] + rank[r];
                sk[q] = key[r];
                if (kVals) sv[q] = val[r];
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
            const uint32_t i = r * BLOCK + tid;
            if (i < tile_n) {
                const K k = sk[i];
                const uint32_t dest = dglob[(uint32_t)(k >> shift) & dmask] + i;
                if constexpr (Emit::kOn) {
                    emit(dest, (uint64_t)k, kVals ? (uint64_t)sv[i] : 0ull);
                } else {
                    kout[dest] = k;
                    if (kVals) vout[dest] = sv[i];
                }
            }
        }
        __syncthreads();
    }
}

constexpr uint64_t kSortPad = 4;
// sort tile: kSortBlock threads x kSortItems keys (a producer that counts the
// first digit itself must use the same tiles: digit-major counts[d][tile])
constexpr int kSortBlock = 256, kSortItems = 12, kSortMinBlocks = 3, kSortTile = kSortBlock * kSortItems;

// one downsweep instantiation: sets its shared-memory limit and caches its
// occupancy on first use, then launches a persistent grid
template <typename K, typename V, bool kVals, int BLOCK, int ITEMS, int MINB, int NBITS, typename Emit = NoEmit,
          typename Load = NoLoad>
void launch_downsweep(const K* kin, const V* vin, K* kout, V* vout, uint64_t n, int shift,
                      uint32_t dmask, const uint32_t* offs, uint32_t ntiles, const uint32_t* totals,
                      cudaStream_t s, Emit emit = Emit(), Load load = Load()) {
    constexpr int TILE = BLOCK * ITEMS;
    constexpr size_t smem = 2 * TILE * (sizeof(K) + (kVals ? sizeof(V) : 0));
    auto kern = radix_downsweep_tma<K, V, kVals, BLOCK, ITEMS, MINB, NBITS, Emit, Load>;
    static int per_sm = 0;  // resident blocks per SM
    if (per_sm == 0) {
        TM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        TM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BLOCK, smem));
        if (per_sm < 1) per_sm = 1;
    }
    const unsigned pgrid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)sm_count() * per_sm);
    TM_LAUNCH("radix_downsweep", s, kern, pgrid, BLOCK, smem, kin, vin, kout, vout, n, shift, dmask, offs,
              ntiles, totals, emit, load);
}

// one pass configuration: tile = BLOCK * ITEMS keys
template <typename K, typename V, int BLOCK, int ITEMS, int MINB, typename Emit = NoEmit, typename Load = NoLoad>
void radix_sort_cfg(K*& keys, V*& vals, K*& keys_alt, V*& vals_alt, uint64_t n,
                    int bit_lo, int bit_hi, cudaStream_t s, const uint32_t* first_counts, Emit emit = Emit(),
                    Load load = Load()) {
    constexpr int TILE = BLOCK * ITEMS;
    const bool with_vals = vals != nullptr;
    const int passes = radix_passes(bit_hi - bit_lo);
    const uint32_t ntiles = (uint32_t)((n + TILE - 1) / TILE);
    const uint64_t ncount = (uint64_t)kRadix * ntiles;
    uint32_t* counts = dalloc<uint32_t>(2 * ncount + (uint64_t)kRadix * passes, s);
    uint32_t* offs = counts + ncount;
    uint32_t* totals = offs + ncount;  // kRadix digit totals (per pass, reused)
    // the key bits spread evenly over ceil(bits / 8) passes (a producer that
    // counts the first digit itself uses the same width: radix_digit_width)
    int shift = bit_lo;
    for (int p = 0; p < passes; ++p) {
        const int width = radix_digit_width(bit_hi - shift, passes - p);
        const uint32_t dmask = (1u << width) - 1u;
        const uint32_t* cin = counts;
        if (p == 0 && first_counts) {
            cin = first_counts;  // the producer of the keys already counted pass 0
        } else {
            TM_LAUNCH("radix_upsweep", s, (radix_upsweep<K, BLOCK, ITEMS>), ntiles, BLOCK, 0, keys, n, shift,
                      dmask, counts, ntiles);
        }
        TM_LAUNCH("radix_scan", s, radix_scan_counts, dmask + 1, kRowBlock, 0, cin, ntiles,
                  offs, totals);
        V* vin = with_vals ? vals : nullptr;
        V* vout = with_vals ? vals_alt : nullptr;
// (u64 keys + u64 payloads: 96 KB of tile stages per block, so 2 resident
// blocks per SM and the register budget of 2)
#define TM_DOWNSWEEP_AS(HV, NB, E, L, ev, lv)                                                                   \
    launch_downsweep<K, V, HV, BLOCK, ITEMS, (HV && sizeof(K) + sizeof(V) >= 16) ? 2 : MINB, NB, E, L>(         \
        keys, vin, keys_alt, vout, n, shift, dmask, offs, ntiles, totals, s, ev, lv)
#define TM_DOWNSWEEP(HV, NB)                                                                                    \
    do {                                                                                                        \
        const bool el = Emit::kOn && p == passes - 1, lf = Load::kOn && p == 0;                                 \
        if (el && lf) TM_DOWNSWEEP_AS(HV, NB, Emit, Load, emit, load);                                          \
        else if (el) TM_DOWNSWEEP_AS(HV, NB, Emit, NoLoad, emit, NoLoad());                                     \
        else if (lf) TM_DOWNSWEEP_AS(HV, NB, NoEmit, Load, NoEmit(), load);                                     \
        else TM_DOWNSWEEP_AS(HV, NB, NoEmit, NoLoad, NoEmit(), NoLoad());                                       \
    } while (0)
        if (with_vals) {
            if (width <= 4) TM_DOWNSWEEP(true, 4);
            else if (width <= 6) TM_DOWNSWEEP(true, 6);
            else if (width <= 7) TM_DOWNSWEEP(true, 7);
            else if (width <= 8) TM_DOWNSWEEP(true, 8);
            else TM_DOWNSWEEP(true, 9);
            V* tv = vals;
            vals = vals_alt;
            vals_alt = tv;
        } else {
            if (Emit::kOn || Load::kOn) throw tm_error(1, "radix_sort: emitters and loaders sort key + value");
            if (width <= 4) TM_DOWNSWEEP_AS(false, 4, NoEmit, NoLoad, NoEmit(), NoLoad());
            else if (width <= 6) TM_DOWNSWEEP_AS(false, 6, NoEmit, NoLoad, NoEmit(), NoLoad());
            else if (width <= 7) TM_DOWNSWEEP_AS(false, 7, NoEmit, NoLoad, NoEmit(), NoLoad());
            else if (width <= 8) TM_DOWNSWEEP_AS(false, 8, NoEmit, NoLoad, NoEmit(), NoLoad());
            else TM_DOWNSWEEP_AS(false, 9, NoEmit, NoLoad, NoEmit(), NoLoad());
        }
#undef TM_DOWNSWEEP
#undef TM_DOWNSWEEP_AS
        shift += width;
        K* tk = keys;
        keys = keys_alt;
        keys_alt = tk;
    }
    dfree(counts, s);
}

// Stable sort of keys (and u32 or u64 values when vals != nullptr) on key bits
// [bit_lo, bit_hi).  Buffers need kSortPad elements of slack (TMA tile loads
// round up to 16 bytes).  On return keys/vals point at the sorted data; the *_alt
// pointers at the scratch halves (pointers may be swapped).
// (no pass runs for n <= 1 or an empty bit range: the input order is the output)
template <typename K, typename V, typename Emit>
__global__ void emit_in_order_kernel(const K* __restrict__ keys, const V* __restrict__ vals, uint64_t n, Emit emit) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        emit((uint32_t)i, (uint64_t)keys[i], vals ? (uint64_t)vals[i] : 0ull);
}

// With an emitter the last pass hands every (position, key, value) to it
// instead of writing the sorted arrays (which are then scratch).
// With a loader the first pass reads its tiles through it (keys / vals are
// scratch from the start; n > 1 and a non-empty bit range are the caller's to
// ensure).
template <typename K, typename V = uint32_t, typename Emit = NoEmit, typename Load = NoLoad>
void radix_sort(K*& keys, V*& vals, K*& keys_alt, V*& vals_alt, uint64_t n,
                int bit_lo, int bit_hi, cudaStream_t s, const uint32_t* first_counts = nullptr, Emit emit = Emit(),
                Load load = Load()) {
    if (n <= 1 || bit_hi <= bit_lo) {
        if constexpr (Emit::kOn) {
            if (n) {
                const K* kc = keys;
                const V* vc = vals;
                TM_LAUNCH("radix_downsweep", s, (emit_in_order_kernel<K, V, Emit>),
                          (unsigned)std::min<uint64_t>((n + 255) / 256, 1024), 256, 0, kc, vc, n, emit);
            }
        }
        return;
    }
    // 256 threads x 12 keys, 3 blocks per SM: the same downsweep time as 8
    // keys x 4 blocks with a third fewer tiles, so the count matrix's upsweep
    // and row scan shrink (profiles/sortbench.cu sweeps 256/512 threads x
    // 4-16 keys on B200: 20M node keys 0.457 -> 0.448 ms)
    radix_sort_cfg<K, V, kSortBlock, kSortItems, kSortMinBlocks, Emit, Load>(keys, vals, keys_alt, vals_alt, n, bit_lo,
                                                                             bit_hi, s, first_counts, emit, load);
}

inline int bit_width_u64(uint64_t x) {
    int b = 0;
    while (x) {
        ++b;
        x >>= 1;
    }
    return b;
}

}  // namespace tmb
