// tm_primitives.cuh -- own-written device-wide scan and stable LSD radix sort.
//
// The radix sort orders the incident records by (node, t, ordinal) exactly as
// the reference's std::sort with the (t, ordinal) comparator followed by the
// CSR fill does (graph.cpp:37-41, indexes.cpp:7-26): keys are stable-sorted,
// and records enter the sort in (t, ordinal) order, so ties keep input order.
//
// Both primitives are single-pass over HBM per digit / per scan:
//  * scan: one kernel, tiles claim ids from an atomic counter and chain their
//    prefixes with decoupled look-back (aggregate / inclusive status words);
//  * sort ("onesweep"): one histogram kernel reads the keys once for all digit
//    passes; each pass is then one kernel that ranks its 4096-key tile with
//    per-warp __match_any_sync (stable), publishes per-digit tile counts,
//    looks back across earlier tiles per digit, reorders the tile in shared
//    memory and writes each digit run as one burst.
#pragma once

#include <cstdlib>

#include "tm_internal.cuh"

namespace tmb {

// ---------------------------------------------------------------------------
// decoupled look-back status words: 2-bit flag | 62-bit value
constexpr uint64_t kStAgg = 1ull << 62;
constexpr uint64_t kStInc = 2ull << 62;
constexpr uint64_t kStVal = (1ull << 62) - 1;

__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

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

// warp-cooperative look-back: sum of predecessors of `tile` in status[idx(p)]
template <typename Idx>
__device__ __forceinline__ uint64_t warp_lookback(const uint64_t* status, int64_t tile, Idx idx) {
    const int lane = threadIdx.x & 31;
    uint64_t acc = 0;
    int64_t p = tile - 1;
    while (p >= 0) {
        const int64_t q = p - lane;
        uint64_t s = kStInc;  // lanes past tile 0 behave as zero-valued inclusive
        if (q >= 0) {
            do {
                s = ld_status(status + idx(q));
            } while ((s >> 62) == 0);
        }
        const unsigned inc_mask = __ballot_sync(0xffffffffu, (s >> 62) == 2);
        const int first = inc_mask ? __ffs(inc_mask) - 1 : 32;
        uint64_t v = (lane <= first && q >= 0) ? (s & kStVal) : 0;
        acc += warp_sum(v);
        if (inc_mask) break;
        p -= 32;
    }
    return acc;
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
__global__ void __launch_bounds__(1024) scan_partials(T* partials, uint32_t g) {
    // g <= 1024: one element per thread, exclusive in place, total at [g]
    T v = threadIdx.x < g ? partials[threadIdx.x] : T(0);
    __shared__ T total;
    T ex = block_exclusive_scan<T, 32>(v, &total);
    if (threadIdx.x < g) partials[threadIdx.x] = ex;
    if (threadIdx.x == 0) partials[g] = total;
}

template <typename T, typename Load>
__global__ void __launch_bounds__(kScanBlock) scan_chunk_down(Load load, uint64_t n, uint64_t chunk,
                                                              const T* __restrict__ partials, T* out) {
    __shared__ T stage[kScanTile + kScanTile / 32];
    __shared__ T s_tot;
    const uint64_t b0 = (uint64_t)blockIdx.x * chunk;
    const uint64_t b1 = b0 + chunk < n ? b0 + chunk : n;
    T carry = partials[blockIdx.x];
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
            if (i < b1) out[i] = stage[j + (j >> 5)];
        }
        carry += s_tot;
        __syncthreads();
    }
    if (b1 == n && b0 < b1 && threadIdx.x == 0) out[n] = carry;
}

// out[0..n] = exclusive prefix of load(0..n-1); out[n] = total.
template <typename T, typename Load>
void exclusive_scan(Load load, uint64_t n, T* out, cudaStream_t s) {
    if (n == 0) {
        TM_CUDA(cudaMemsetAsync(out, 0, sizeof(T), s));
        return;
    }
    uint64_t g = (uint64_t)sm_count() * 4;
    if (g > 1024) g = 1024;
    uint64_t chunk = (n + g - 1) / g;
    chunk = (chunk + kScanTile - 1) / kScanTile * kScanTile;
    g = (n + chunk - 1) / chunk;
    T* partials = dalloc<T>(g + 1, s);
    TM_LAUNCH("scan", s, (scan_chunk_reduce<T, Load>), (unsigned)g, kScanBlock, 0, load, n, chunk,
              partials);
    TM_LAUNCH("scan", s, scan_partials<T>, 1, 1024, 0, partials, (uint32_t)g);
    TM_LAUNCH("scan", s, (scan_chunk_down<T, Load>), (unsigned)g, kScanBlock, 0, load, n, chunk,
              partials, out);
    dfree(partials, s);
}

// ---------------------------------------------------------------------------
// onesweep stable LSD radix sort of (key, u32 value) pairs, 8-bit digits
constexpr int kOsBlock = 512;
constexpr int kOsWarps = kOsBlock / 32;
constexpr int kOsItems = 8;
constexpr int kOsTile = kOsBlock * kOsItems;  // 4096
constexpr int kRadix = 256;
constexpr int kMaxPasses = 8;

template <typename K>
__global__ void __launch_bounds__(256) onesweep_hist(const K* __restrict__ keys, uint64_t n,
                                                     int passes, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kMaxPasses][kRadix];
    for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n;
         base += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = base + threadIdx.x;
        const bool valid = i < n;
        const K k = valid ? keys[i] : K(0);
        for (int p = 0; p < passes; ++p) {
            const uint32_t d = valid ? ((uint32_t)(k >> (8 * p)) & 255u) : 256u;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (valid && (peers & lt) == 0) atomicAdd(&h[p][d], (uint32_t)__popc(peers));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
        const uint32_t c = (&h[0][0])[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

// classic upsweep: per-tile digit counts, counts[d * ntiles + tile]
template <typename K>
__global__ void __launch_bounds__(kOsBlock) radix_upsweep(const K* __restrict__ keys, uint64_t n,
                                                          int shift, uint32_t* __restrict__ counts,
                                                          uint32_t ntiles) {
    __shared__ uint32_t hist[kOsWarps][kRadix];
    for (int i = threadIdx.x; i < kOsWarps * kRadix; i += kOsBlock) (&hist[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t base = (uint64_t)blockIdx.x * kOsTile + (uint64_t)w * (kOsItems * 32);
    K k[kOsItems];
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
        const uint64_t i = base + r * 32 + lane;
        k[r] = i < n ? keys[i] : K(0);
    }
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
        const uint64_t i = base + r * 32 + lane;
        if (i < n) atomicAdd(&hist[w][(uint32_t)(k[r] >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < kRadix) {
        uint32_t s = 0;
#pragma unroll
        for (int ww = 0; ww < kOsWarps; ++ww) s += hist[ww][threadIdx.x];
        counts[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = s;
    }
}

// per pass: exclusive scan of the 256 digit counts (one block per pass)
static __global__ void __launch_bounds__(256) onesweep_digit_base(uint32_t* hist) {
    uint32_t* h = hist + blockIdx.x * kRadix;
    const uint32_t v = h[threadIdx.x];
    const uint32_t ex = block_exclusive_scan<uint32_t, 8>(v, nullptr);
    h[threadIdx.x] = ex;
}

template <typename K, bool kClassic>
__global__ void __launch_bounds__(kOsBlock) onesweep_pass(const K* __restrict__ kin,
                                                          const uint32_t* __restrict__ vin,
                                                          K* __restrict__ kout,
                                                          uint32_t* __restrict__ vout, uint64_t n,
                                                          int shift,
                                                          const uint32_t* __restrict__ digit_base,
                                                          uint64_t* status, uint32_t* tile_ctr,
                                                          const uint32_t* __restrict__ tile_offsets,
                                                          uint32_t ntiles) {
    extern __shared__ __align__(16) unsigned char os_smem[];
    K* skeys = reinterpret_cast<K*>(os_smem);
    uint32_t* svals = reinterpret_cast<uint32_t*>(skeys + kOsTile);
    __shared__ uint32_t wcnt[kOsWarps][kRadix];
    __shared__ uint32_t dstart[kRadix];
    __shared__ uint32_t dglob[kRadix];
    __shared__ uint32_t s_tile;

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) s_tile = kClassic ? blockIdx.x : atomicAdd(tile_ctr, 1u);
    for (int i = tid; i < kOsWarps * kRadix; i += kOsBlock) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t tbase = (uint64_t)tile * kOsTile;
    const unsigned lt = (1u << lane) - 1u;

    K key[kOsItems];
    uint32_t val[kOsItems];
    uint32_t rank[kOsItems];
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
        const uint64_t i = tbase + (uint64_t)w * (kOsItems * 32) + r * 32 + lane;
        const bool valid = i < n;
        key[r] = valid ? kin[i] : K(0);
        val[r] = valid ? vin[i] : 0u;
    }
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
        const uint64_t i = tbase + (uint64_t)w * (kOsItems * 32) + r * 32 + lane;
        const bool valid = i < n;
        const uint32_t d = valid ? ((uint32_t)(key[r] >> shift) & 255u) : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t prev = valid ? wcnt[w][d] : 0u;
        rank[r] = prev + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0) wcnt[w][d] = prev + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    uint32_t cnt = 0;
    if (tid < kRadix) {
        uint32_t run = 0;
#pragma unroll
        for (int ww = 0; ww < kOsWarps; ++ww) {
            const uint32_t c = wcnt[ww][tid];
            wcnt[ww][tid] = run;
            run += c;
        }
        cnt = run;
        if (!kClassic)
            st_status(status + (uint64_t)tile * kRadix + tid, (tile == 0 ? kStInc : kStAgg) | cnt);
    }
    const uint32_t ex = block_exclusive_scan<uint32_t, kOsWarps>(cnt, nullptr);
    if (tid < kRadix && kClassic) {
        dstart[tid] = ex;
        dglob[tid] = tile_offsets[(uint64_t)tid * ntiles + tile];
    } else if (tid < kRadix) {
        dstart[tid] = ex;
        uint64_t pre = 0;
        if (tile) {
            // serial look-back per digit (the predecessor is usually already inclusive)
            int64_t p = (int64_t)tile - 1;
            bool done = false;
            while (!done) {
                uint64_t sv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    sv[j] = (p - j >= 0) ? ld_status(status + (uint64_t)(p - j) * kRadix + tid) : kStInc;
#pragma unroll
                for (int j = 0; j < 4 && !done; ++j) {
                    uint64_t s = sv[j];
                    while ((s >> 62) == 0) s = ld_status(status + (uint64_t)(p - j) * kRadix + tid);
                    pre += (p - j >= 0) ? (s & kStVal) : 0;
                    if ((s >> 62) == 2) done = true;
                }
                p -= 4;
            }
            st_status(status + (uint64_t)tile * kRadix + tid, kStInc | (pre + cnt));
        }
        dglob[tid] = digit_base[tid] + (uint32_t)pre;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
        const uint64_t i = tbase + (uint64_t)w * (kOsItems * 32) + r * 32 + lane;
        if (i < n) {
            const uint32_t d = (uint32_t)(key[r] >> shift) & 255u;
            const uint32_t q = dstart[d] + wcnt[w][d] + rank[r];
            skeys[q] = key[r];
            svals[q] = val[r];
        }
    }
    __syncthreads();
    const uint32_t tile_n = (uint32_t)((n - tbase) < (uint64_t)kOsTile ? (n - tbase) : (uint64_t)kOsTile);
    for (uint32_t i = tid; i < tile_n; i += kOsBlock) {
        const K k = skeys[i];
        const uint32_t d = (uint32_t)(k >> shift) & 255u;
        const uint32_t dest = dglob[d] + (i - dstart[d]);
        kout[dest] = k;
        vout[dest] = svals[i];
    }
}

// Sorts (keys, vals) on key bits [0, bits).  On return keys/vals point at the
// sorted data; *_alt point at the scratch halves (pointers may be swapped).
inline bool classic_sort() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TM_SORT");
        v = (e && e[0] == 'o') ? 0 : 1;  // default: classic reduce-then-scan
    }
    return v == 1;
}

template <typename K>
void radix_sort_pairs(K*& keys, uint32_t*& vals, K*& keys_alt, uint32_t*& vals_alt, uint64_t n,
                      int bits, cudaStream_t s) {
    if (n <= 1 || bits <= 0) return;
    const int passes = (bits + 7) / 8;
    const uint32_t ntiles = (uint32_t)((n + kOsTile - 1) / kOsTile);
    const size_t smem = kOsTile * (sizeof(K) + sizeof(uint32_t));
    static bool attr_set = false;
    if (!attr_set) {
        TM_CUDA(cudaFuncSetAttribute(onesweep_pass<K, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        TM_CUDA(cudaFuncSetAttribute(onesweep_pass<K, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set = true;
    }
    auto swap_bufs = [&] {
        K* tk = keys;
        keys = keys_alt;
        keys_alt = tk;
        uint32_t* tv = vals;
        vals = vals_alt;
        vals_alt = tv;
    };
    if (classic_sort()) {
        const uint64_t ncount = (uint64_t)kRadix * ntiles;
        uint32_t* counts = dalloc<uint32_t>(2 * ncount + 1, s);
        uint32_t* offs = counts + ncount;
        for (int p = 0; p < passes; ++p) {
            TM_LAUNCH("radix_upsweep", s, radix_upsweep<K>, ntiles, kOsBlock, 0, keys, n, 8 * p,
                      counts, ntiles);
            exclusive_scan<uint32_t>(ArrayLoad<uint32_t>{counts}, ncount, offs, s);
            TM_LAUNCH("radix_downsweep", s, (onesweep_pass<K, true>), ntiles, kOsBlock, smem, keys,
                      vals, keys_alt, vals_alt, n, 8 * p, nullptr, nullptr, nullptr, offs, ntiles);
            swap_bufs();
        }
        dfree(counts, s);
        return;
    }
    const uint64_t nstatus = (uint64_t)passes * ntiles * kRadix;
    // [hist passes*256 u32][tile counters passes u32] [status u64 ...]
    const size_t hist_bytes = ((size_t)passes * kRadix + kMaxPasses) * sizeof(uint32_t);
    const size_t bytes = hist_bytes + nstatus * sizeof(uint64_t) + 16;
    unsigned char* scratch = dalloc<unsigned char>(bytes, s);
    TM_CUDA(cudaMemsetAsync(scratch, 0, bytes, s));
    uint32_t* hist = reinterpret_cast<uint32_t*>(scratch);
    uint32_t* ctr = hist + (size_t)passes * kRadix;
    uint64_t* status = reinterpret_cast<uint64_t*>(scratch + ((hist_bytes + 15) & ~size_t(15)));
    uint64_t hist_grid = (n + 255) / 256;
    const uint64_t cap = (uint64_t)sm_count() * 8;
    if (hist_grid > cap) hist_grid = cap;
    TM_LAUNCH("onesweep_hist", s, onesweep_hist<K>, (unsigned)hist_grid, 256, 0, keys, n, passes,
              hist);
    TM_LAUNCH("onesweep_base", s, onesweep_digit_base, (unsigned)passes, 256, 0, hist);
    for (int p = 0; p < passes; ++p) {
        TM_LAUNCH("onesweep_pass", s, (onesweep_pass<K, false>), ntiles, kOsBlock, smem, keys, vals,
                  keys_alt, vals_alt, n, 8 * p, hist + (size_t)p * kRadix,
                  status + (uint64_t)p * ntiles * kRadix, ctr + p, nullptr, ntiles);
        swap_bufs();
    }
    dfree(scratch, s);
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
