// tm_primitives.cuh -- own-written device-wide scan and stable LSD radix sort.
//
// The radix sort orders the incident records by (node, t, ordinal) exactly as
// the reference's std::sort with the (t, ordinal) comparator followed by the
// CSR fill does (graph.cpp:37-41, indexes.cpp:7-26): keys are stable-sorted,
// and records enter the sort in (t, ordinal) order, so ties keep input order.
//
// Scan: reduce-then-scan, 2048 items per 256-thread tile.
// Sort: 8-bit digits, 4096 keys per 256-thread tile; per-warp match_any
// ranking keeps stability; the tile is reordered in shared memory before the
// scatter so that each digit run leaves as one coalesced burst.
#pragma once

#include "tm_internal.cuh"

namespace tmb {

constexpr int kScanBlock = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanBlock * kScanItems;

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

// exclusive scan across a 256-thread block; returns this thread's prefix and
// writes the block total to *total (if non-null).
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* total) {
    __shared__ T warp_tot[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T inc = warp_inclusive_scan(v);
    if (lane == 31) warp_tot[w] = inc;
    __syncthreads();
    if (w == 0) {
        T x = lane < 8 ? warp_tot[lane] : T(0);
        T xi = warp_inclusive_scan(x);
        if (lane < 8) warp_tot[lane] = xi - x;
        if (lane == 7 && total) *total = xi;
    }
    __syncthreads();
    T r = warp_tot[w] + inc - v;
    __syncthreads();
    return r;
}

template <typename T>
struct ArrayLoad {
    const T* p;
    __device__ __forceinline__ T operator()(uint64_t i) const { return p[i]; }
};

template <typename T, typename Load>
__global__ void __launch_bounds__(kScanBlock) scan_reduce_kernel(Load load, uint64_t n, T* sums) {
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    T s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        uint64_t i = base + (uint64_t)k * kScanBlock + threadIdx.x;
        if (i < n) s += load(i);
    }
    s = warp_sum(s);
    __shared__ T ws[8];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        T t = 0;
        for (int w = 0; w < 8; ++w) t += ws[w];
        sums[blockIdx.x] = t;
    }
}

template <typename T, typename Load>
__global__ void __launch_bounds__(kScanBlock) scan_down_kernel(Load load, uint64_t n,
                                                              const T* tile_off, T* out) {
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    T v[kScanItems];
    T ts = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        uint64_t i = base + k;
        v[k] = i < n ? load(i) : T(0);
        ts += v[k];
    }
    T run = block_exclusive_scan<T>(ts, nullptr) + tile_off[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        uint64_t i = base + k;
        if (i < n) out[i] = run;
        run += v[k];
    }
    if (base <= n - 1 && n - 1 < base + kScanItems) out[n] = run;
}

template <typename T>
__global__ void zero_one_kernel(T* p) { *p = T(0); }

// out[0..n] = exclusive prefix of load(0..n-1); out[n] = total.
template <typename T, typename Load>
void exclusive_scan(Load load, uint64_t n, T* out, cudaStream_t s) {
    if (n == 0) {
        TM_CUDA(cudaMemsetAsync(out, 0, sizeof(T), s));
        return;
    }
    const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
    T* tile_off = dalloc<T>(tiles + 1, s);
    if (tiles == 1) {
        TM_CUDA(cudaMemsetAsync(tile_off, 0, sizeof(T), s));
    } else {
        T* sums = dalloc<T>(tiles, s);
        TM_LAUNCH("scan_reduce", s, (scan_reduce_kernel<T, Load>), (unsigned)tiles, kScanBlock, 0,
                  load, n, sums);
        exclusive_scan<T>(ArrayLoad<T>{sums}, tiles, tile_off, s);
        dfree(sums, s);
    }
    TM_LAUNCH("scan_down", s, (scan_down_kernel<T, Load>), (unsigned)tiles, kScanBlock, 0, load, n,
              tile_off, out);
    dfree(tile_off, s);
}

// ---------------------------------------------------------------------------
// stable LSD radix sort of (key, u32 value) pairs
constexpr int kRsBlock = 256;
constexpr int kRsWarps = kRsBlock / 32;
constexpr int kRsItems = 16;
constexpr int kRsTile = kRsBlock * kRsItems;  // 4096
constexpr int kRsRadix = 256;

template <typename K>
__global__ void __launch_bounds__(kRsBlock) radix_upsweep(const K* __restrict__ keys, uint64_t n,
                                                          int shift, uint32_t* __restrict__ counts,
                                                          uint32_t ntiles) {
    __shared__ uint32_t hist[kRsWarps][kRsRadix];
    for (int i = threadIdx.x; i < kRsWarps * kRsRadix; i += kRsBlock) (&hist[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t base = (uint64_t)blockIdx.x * kRsTile + (uint64_t)w * (kRsItems * 32);
#pragma unroll 4
    for (int r = 0; r < kRsItems; ++r) {
        uint64_t i = base + r * 32 + lane;
        if (i < n) atomicAdd(&hist[w][(uint32_t)(keys[i] >> shift) & 255u], 1u);
    }
    __syncthreads();
    const int d = threadIdx.x;
    uint32_t s = 0;
#pragma unroll
    for (int ww = 0; ww < kRsWarps; ++ww) s += hist[ww][d];
    counts[(uint64_t)d * ntiles + blockIdx.x] = s;
}

template <typename K>
__global__ void __launch_bounds__(kRsBlock) radix_downsweep(const K* __restrict__ kin,
                                                            const uint32_t* __restrict__ vin,
                                                            K* __restrict__ kout,
                                                            uint32_t* __restrict__ vout, uint64_t n,
                                                            int shift,
                                                            const uint32_t* __restrict__ offsets,
                                                            uint32_t ntiles) {
    extern __shared__ __align__(16) unsigned char rs_smem[];
    K* skeys = reinterpret_cast<K*>(rs_smem);
    uint32_t* svals = reinterpret_cast<uint32_t*>(skeys + kRsTile);
    __shared__ uint32_t wcnt[kRsWarps][kRsRadix];
    __shared__ uint32_t dstart[kRsRadix];
    __shared__ uint32_t dbase[kRsRadix];

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int i = tid; i < kRsWarps * kRsRadix; i += kRsBlock) (&wcnt[0][0])[i] = 0;
    __syncthreads();

    const uint64_t tbase = (uint64_t)blockIdx.x * kRsTile;
    const unsigned lt = (1u << lane) - 1u;
    K key[kRsItems];
    uint32_t val[kRsItems];
    uint32_t rank[kRsItems];
#pragma unroll
    for (int r = 0; r < kRsItems; ++r) {
        const uint64_t i = tbase + (uint64_t)w * (kRsItems * 32) + r * 32 + lane;
        const bool valid = i < n;
        key[r] = valid ? kin[i] : K(0);
        val[r] = valid ? vin[i] : 0u;
        const uint32_t d = valid ? ((uint32_t)(key[r] >> shift) & 255u) : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t prev = valid ? wcnt[w][d] : 0u;
        rank[r] = prev + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0) wcnt[w][d] = prev + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {
        const int d = tid;
        uint32_t run = 0;
#pragma unroll
        for (int ww = 0; ww < kRsWarps; ++ww) {
            uint32_t c = wcnt[ww][d];
            wcnt[ww][d] = run;
            run += c;
        }
        const uint32_t ex = block_exclusive_scan<uint32_t>(run, nullptr);
        dstart[d] = ex;
        dbase[d] = offsets[(uint64_t)d * ntiles + blockIdx.x];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRsItems; ++r) {
        const uint64_t i = tbase + (uint64_t)w * (kRsItems * 32) + r * 32 + lane;
        if (i < n) {
            const uint32_t d = (uint32_t)(key[r] >> shift) & 255u;
            const uint32_t q = dstart[d] + wcnt[w][d] + rank[r];
            skeys[q] = key[r];
            svals[q] = val[r];
        }
    }
    __syncthreads();
    const uint32_t tile_n = (uint32_t)((n - tbase) < (uint64_t)kRsTile ? (n - tbase) : (uint64_t)kRsTile);
    for (uint32_t i = tid; i < tile_n; i += kRsBlock) {
        const K k = skeys[i];
        const uint32_t d = (uint32_t)(k >> shift) & 255u;
        const uint32_t dest = dbase[d] + (i - dstart[d]);
        kout[dest] = k;
        vout[dest] = svals[i];
    }
}

// Sorts (keys, vals) on key bits [0, bits).  On return keys/vals point at the
// sorted data; *_alt point at the scratch halves (pointers may be swapped).
template <typename K>
void radix_sort_pairs(K*& keys, uint32_t*& vals, K*& keys_alt, uint32_t*& vals_alt, uint64_t n,
                      int bits, cudaStream_t s) {
    if (n <= 1 || bits <= 0) return;
    const uint32_t ntiles = (uint32_t)((n + kRsTile - 1) / kRsTile);
    const uint64_t ncount = (uint64_t)kRsRadix * ntiles;
    uint32_t* counts = dalloc<uint32_t>(ncount, s);
    uint32_t* offs = dalloc<uint32_t>(ncount + 1, s);
    const size_t smem = kRsTile * (sizeof(K) + sizeof(uint32_t));
    static bool attr_set = false;
    if (!attr_set) {
        TM_CUDA(cudaFuncSetAttribute(radix_downsweep<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        attr_set = true;
    }
    for (int shift = 0; shift < bits; shift += 8) {
        TM_LAUNCH("radix_upsweep", s, radix_upsweep<K>, ntiles, kRsBlock, 0, keys, n, shift, counts,
                  ntiles);
        exclusive_scan<uint32_t>(ArrayLoad<uint32_t>{counts}, ncount, offs, s);
        TM_LAUNCH("radix_downsweep", s, radix_downsweep<K>, ntiles, kRsBlock, smem, keys, vals,
                  keys_alt, vals_alt, n, shift, offs, ntiles);
        K* tk = keys;
        keys = keys_alt;
        keys_alt = tk;
        uint32_t* tv = vals;
        vals = vals_alt;
        vals_alt = tv;
    }
    dfree(counts, s);
    dfree(offs, s);
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
