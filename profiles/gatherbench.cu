// Random 8-byte gathers from a 4.8 GB record array (the gather_s pattern at
// config 4: 1.2G incident records reading 600M 8-byte edge records), with the
// load flavours and the L2 fetch-granularity limit as variants.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gatherbench gatherbench.cu
//   ./gatherbench [fetch_granularity_bytes]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void make_idx(uint32_t* idx, uint64_t R, uint64_t m) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < R; i += (uint64_t)gridDim.x * blockDim.x)
        idx[i] = (uint32_t)(mix(i) % m);
}

template <int V>
__device__ __forceinline__ uint64_t load(const uint64_t* p) {
    if (V == 0) {  // two 32-bit read-only loads (what gather_s compiles to)
        const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
        return (uint64_t)__ldg(q) | ((uint64_t)__ldg(q + 1) << 32);
    } else if (V == 1) {
        return __ldg(reinterpret_cast<const unsigned long long*>(p));
    } else if (V == 2) {
        return __ldcg(reinterpret_cast<const unsigned long long*>(p));
    } else if (V == 3) {
        uint64_t v;
        asm volatile("ld.global.nc.L1::no_allocate.b64 %0, [%1];" : "=l"(v) : "l"(p));
        return v;
    } else if (V == 4) {
        uint64_t v;
        asm volatile("ld.global.L1::no_allocate.b64 %0, [%1];" : "=l"(v) : "l"(p));
        return v;
    } else if (V == 6) {
        uint64_t v;
        asm volatile("ld.volatile.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
        return v;
    } else if (V == 7) {  // one 32-bit load only
        return __ldg(reinterpret_cast<const uint32_t*>(p));
    } else if (V == 8) {
        uint64_t v;
        asm volatile("{ .reg .b64 pol; createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
                     "ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], pol; }" : "=l"(v) : "l"(p));
        return v;
    } else if (V == 9) {  // L2 atomic (32-byte granularity at L2)
        return atomicOr(reinterpret_cast<unsigned long long*>(const_cast<uint64_t*>(p)), 0ull);
    } else {
        return *p;
    }
}

template <int V>
__global__ void __launch_bounds__(256) gather(const uint64_t* __restrict__ E, const uint32_t* __restrict__ idx,
                                              uint64_t R, uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < R; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = __ldcs(idx + i);
        __stcs(out + i, load<V>(E + p));
    }
}

// cp.async 8 B per thread into shared memory, then read back
__global__ void __launch_bounds__(256) gather_cpa(const uint64_t* __restrict__ E, const uint32_t* __restrict__ idx,
                                                  uint64_t R, uint64_t* __restrict__ out) {
    __shared__ uint64_t buf[256];
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < R; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = __ldcs(idx + i);
        const unsigned sa = (unsigned)__cvta_generic_to_shared(&buf[threadIdx.x]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(sa), "l"(E + p));
        asm volatile("cp.async.wait_all;" ::: "memory");
        __stcs(out + i, buf[threadIdx.x]);
    }
}
float run_cpa(const uint64_t* E, const uint32_t* idx, uint64_t R, uint64_t* out, int grid) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather_cpa<<<grid, 256>>>(E, idx, R, out);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) gather_cpa<<<grid, 256>>>(E, idx, R, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 3;
}

template <int V>
float run(const uint64_t* E, const uint32_t* idx, uint64_t R, uint64_t* out, int grid) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather<V><<<grid, 256>>>(E, idx, R, out);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) gather<V><<<grid, 256>>>(E, idx, R, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 3;
}

int main(int argc, char** argv) {
    if (argc > 1) {
        size_t g = atoi(argv[1]);
        CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g));
    }
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    const uint64_t m = 600000000ull, R = 1200000000ull;
    uint64_t *E, *out;
    uint32_t* idx;
    CK(cudaMalloc(&E, m * 8));
    CK(cudaMalloc(&out, R * 8));
    CK(cudaMalloc(&idx, R * 4));
    CK(cudaMemset(E, 1, m * 8));
    make_idx<<<148 * 8, 256>>>(idx, R, m);
    CK(cudaDeviceSynchronize());
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int grid : {sms * 8, sms * 32}) {
        printf("fetch_granularity %zu grid %d\n", got, grid);
        printf("  v0 two u32 ldg      %8.3f ms\n", run<0>(E, idx, R, out, grid));
        printf("  v1 u64 ldg          %8.3f ms\n", run<1>(E, idx, R, out, grid));
        printf("  v2 u64 ldcg         %8.3f ms\n", run<2>(E, idx, R, out, grid));
        printf("  v3 nc no_allocate   %8.3f ms\n", run<3>(E, idx, R, out, grid));
        printf("  v4 no_allocate      %8.3f ms\n", run<4>(E, idx, R, out, grid));
        printf("  v5 plain            %8.3f ms\n", run<5>(E, idx, R, out, grid));
        printf("  v6 volatile         %8.3f ms\n", run<6>(E, idx, R, out, grid));
        printf("  v7 u32 only         %8.3f ms\n", run<7>(E, idx, R, out, grid));
        printf("  v8 nc evict_first   %8.3f ms\n", run<8>(E, idx, R, out, grid));
        printf("  v9 atomicOr 0       %8.3f ms\n", run<9>(E, idx, R, out, grid));
        printf("  v10 cp.async 8B     %8.3f ms\n", run_cpa(E, idx, R, out, grid));
    }
    return 0;
}
