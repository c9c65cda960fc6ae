// rankbench.cu -- throughput of the warp primitives a radix-sort ranking can
// be built from (match.any, vote.ballot, shfl, shared-memory atomics), measured
// in warp-instructions per clock per SM on the box's GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rankbench rankbench.cu
#include <cstdio>
#include <cstdint>

constexpr int ITERS = 4096;

template <int KIND>
__global__ void __launch_bounds__(256) prim(uint32_t* out, uint32_t seed) {
    __shared__ uint32_t cnt[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += 256) (&cnt[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = seed * 2654435761u + threadIdx.x * 40503u + blockIdx.x;
    uint32_t acc = 0;
#pragma unroll 4
    for (int it = 0; it < ITERS; ++it) {
        x = x * 1664525u + 1013904223u;
        const uint32_t d = x >> 24;
        if (KIND == 0) {
            acc += __match_any_sync(0xffffffffu, d);
        } else if (KIND == 1) {
            uint32_t m = 0xffffffffu;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const uint32_t v = __ballot_sync(0xffffffffu, (d >> b) & 1u);
                m &= ((d >> b) & 1u) ? v : ~v;
            }
            acc += m;
        } else if (KIND == 2) {
            acc += __shfl_sync(0xffffffffu, x, (lane + it) & 31);
        } else if (KIND == 3) {
            acc += atomicAdd(&cnt[w][d], 1u);
        } else if (KIND == 4) {
            acc += __ballot_sync(0xffffffffu, d & 1u);
        } else if (KIND == 5) {
            acc += __reduce_add_sync(0xffffffffu, d);
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int KIND>
static void run(const char* name, int nsm, int per_instr) {
    uint32_t* out;
    cudaMalloc(&out, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int blocks = nsm * 8;  // 64 warps per SM
    prim<KIND><<<blocks, 256>>>(out, 1);
    cudaEventRecord(a);
    prim<KIND><<<blocks, 256>>>(out, 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_instr = (double)blocks * 8 * ITERS * per_instr;
    const double clocks = ms * 1e-3 * clk_khz * 1e3;
    printf("%-22s %8.3f ms  %.3f warp-instr/clk/SM  (%.1f clk per warp-instr per SM)\n", name, ms,
           warp_instr / clocks / nsm, clocks * nsm / warp_instr);
    cudaFree(out);
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    run<0>("match.any.b32", nsm, 1);
    run<1>("8x ballot (WLMS)", nsm, 8);
    run<2>("shfl.idx", nsm, 1);
    run<3>("smem atomicAdd ret", nsm, 1);
    run<4>("1x ballot", nsm, 1);
    run<5>("redux.add", nsm, 1);
    return 0;
}
