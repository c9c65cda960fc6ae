// sortbench.cu -- microbenchmark of the build's radix sort (tm_primitives.cuh)
// on the two key shapes the graph build sorts: node keys (node << 32 | record,
// 2m of them, nb key bits) and pair keys (min << 32 | edge, m of them).
// Checks the result is sorted and stable, prints per-kernel device times.
//   make -C profiles sortbench && profiles/sortbench [m] [n]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../include/tmotif_b200.h"
#include "../paper_2204_09236_b200/csrc/tm_primitives.cuh"

using namespace tmb;

template <int BLOCK, int ITEMS, int MINB>
static void run(const char* label, std::vector<uint64_t>& h, int bit_lo, int bit_hi, int reps) {
    const uint64_t n = h.size();
    uint64_t *k0, *k1;
    cudaMalloc(&k0, (n + kSortPad) * 8);
    cudaMalloc(&k1, (n + kSortPad) * 8);
    uint32_t *v0 = nullptr, *v1 = nullptr;
    cudaStream_t s = 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps + 2; ++r) {
        cudaMemcpy(k0, h.data(), n * 8, cudaMemcpyHostToDevice);
        if (r == 2) {
            tm_kernel_timing_reset();
            tm_kernel_timing_enable(1);
        }
        uint64_t* a = k0;
        uint64_t* b = k1;
        cudaEventRecord(e0, s);
        radix_sort_cfg<uint64_t, BLOCK, ITEMS, MINB>(a, v0, b, v1, n, bit_lo, bit_hi, s, nullptr);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 2 && ms < best) best = ms;
        if (r == reps + 1) {
            std::vector<uint64_t> out(n);
            cudaMemcpy(out.data(), a, n * 8, cudaMemcpyDeviceToHost);
            const uint64_t km = ((bit_hi >= 64) ? ~0ull : ((1ull << bit_hi) - 1)) & ~((1ull << bit_lo) - 1);
            uint64_t bad = 0;
            for (uint64_t i = 1; i < n; ++i) {
                const uint64_t x = out[i - 1] & km, y = out[i] & km;
                if (x > y || (x == y && out[i - 1] > out[i])) ++bad;  // low bits = input index
            }
            printf("%s: n=%llu bits [%d,%d) best %.3f ms (%.1f GB/s r+w per pass)  unsorted/unstable=%llu\n",
                   label, (unsigned long long)n, bit_lo, bit_hi, best,
                   16.0 * n * ((bit_hi - bit_lo + 7) / 8) / (best * 1e6), (unsigned long long)bad);
        }
    }
    tm_kernel_timing_enable(0);
    const char* names[] = {"radix_upsweep", "radix_scan", "radix_downsweep"};
    for (const char* nm : names) {
        double t = 0;
        uint64_t l = 0;
        tm_kernel_timing_get(nm, &t, &l);
        printf("   %-16s %8.4f ms/sort  (%llu launches/sort)\n", nm, t / reps, (unsigned long long)(l / reps));
    }
    cudaFree(k0);
    cudaFree(k1);
}

int main(int argc, char** argv) {
    const uint64_t m = argc > 1 ? strtoull(argv[1], nullptr, 10) : 10000000ull;
    const uint64_t n = argc > 2 ? strtoull(argv[2], nullptr, 10) : 1000000ull;
    int nb = 1;
    while ((1ull << nb) < n) ++nb;
    std::mt19937_64 rng(2204);
    // power-law-ish node draw (Chung-Lu weights ~ i^-0.6)
    std::vector<double> cw(n);
    double acc = 0;
    for (uint64_t i = 0; i < n; ++i) cw[i] = (acc += 1.0 / std::pow((double)(i + 1), 0.6));
    auto draw = [&]() {
        const double x = std::uniform_real_distribution<double>(0, acc)(rng);
        return (uint64_t)(std::lower_bound(cw.begin(), cw.end(), x) - cw.begin());
    };
    std::vector<uint64_t> node(2 * m), pair(m);
    for (uint64_t r = 0; r < 2 * m; ++r) node[r] = (draw() << 32) | r;
    for (uint64_t p = 0; p < m; ++p) pair[p] = (draw() << 32) | p;
    // tile shapes (BLOCK threads x ITEMS keys, MINB blocks per SM); the product uses 256 x 8, 4
    run<kSortBlock, kSortItems, kSortMinBlocks>("node keys (product tiles)", node, 32, 32 + nb, 5);
    run<kSortBlock, kSortItems, kSortMinBlocks>("pair keys (product tiles)", pair, 32, 32 + nb, 5);
    if (argc > 3) {
        run<256, 8, 5>("node keys 256x8/5", node, 32, 32 + nb, 5);
        run<256, 8, 6>("node keys 256x8/6", node, 32, 32 + nb, 5);
        run<256, 12, 3>("node keys 256x12/3", node, 32, 32 + nb, 5);
        run<256, 16, 2>("node keys 256x16/2", node, 32, 32 + nb, 5);
        run<512, 8, 2>("node keys 512x8/2", node, 32, 32 + nb, 5);
        run<512, 4, 4>("node keys 512x4/4", node, 32, 32 + nb, 5);
        run<256, 4, 8>("node keys 256x4/8", node, 32, 32 + nb, 5);
    }
    return 0;
}
