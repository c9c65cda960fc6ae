// tm_graph.cu -- GPU construction of the temporal adjacency.
//
// Replaces TemporalGraph::build (graph.cpp:13-44), NodeSequenceIndex
// (indexes.cpp:7-26) and PairEdgeIndex (indexes.cpp:28-58):
//   1. validate endpoints, find t range, detect already-sorted input;
//   2. stable radix sort of edges by t (skipped when already sorted), so the
//      edge order is the reference's (t, ordinal) total order;
//   3. stable radix sort of the 2m incident records (emitted in that order)
//      by node -> S, the per-node time-ordered sequences;
//   4. stable radix sort of S by (node, other) -> G, the same records grouped
//      by neighbour; its (v, w) groups are the per-pair time-sorted edge lists.
#include "tm_primitives.cuh"

namespace tmb {

namespace {

struct BuildStats {
    long long tmin;
    long long tmax;
    unsigned int bad;
    unsigned int unsorted;
    unsigned int max_degree;
    unsigned int pad;
};

__global__ void validate_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                const int64_t* __restrict__ t, uint64_t m, uint64_t n,
                                BuildStats* st) {
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    unsigned bad = 0, uns = 0;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = src[k], b = dst[k];
        const long long tk = t[k];
        bad |= (a == b) | (a >= n) | (b >= n) | (a > kNodeMask) | (b > kNodeMask);
        lo = min(lo, tk);
        hi = max(hi, tk);
        if (k + 1 < m) uns |= (t[k + 1] < tk);
    }
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

__global__ void time_keys_kernel(const int64_t* __restrict__ t, uint64_t m, int64_t tmin,
                                 uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (uint64_t)gridDim.x * blockDim.x) {
        keys[k] = (uint64_t)t[k] - (uint64_t)tmin;
        vals[k] = (uint32_t)k;
    }
}

// record r = 2p + side of the p-th edge in (t, ordinal) order
__global__ void node_keys_kernel(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ src,
                                 const uint32_t* __restrict__ dst, uint64_t R,
                                 uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p = r >> 1;
        const uint32_t k = perm ? perm[p] : (uint32_t)p;
        keys[r] = (r & 1) ? dst[k] : src[k];
        vals[r] = (uint32_t)r;
    }
}

__global__ void gather_s_kernel(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ src,
                                const uint32_t* __restrict__ dst, const int64_t* __restrict__ t,
                                const uint32_t* __restrict__ skeys,
                                const uint32_t* __restrict__ svals, uint64_t R,
                                int64_t* __restrict__ S_t, uint32_t* __restrict__ S_nbr,
                                uint32_t* __restrict__ S_ord, uint32_t* __restrict__ S_node) {
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < R;
         q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = svals[q];
        const uint32_t p = r >> 1, side = r & 1u;
        const uint32_t k = perm ? perm[p] : p;
        S_t[q] = t[k];
        S_ord[q] = k;
        S_node[q] = skeys[q];
        S_nbr[q] = (side ? src[k] : dst[k]) | (side << 31);
    }
}

// off[x] = first position of node x (boundary fill over the sorted node ids)
__global__ void offsets_kernel(const uint32_t* __restrict__ node, uint64_t R, uint64_t n,
                               uint32_t* __restrict__ off) {
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < R;
         q += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t cur = node[q];
        const int64_t prev = q ? (int64_t)node[q - 1] : -1;
        for (int64_t x = prev + 1; x <= cur; ++x) off[x] = (uint32_t)q;
        if (q == R - 1)
            for (int64_t x = cur + 1; x <= (int64_t)n; ++x) off[x] = (uint32_t)R;
    }
}

__global__ void max_degree_kernel(const uint32_t* __restrict__ off, uint64_t n, BuildStats* st) {
    unsigned mx = 0;
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x)
        mx = max(mx, off[u + 1] - off[u]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&st->max_degree, mx);
}

__global__ void group_keys_kernel(const uint32_t* __restrict__ S_node,
                                  const uint32_t* __restrict__ S_nbr, uint64_t R, int nb,
                                  uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < R;
         q += (uint64_t)gridDim.x * blockDim.x) {
        keys[q] = ((uint64_t)S_node[q] << nb) | (S_nbr[q] & kNodeMask);
        vals[q] = (uint32_t)q;
    }
}

__global__ void gather_g_kernel(const uint64_t* __restrict__ gkeys,
                                const uint32_t* __restrict__ gvals, uint64_t R, int nb,
                                const uint32_t* __restrict__ off, const int64_t* __restrict__ S_t,
                                const uint32_t* __restrict__ S_ord,
                                const uint32_t* __restrict__ S_nbr,
                                const uint32_t* __restrict__ S_pg, int64_t* __restrict__ G_t,
                                uint32_t* __restrict__ G_ord, uint32_t* __restrict__ G_w2,
                                uint32_t* __restrict__ G_pg, uint32_t* __restrict__ S_gidx) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < R;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = gvals[k];
        const uint64_t key = gkeys[k];
        const uint32_t node = (uint32_t)(key >> nb);
        const uint32_t first = (k == 0 || gkeys[k - 1] != key) ? kFirstBit : 0u;
        const uint32_t last = (k == R - 1 || gkeys[k + 1] != key) ? kLastBit : 0u;
        const uint32_t pos = q - off[node];
        G_t[k] = S_t[q];
        G_ord[k] = S_ord[q];
        G_pg[k] = S_pg[q];
        G_w2[k] = pos | first | last | (S_nbr[q] & kDirBit);
        S_gidx[q] = (uint32_t)k;
    }
}

__global__ void group_table_kernel(const uint64_t* __restrict__ gkeys,
                                   const uint32_t* __restrict__ G_w2,
                                   const uint32_t* __restrict__ gscan, uint64_t R, uint64_t nmask,
                                   uint32_t* __restrict__ grp_nbr, uint32_t* __restrict__ grp_off) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < R;
         k += (uint64_t)gridDim.x * blockDim.x) {
        if (G_w2[k] & kFirstBit) {
            const uint32_t g = gscan[k];
            grp_off[g] = (uint32_t)k;
            grp_nbr[g] = (uint32_t)(gkeys[k] & nmask);
        }
        if (k == R - 1) grp_off[gscan[R]] = (uint32_t)R;
    }
}

__global__ void node_group_kernel(const uint32_t* __restrict__ off,
                                  const uint32_t* __restrict__ gscan, uint64_t n,
                                  uint32_t* __restrict__ node_grp) {
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u <= n;
         u += (uint64_t)gridDim.x * blockDim.x)
        node_grp[u] = gscan[off[u]];
}

struct OutwardLoad {
    const uint32_t* nbr;
    __device__ __forceinline__ uint32_t operator()(uint64_t i) const {
        return (nbr[i] & kDirBit) ? 0u : 1u;
    }
};
struct InwardG {
    const uint32_t* w2;
    __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return w2[i] >> 31; }
};
struct FirstG {
    const uint32_t* w2;
    __device__ __forceinline__ uint32_t operator()(uint64_t i) const {
        return (w2[i] >> 29) & 1u;
    }
};

// forward(u -> x): mode 0 degree rank (deg, id), mode 1 node index
struct ForwardFlag {
    const uint32_t* node;
    const uint32_t* nbr;
    const uint32_t* off;
    int mode;
    __device__ __forceinline__ uint32_t operator()(uint64_t q) const {
        const uint32_t u = node[q], x = nbr[q] & kNodeMask;
        if (mode == 1) return x > u ? 1u : 0u;
        const uint32_t du = off[u + 1] - off[u], dx = off[x + 1] - off[x];
        return (dx > du || (dx == du && x > u)) ? 1u : 0u;
    }
};

__global__ void forward_scatter_kernel(ForwardFlag flag, const uint32_t* __restrict__ fscan,
                                       uint64_t R, const int64_t* __restrict__ S_t,
                                       const uint32_t* __restrict__ S_ord, int64_t* __restrict__ F_t,
                                       uint32_t* __restrict__ F_nbr, uint32_t* __restrict__ F_ord,
                                       uint32_t* __restrict__ F_node) {
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < R;
         q += (uint64_t)gridDim.x * blockDim.x) {
        if (flag(q)) {
            const uint32_t j = fscan[q];
            F_t[j] = S_t[q];
            F_nbr[j] = flag.nbr[q];
            F_ord[j] = S_ord[q];
            F_node[j] = flag.node[q];
        }
    }
}

__global__ void forward_off_kernel(const uint32_t* __restrict__ off,
                                   const uint32_t* __restrict__ fscan, uint64_t n,
                                   uint32_t* __restrict__ F_off) {
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u <= n;
         u += (uint64_t)gridDim.x * blockDim.x)
        F_off[u] = fscan[off[u]];
}

unsigned grid_for(uint64_t work, int block = 256) {
    const uint64_t cap = (uint64_t)sm_count() * 8;
    uint64_t g = (work + block - 1) / block;
    if (g < 1) g = 1;
    return (unsigned)(g < cap ? g : cap);
}

}  // namespace

void build_graph(DeviceGraph& g, const uint32_t* d_src, const uint32_t* d_dst, const int64_t* d_t,
                 uint64_t m, uint64_t n) {
    cudaStream_t s = g.stream;
    if (2 * m > 0xFFFFFFF0ull) throw tm_error(9, "graph too large: 2m must fit 32-bit positions");
    if (n > kNodeMask) throw tm_error(9, "graph too large: node ids must fit 31 bits");
    g.n = n;
    g.m = m;
    g.R = 2 * m;
    const uint64_t R = g.R;

    BuildStats* d_st = dalloc<BuildStats>(1, s);
    BuildStats h_st{LLONG_MAX, LLONG_MIN, 0, 0, 0, 0};
    TM_CUDA(cudaMemcpyAsync(d_st, &h_st, sizeof(h_st), cudaMemcpyHostToDevice, s));
    if (m) {
        TM_LAUNCH("validate", s, validate_kernel, grid_for(m), 256, 0, d_src, d_dst, d_t, m, n,
                  d_st);
    }
    TM_CUDA(cudaMemcpyAsync(&h_st, d_st, sizeof(h_st), cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    if (h_st.bad) {
        dfree(d_st, s);
        throw tm_error(1, "self-loop or out-of-range endpoint in edge list");
    }

    g.off = dalloc<uint32_t>(n + 1, s);
    g.node_grp = dalloc<uint32_t>(n + 1, s);
    g.S_t = dalloc<int64_t>(R, s);
    g.S_nbr = dalloc<uint32_t>(R, s);
    g.S_ord = dalloc<uint32_t>(R, s);
    g.S_node = dalloc<uint32_t>(R, s);
    g.S_pg = dalloc<uint32_t>(R + 1, s);
    g.S_gidx = dalloc<uint32_t>(R, s);
    g.G_t = dalloc<int64_t>(R, s);
    g.G_ord = dalloc<uint32_t>(R, s);
    g.G_w2 = dalloc<uint32_t>(R, s);
    g.G_pg = dalloc<uint32_t>(R, s);
    g.G_dscan = dalloc<uint32_t>(R + 1, s);
    g.grp_nbr = dalloc<uint32_t>(R, s);
    g.grp_off = dalloc<uint32_t>(R + 1, s);

    if (m == 0) {
        TM_CUDA(cudaMemsetAsync(g.off, 0, (n + 1) * sizeof(uint32_t), s));
        TM_CUDA(cudaMemsetAsync(g.node_grp, 0, (n + 1) * sizeof(uint32_t), s));
        TM_CUDA(cudaMemsetAsync(g.S_pg, 0, sizeof(uint32_t), s));
        TM_CUDA(cudaMemsetAsync(g.G_dscan, 0, sizeof(uint32_t), s));
        TM_CUDA(cudaMemsetAsync(g.grp_off, 0, sizeof(uint32_t), s));
        g.ng = 0;
        g.max_degree = 0;
        dfree(d_st, s);
        return;
    }

    // 2. (t, ordinal) order of the edges
    uint32_t* perm = nullptr;
    if (h_st.unsorted) {
        uint64_t* k0 = dalloc<uint64_t>(m, s);
        uint64_t* k1 = dalloc<uint64_t>(m, s);
        uint32_t* v0 = dalloc<uint32_t>(m, s);
        uint32_t* v1 = dalloc<uint32_t>(m, s);
        TM_LAUNCH("time_keys", s, time_keys_kernel, grid_for(m), 256, 0, d_t, m,
                  (int64_t)h_st.tmin, k0, v0);
        const int tbits = bit_width_u64((uint64_t)h_st.tmax - (uint64_t)h_st.tmin);
        radix_sort_pairs<uint64_t>(k0, v0, k1, v1, m, tbits, s);
        perm = v0;
        dfree(k0, s);
        dfree(k1, s);
        dfree(v1, s);
    }

    // 3. S: stable sort of incident records by node
    const int nb = bit_width_u64(n > 1 ? n - 1 : 1);
    uint32_t* nk0 = dalloc<uint32_t>(R, s);
    uint32_t* nk1 = dalloc<uint32_t>(R, s);
    uint32_t* nv0 = dalloc<uint32_t>(R, s);
    uint32_t* nv1 = dalloc<uint32_t>(R, s);
    TM_LAUNCH("node_keys", s, node_keys_kernel, grid_for(R), 256, 0, perm, d_src, d_dst, R, nk0,
              nv0);
    radix_sort_pairs<uint32_t>(nk0, nv0, nk1, nv1, R, nb, s);
    TM_LAUNCH("gather_s", s, gather_s_kernel, grid_for(R), 256, 0, perm, d_src, d_dst, d_t, nk0,
              nv0, R, g.S_t, g.S_nbr, g.S_ord, g.S_node);
    dfree(nk0, s);
    dfree(nk1, s);
    dfree(nv0, s);
    dfree(nv1, s);
    if (perm) dfree(perm, s);

    TM_LAUNCH("offsets", s, offsets_kernel, grid_for(R), 256, 0, g.S_node, R, n, g.off);
    TM_LAUNCH("max_degree", s, max_degree_kernel, grid_for(n), 256, 0, g.off, n, d_st);
    exclusive_scan<uint32_t>(OutwardLoad{g.S_nbr}, R, g.S_pg, s);

    // 4. G: stable sort of S by (node, other)
    uint64_t* gk0 = dalloc<uint64_t>(R, s);
    uint64_t* gk1 = dalloc<uint64_t>(R, s);
    uint32_t* gv0 = dalloc<uint32_t>(R, s);
    uint32_t* gv1 = dalloc<uint32_t>(R, s);
    TM_LAUNCH("group_keys", s, group_keys_kernel, grid_for(R), 256, 0, g.S_node, g.S_nbr, R, nb,
              gk0, gv0);
    radix_sort_pairs<uint64_t>(gk0, gv0, gk1, gv1, R, 2 * nb, s);
    TM_LAUNCH("gather_g", s, gather_g_kernel, grid_for(R), 256, 0, gk0, gv0, R, nb, g.off, g.S_t,
              g.S_ord, g.S_nbr, g.S_pg, g.G_t, g.G_ord, g.G_w2, g.G_pg, g.S_gidx);
    exclusive_scan<uint32_t>(InwardG{g.G_w2}, R, g.G_dscan, s);
    uint32_t* gscan = dalloc<uint32_t>(R + 1, s);
    exclusive_scan<uint32_t>(FirstG{g.G_w2}, R, gscan, s);
    TM_LAUNCH("group_table", s, group_table_kernel, grid_for(R), 256, 0, gk0, g.G_w2, gscan, R,
              (uint64_t)((1ull << nb) - 1), g.grp_nbr, g.grp_off);
    TM_LAUNCH("node_group", s, node_group_kernel, grid_for(n + 1), 256, 0, g.off, gscan, n,
              g.node_grp);
    uint32_t ng32 = 0;
    TM_CUDA(cudaMemcpyAsync(&ng32, gscan + R, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaMemcpyAsync(&h_st, d_st, sizeof(h_st), cudaMemcpyDeviceToHost, s));
    dfree(gk0, s);
    dfree(gk1, s);
    dfree(gv0, s);
    dfree(gv1, s);
    dfree(gscan, s);
    dfree(d_st, s);
    TM_CUDA(cudaStreamSynchronize(s));
    g.ng = ng32;
    g.max_degree = h_st.max_degree;
    if (g.max_degree > kPosMask)
        throw tm_error(9, "node degree exceeds the 29-bit in-node position layout");
}

void build_forward(DeviceGraph& g, int mode) {
    Forward& f = g.fwd[mode];
    if (f.valid) return;
    cudaStream_t s = g.stream;
    const uint64_t R = g.R;
    f.mode = mode;
    f.len = g.m;  // every edge is forward from exactly one endpoint
    f.t = dalloc<int64_t>(g.m, s);
    f.nbr = dalloc<uint32_t>(g.m, s);
    f.ord = dalloc<uint32_t>(g.m, s);
    f.node = dalloc<uint32_t>(g.m, s);
    f.off = dalloc<uint32_t>(g.n + 1, s);
    uint32_t* fscan = dalloc<uint32_t>(R + 1, s);
    ForwardFlag flag{g.S_node, g.S_nbr, g.off, mode};
    exclusive_scan<uint32_t>(flag, R, fscan, s);
    if (R) {
        TM_LAUNCH("forward_scatter", s, forward_scatter_kernel, grid_for(R), 256, 0, flag, fscan, R,
                  g.S_t, g.S_ord, f.t, f.nbr, f.ord, f.node);
    }
    TM_LAUNCH("forward_off", s, forward_off_kernel, grid_for(g.n + 1), 256, 0, g.off, fscan, g.n,
              f.off);
    dfree(fscan, s);
    f.valid = true;
}

void free_graph(DeviceGraph& g) {
    cudaStream_t s = g.stream;
    dfree(g.S_t, s); dfree(g.S_nbr, s); dfree(g.S_ord, s); dfree(g.S_node, s);
    dfree(g.S_pg, s); dfree(g.S_gidx, s); dfree(g.off, s);
    dfree(g.G_t, s); dfree(g.G_ord, s); dfree(g.G_w2, s); dfree(g.G_pg, s);
    dfree(g.G_dscan, s); dfree(g.grp_nbr, s); dfree(g.grp_off, s); dfree(g.node_grp, s);
    for (auto& f : g.fwd) {
        dfree(f.t, s); dfree(f.nbr, s); dfree(f.ord, s); dfree(f.node, s); dfree(f.off, s);
        f.valid = false;
    }
    dfree(g.d_acc, s);
}

}  // namespace tmb
