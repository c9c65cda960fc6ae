// tm_parse.cu -- the reference's edge-list reader (parse_edge_list,
// graph.cpp:73-116) on the GPU: text bytes in, ingestion-order edge arrays
// and the node-id map out, ready for tm_graph_build / tm_count_edges with
// device pointers.
//
// Semantics kept exactly (graph.hpp:60-67): lines split on '\n'; fields are
// runs of non-whitespace (isspace in the C locale: ' ', \t, \n, \v, \f, \r,
// so a trailing '\r' is whitespace); a line whose first field starts with '#'
// or that has no field is skipped; fewer than 3 fields is ParseError(line,
// "expected 3 tokens: SRC DST T"); the third field must be an int64 as
// std::from_chars reads it over the whole field (optional '-', digits, no
// overflow) or ParseError(line, "malformed timestamp '<field>'"); SRC == DST
// is dropped and tallied (or ParseError(line, "self-loop edge '<id>'") when
// dropping is off) and does not register ids; further fields are ignored.
// Node ids are dense in order of first appearance among retained edges, SRC
// before DST.  The first failing line wins.
//
// Pipeline (all device passes, one host read-back for the verdict):
//   1. newline bitmask (one 32-byte word per thread) + word-popcount scan ->
//      line starts;
//   2. one thread per line over a shared-memory stage of the block's 256
//      lines: field bounds, timestamp, token keys (the bytes themselves for
//      tokens of <= 7 bytes, else a 64-bit hash), line kind; the first error
//      line by atomicMin;
//   3. scan of the edge lines -> ingestion index e; occurrences 2e / 2e+1;
//   4. interning: open-addressing table of exact short keys and (hash tag,
//      representative occurrence) long keys with byte compares on tag hits,
//      sized for the expected distinct count and regrown when half full;
//      atomicMin of the occurrence index per slot = first appearance;
//   5. ids = rank of each first appearance (scan of "is first" flags).
#include "tm_primitives.cuh"

namespace tmb {

namespace {

__device__ __forceinline__ bool is_space(unsigned char c) {
    return c == ' ' || (c >= '\t' && c <= '\r');  // \t \n \v \f \r
}

// words of 32 bytes: bit j of nl[w] = (text[32w + j] == '\n')
__global__ void newline_mask_kernel(const unsigned char* __restrict__ text, uint64_t N,
                                    uint32_t* __restrict__ nl, uint64_t W) {
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < W;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = w * 32;
        uint32_t m = 0;
        if (b + 32 <= N && ((reinterpret_cast<uintptr_t>(text + b) & 15) == 0)) {
            const uint4 x = reinterpret_cast<const uint4*>(text + b)[0];
            const uint4 y = reinterpret_cast<const uint4*>(text + b)[1];
            const uint32_t v[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
#pragma unroll
            for (int k = 0; k < 8; ++k)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (((v[k] >> (8 * j)) & 0xffu) == '\n') m |= 1u << (4 * k + j);
        } else {
            for (int j = 0; j < 32 && b + j < N; ++j)
                if (text[b + j] == '\n') m |= 1u << j;
        }
        nl[w] = m;
    }
}

struct PopcLoadNl {
    const uint32_t* m;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return __popc(m[i]); }
};

// line_start[k + 1] = position after the k-th newline; line_start[0] = 0 and
// line_start[L] = N + 1 (so the last line ends at N)
__global__ void line_starts_kernel(const uint32_t* __restrict__ nl, const uint64_t* __restrict__ pref,
                                   uint64_t W, uint64_t N, uint64_t L, uint64_t* __restrict__ ls) {
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < W;
         w += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t m = nl[w];
        uint64_t r = pref[w];
        while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            ls[++r] = w * 32 + j + 1;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ls[0] = 0;
        ls[L] = N + 1;
    }
}

enum : uint8_t { kSkip = 0, kEdge = 1, kDropped = 2, kErrShort = 3, kErrTime = 4, kErrLoop = 5 };

struct LineOut {
    uint8_t* kind;
    uint64_t* s_off;  // first byte of SRC / DST / T fields
    uint64_t* d_off;
    uint64_t* t_off;
    uint32_t* s_len;
    uint32_t* d_len;
    uint32_t* t_len;
    uint64_t* s_key;  // token key: exact bytes | len << 56 (<= 7 bytes) or a 64-bit hash
    uint64_t* d_key;
    int64_t* tv;
};

__device__ __forceinline__ uint64_t mix64(uint64_t h) {
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ull;
    h ^= h >> 33;
    return h;
}

constexpr int kLineBlock = 256;
constexpr uint32_t kStageBytes = 24 * 1024;

// one thread per line; the block's lines are staged in shared memory when
// their bytes fit (typical lines are tens of bytes)
__global__ void __launch_bounds__(kLineBlock) parse_lines_kernel(const unsigned char* __restrict__ text,
                                                                 uint64_t N, const uint64_t* __restrict__ ls,
                                                                 uint64_t L, int drop_loops, LineOut out,
                                                                 unsigned long long* __restrict__ err_line,
                                                                 unsigned long long* __restrict__ dropped) {
    __shared__ __align__(16) unsigned char stage[kStageBytes];
    __shared__ uint32_t s_drop;
    for (uint64_t l0 = (uint64_t)blockIdx.x * kLineBlock; l0 < L; l0 += (uint64_t)gridDim.x * kLineBlock) {
        const uint64_t l1 = l0 + kLineBlock < L ? l0 + kLineBlock : L;
        const uint64_t b0 = ls[l0];
        const uint64_t b1 = min(ls[l1] - (l1 == L ? 1 : 0), N);  // end of the block's last line
        const bool staged = b1 - b0 <= kStageBytes;
        if (threadIdx.x == 0) s_drop = 0;
        if (staged)
            for (uint64_t i = b0 + threadIdx.x; i < b1; i += kLineBlock) stage[i - b0] = text[i];
        __syncthreads();
        const uint64_t l = l0 + threadIdx.x;
        if (l < l1) {
            const uint64_t beg = ls[l], end = min(ls[l + 1] - 1, N);  // [beg, end) without '\n'
            auto at = [&](uint64_t i) -> unsigned char { return staged ? stage[i - b0] : text[i]; };
            uint64_t fo[3] = {0, 0, 0};
            uint32_t fl[3] = {0, 0, 0};
            uint64_t fh[2] = {0xcbf29ce484222325ull, 0xcbf29ce484222325ull};
            int nf = 0;
            bool neg = false, bad_t = false;
            uint64_t tval = 0;
            uint64_t i = beg;
            while (nf < 3) {
                while (i < end && is_space(at(i))) ++i;
                if (i >= end) break;
                fo[nf] = i;
                const uint64_t s0 = i;
                if (nf < 2) {
                    uint64_t h = fh[nf], pk = 0;
                    while (i < end && !is_space(at(i))) {
                        const unsigned char c = at(i);
                        h = (h ^ c) * 0x100000001b3ull;  // FNV-1a
                        if (i - s0 < 7) pk |= (uint64_t)c << (8 * (i - s0));
                        ++i;
                    }
                    // token key: exact (bytes | len << 56) up to 7 bytes, else a hash
                    fh[nf] = i - s0 <= 7 ? (pk | ((uint64_t)(i - s0) << 56)) : mix64(h ^ (i - s0));
                } else {
                    // std::from_chars<int64_t> over the whole field
                    neg = at(i) == '-';
                    uint64_t j = neg ? i + 1 : i;
                    bool any = false;
                    const uint64_t lim = neg ? 9223372036854775808ull : 9223372036854775807ull;
                    while (j < end && !is_space(at(j))) {
                        const unsigned char c = at(j);
                        if (c < '0' || c > '9') {
                            bad_t = true;
                        } else if (!bad_t) {
                            const uint64_t d = c - '0';
                            if (tval > (lim - d) / 10) bad_t = true;  // overflow
                            else tval = tval * 10 + d;
                            any = true;
                        }
                        ++j;
                    }
                    if (!any) bad_t = true;
                    i = j;
                }
                fl[nf] = (uint32_t)(i - s0);
                if (nf == 0 && at(s0) == '#') break;  // comment line
                ++nf;
            }
            uint8_t kind;
            if (nf == 0) {
                kind = kSkip;  // blank or comment
            } else if (nf < 3) {
                kind = kErrShort;
            } else if (bad_t) {
                kind = kErrTime;
            } else {
                bool same = fl[0] == fl[1] && fh[0] == fh[1];
                for (uint32_t k = 0; same && k < fl[0]; ++k) same = at(fo[0] + k) == at(fo[1] + k);
                kind = same ? (drop_loops ? kDropped : kErrLoop) : kEdge;
            }
            out.kind[l] = kind;
            if (kind == kEdge) {
                out.s_off[l] = fo[0];
                out.d_off[l] = fo[1];
                out.s_len[l] = fl[0];
                out.d_len[l] = fl[1];
                out.s_key[l] = fh[0];
                out.d_key[l] = fh[1];
                out.tv[l] = neg ? (int64_t)(0 - tval) : (int64_t)tval;
            } else if (kind >= kErrShort) {
                out.s_off[l] = fo[0];
                out.s_len[l] = fl[0];
                out.t_off[l] = fo[2];
                out.t_len[l] = fl[2];
                atomicMin(err_line, (unsigned long long)l);
            } else if (kind == kDropped) {
                atomicAdd(&s_drop, 1u);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && s_drop) atomicAdd(dropped, (unsigned long long)s_drop);
        __syncthreads();
    }
}

struct EdgeFlagLoad {
    const uint8_t* kind;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return kind[i] == kEdge ? 1u : 0u; }
};

constexpr unsigned long long kEmpty = ~0ull;

// occurrence o = 2 * line + side (side 0: SRC, 1: DST) of an edge line
__device__ __forceinline__ uint64_t occ_off(const LineOut& in, uint64_t o) {
    return (o & 1) ? in.d_off[o >> 1] : in.s_off[o >> 1];
}
__device__ __forceinline__ uint32_t occ_len(const LineOut& in, uint64_t o) {
    return (o & 1) ? in.d_len[o >> 1] : in.s_len[o >> 1];
}
__device__ __forceinline__ bool same_token(const unsigned char* __restrict__ text, const LineOut& in, uint32_t a,
                                           uint32_t b) {
    const uint32_t n = occ_len(in, a);
    if (occ_len(in, b) != n) return false;
    const unsigned char* p = text + occ_off(in, a);
    const unsigned char* q = text + occ_off(in, b);
    for (uint32_t k = 0; k < n; ++k)
        if (p[k] != q[k]) return false;
    return true;
}

constexpr uint32_t kNoSlot = 0xffffffffu;

// Table entries: tokens of <= 7 bytes by their exact key (top byte = length
// <= 7: no text access at all); longer ones as 0x80 << 56 | 24-bit hash tag
// << 32 | representative occurrence, confirmed by a byte compare on a tag
// hit.  Sized for the expected distinct count (L2-resident when it is small);
// a probe run longer than kMaxProbe means the table is too full: the thread
// flags it and stops, and the host retries with a 4x larger table.
__global__ void intern_kernel(const unsigned char* __restrict__ text, LineOut in, uint64_t occs,
                              unsigned long long* __restrict__ table, uint64_t mask,
                              uint32_t* __restrict__ first, uint32_t* __restrict__ occ_slot,
                              uint32_t* __restrict__ overflow, int bounded) {
    constexpr uint32_t kMaxProbe = 512;
    for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < occs;
         o += (uint64_t)gridDim.x * blockDim.x) {
        if (in.kind[o >> 1] != kEdge) {
            occ_slot[o] = kNoSlot;
            continue;
        }
        const uint64_t k = (o & 1) ? in.d_key[o >> 1] : in.s_key[o >> 1];
        const bool exact = occ_len(in, o) <= 7;
        const uint64_t h = exact ? mix64(k) : k;
        const unsigned long long key = exact ? k : (0x80ull << 56) | ((h >> 40) << 32) | o;
        uint64_t slot = h & mask;
        for (uint32_t probe = 0;; ++probe) {
            if (bounded && probe > kMaxProbe) {
                atomicExch(overflow, 1u);
                return;
            }
            unsigned long long cur = table[slot];
            if (cur == kEmpty) {
                cur = atomicCAS(&table[slot], kEmpty, key);
                if (cur == kEmpty) break;
            }
            if (exact ? cur == key
                      : ((cur >> 32) == (key >> 32) &&
                         same_token(text, in, (uint32_t)cur, (uint32_t)o)))
                break;
            slot = (slot + 1) & mask;
        }
        occ_slot[o] = (uint32_t)slot;
        if ((uint32_t)o < first[slot]) atomicMin(&first[slot], (uint32_t)o);
    }
}

struct FirstFlagLoad {
    const uint32_t* occ_slot;
    const uint32_t* first;
    __device__ __forceinline__ uint32_t operator()(uint64_t o) const {
        const uint32_t sl = occ_slot[o];
        return sl != kNoSlot && first[sl] == (uint32_t)o ? 1u : 0u;
    }
};

// ids: the rank of the token's first appearance; edges to their ingestion
// index; node tokens in id order
__global__ void assign_ids_kernel(LineOut in, const uint64_t* __restrict__ eidx,
                                  const uint32_t* __restrict__ occ_slot, const uint32_t* __restrict__ first,
                                  const uint32_t* __restrict__ rank, uint64_t occs, uint32_t* __restrict__ src,
                                  uint32_t* __restrict__ dst, int64_t* __restrict__ t,
                                  uint64_t* __restrict__ node_off, uint32_t* __restrict__ node_len) {
    for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < occs;
         o += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t sl = occ_slot[o];
        if (sl == kNoSlot) continue;
        const uint32_t f = first[sl];
        const uint32_t id = rank[f];
        const uint64_t e = eidx[o >> 1];
        if (o & 1) {
            dst[e] = id;
        } else {
            src[e] = id;
            t[e] = in.tv[o >> 1];
        }
        if (f == (uint32_t)o) {
            node_off[id] = occ_off(in, o);
            node_len[id] = occ_len(in, o);
        }
    }
}

// ---- write_edge_list (graph.cpp:170-175) for decimal node ids ------------
__device__ __forceinline__ uint32_t dec_digits(uint64_t v) {
    uint32_t d = 1;
    while (v >= 10) {
        v /= 10;
        ++d;
    }
    return d;
}
__device__ __forceinline__ uint64_t abs_t(int64_t t) { return t < 0 ? 0ull - (uint64_t)t : (uint64_t)t; }
__device__ __forceinline__ uint32_t line_bytes(uint32_t a, uint32_t b, int64_t t) {
    return dec_digits(a) + 1 + dec_digits(b) + 1 + (t < 0 ? 1 : 0) + dec_digits(abs_t(t)) + 1;
}
struct LineLenLoad {
    const uint32_t* src;
    const uint32_t* dst;
    const int64_t* t;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return line_bytes(src[i], dst[i], t[i]); }
};
__device__ __forceinline__ char* put_dec(char* p, uint64_t v, uint32_t nd) {
    for (uint32_t k = nd; k > 0; --k) {
        p[k - 1] = (char)('0' + v % 10);
        v /= 10;
    }
    return p + nd;
}
__global__ void write_lines_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                                   const int64_t* __restrict__ t, const uint64_t* __restrict__ pos, uint64_t m,
                                   char* __restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        char* p = out + pos[i];
        p = put_dec(p, src[i], dec_digits(src[i]));
        *p++ = ' ';
        p = put_dec(p, dst[i], dec_digits(dst[i]));
        *p++ = ' ';
        if (t[i] < 0) *p++ = '-';
        const uint64_t a = abs_t(t[i]);
        p = put_dec(p, a, dec_digits(a));
        *p = '\n';
    }
}

unsigned grid_of(uint64_t work) {
    const uint64_t cap = (uint64_t)sm_count() * 8;
    uint64_t g = (work + 255) / 256;
    if (g < 1) g = 1;
    return (unsigned)(g < cap ? g : cap);
}

}  // namespace

ParsedEdges parse_edge_list_device(const unsigned char* d_text, uint64_t N, bool drop_self_loops,
                                   cudaStream_t s) {
    ParsedEdges P;
    P.stream = s;
    const uint64_t W = (N + 31) / 32;
    // 1. line starts
    uint32_t* nl = dalloc<uint32_t>(W + 1, s);
    uint64_t* pref = dalloc<uint64_t>(W + 1, s);
    if (W) {
        TM_LAUNCH("parse_newlines", s, newline_mask_kernel, grid_of(W), 256, 0, d_text, N, nl, W);
        exclusive_scan<uint64_t>(PopcLoadNl{nl}, W, pref, s);
    } else {
        TM_CUDA(cudaMemsetAsync(pref, 0, sizeof(uint64_t), s));
    }
    uint64_t newlines = 0;
    TM_CUDA(cudaMemcpyAsync(&newlines, pref + W, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    const uint64_t L = newlines + 1;
    if (2 * L > 0xFFFFFFF0ull) throw tm_error(9, "edge list too large: 2 x lines must fit 32 bits");
    uint64_t* ls = dalloc<uint64_t>(L + 1, s);
    TM_LAUNCH("parse_line_starts", s, line_starts_kernel, grid_of(W ? W : 1), 256, 0, nl, pref, W, N, L, ls);
    dfree(nl, s);
    dfree(pref, s);

    // 2. per-line fields
    LineOut lo;
    lo.kind = dalloc<uint8_t>(L, s);
    lo.s_off = dalloc<uint64_t>(L, s);
    lo.d_off = dalloc<uint64_t>(L, s);
    lo.t_off = dalloc<uint64_t>(L, s);
    lo.s_len = dalloc<uint32_t>(L, s);
    lo.d_len = dalloc<uint32_t>(L, s);
    lo.t_len = dalloc<uint32_t>(L, s);
    lo.s_key = dalloc<uint64_t>(L, s);
    lo.d_key = dalloc<uint64_t>(L, s);
    lo.tv = dalloc<int64_t>(L, s);
    unsigned long long* flags = dalloc<unsigned long long>(2, s);  // [0] first error line, [1] dropped
    const unsigned long long init[2] = {~0ull, 0ull};
    TM_CUDA(cudaMemcpyAsync(flags, init, sizeof(init), cudaMemcpyHostToDevice, s));
    {
        uint64_t g = (L + kLineBlock - 1) / kLineBlock;
        const uint64_t cap = (uint64_t)sm_count() * 8;
        if (g > cap) g = cap;
        TM_LAUNCH("parse_lines", s, parse_lines_kernel, (unsigned)g, kLineBlock, 0, d_text, N, ls, L,
                  drop_self_loops ? 1 : 0, lo, flags, flags + 1);
    }
    uint64_t* eidx = dalloc<uint64_t>(L + 1, s);
    exclusive_scan<uint64_t>(EdgeFlagLoad{lo.kind}, L, eidx, s);
    unsigned long long hflags[2];
    uint64_t m = 0;
    TM_CUDA(cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaMemcpyAsync(&m, eidx + L, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    auto release_lines = [&] {
        dfree(lo.kind, s); dfree(lo.s_off, s); dfree(lo.d_off, s); dfree(lo.t_off, s); dfree(lo.s_len, s);
        dfree(lo.d_len, s); dfree(lo.t_len, s); dfree(lo.s_key, s); dfree(lo.d_key, s); dfree(lo.tv, s);
        dfree(flags, s); dfree(eidx, s); dfree(ls, s);
    };
    if (hflags[0] != ~0ull) {
        // the first failing line: the reference's ParseError text
        const uint64_t l = hflags[0];
        uint8_t kind = 0;
        uint64_t so = 0, to = 0;
        uint32_t sl = 0, tl = 0;
        TM_CUDA(cudaMemcpyAsync(&kind, lo.kind + l, 1, cudaMemcpyDeviceToHost, s));
        TM_CUDA(cudaMemcpyAsync(&so, lo.s_off + l, 8, cudaMemcpyDeviceToHost, s));
        TM_CUDA(cudaMemcpyAsync(&sl, lo.s_len + l, 4, cudaMemcpyDeviceToHost, s));
        TM_CUDA(cudaMemcpyAsync(&to, lo.t_off + l, 8, cudaMemcpyDeviceToHost, s));
        TM_CUDA(cudaMemcpyAsync(&tl, lo.t_len + l, 4, cudaMemcpyDeviceToHost, s));
        TM_CUDA(cudaStreamSynchronize(s));
        std::string field;
        const uint64_t fo = kind == kErrTime ? to : so;
        const uint32_t fln = kind == kErrTime ? tl : sl;
        if (kind != kErrShort && fln) {
            field.resize(fln);
            TM_CUDA(cudaMemcpyAsync(&field[0], d_text + fo, fln, cudaMemcpyDeviceToHost, s));
            TM_CUDA(cudaStreamSynchronize(s));
        }
        release_lines();
        std::string what = kind == kErrShort  ? "expected 3 tokens: SRC DST T"
                           : kind == kErrTime ? "malformed timestamp '" + field + "'"
                                              : "self-loop edge '" + field + "'";
        throw parse_error(l + 1, "line " + std::to_string(l + 1) + ": " + what);
    }
    P.m = m;
    P.dropped = hflags[1];

    // 3. occurrences o = 2 * line + side (non-edge lines are holes)
    P.t = dalloc<int64_t>(m, s);
    P.src = dalloc<uint32_t>(m, s);
    P.dst = dalloc<uint32_t>(m, s);
    const uint64_t occs = 2 * L;
    const uint64_t toks = 2 * m;  // tokens actually present

    // 4. interning: first a table for max(2^20, tokens / 16) distinct tokens
    //    at load <= 1/2, 4x larger whenever a probe run overflows
    uint64_t want = std::max<uint64_t>(1ull << 20, toks / 16);
    uint64_t cap_max = 1024;
    while (cap_max < toks + toks / 2 + 1) cap_max <<= 1;
    uint64_t cap = 1024;
    while (cap < 2 * want) cap <<= 1;
    cap = std::min(cap, cap_max);
    uint32_t* occ_slot = dalloc<uint32_t>(occs, s);
    uint32_t* first = nullptr;
    uint32_t* overflow = dalloc<uint32_t>(1, s);
    for (;;) {
        unsigned long long* table = dalloc<unsigned long long>(cap, s);
        first = dalloc<uint32_t>(cap, s);
        TM_CUDA(cudaMemsetAsync(table, 0xff, cap * sizeof(unsigned long long), s));
        TM_CUDA(cudaMemsetAsync(first, 0xff, cap * sizeof(uint32_t), s));
        TM_CUDA(cudaMemsetAsync(overflow, 0, sizeof(uint32_t), s));
        const int bounded = cap < cap_max;  // the largest table holds every token at load <= 2/3
        if (toks)
            TM_LAUNCH("parse_intern", s, intern_kernel, grid_of(occs), 256, 0, d_text, lo, occs, table, cap - 1,
                      first, occ_slot, overflow, bounded);
        uint32_t hov = 0;
        TM_CUDA(cudaMemcpyAsync(&hov, overflow, sizeof(hov), cudaMemcpyDeviceToHost, s));
        dfree(table, s);
        TM_CUDA(cudaStreamSynchronize(s));
        if (!hov) break;
        dfree(first, s);
        cap = std::min(cap * 4, cap_max);
    }
    dfree(overflow, s);
    // 5. ids by first appearance
    uint32_t* rank = dalloc<uint32_t>(occs + 1, s);
    uint32_t n32 = 0;
    if (toks) {
        exclusive_scan<uint32_t>(FirstFlagLoad{occ_slot, first}, occs, rank, s);
        TM_CUDA(cudaMemcpyAsync(&n32, rank + occs, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        TM_CUDA(cudaStreamSynchronize(s));
    }
    P.n = n32;
    P.node_off = dalloc<uint64_t>(P.n, s);
    P.node_len = dalloc<uint32_t>(P.n, s);
    if (toks)
        TM_LAUNCH("parse_ids", s, assign_ids_kernel, grid_of(occs), 256, 0, lo, eidx, occ_slot, first, rank, occs,
                  P.src, P.dst, P.t, P.node_off, P.node_len);
    dfree(first, s);
    dfree(occ_slot, s);
    dfree(rank, s);
    release_lines();
    return P;
}

uint64_t edge_list_text_bytes(const uint32_t* d_src, const uint32_t* d_dst, const int64_t* d_t, uint64_t m,
                              cudaStream_t s) {
    if (m == 0) return 0;
    uint64_t* pos = dalloc<uint64_t>(m + 1, s);
    exclusive_scan<uint64_t>(LineLenLoad{d_src, d_dst, d_t}, m, pos, s);
    uint64_t bytes = 0;
    TM_CUDA(cudaMemcpyAsync(&bytes, pos + m, 8, cudaMemcpyDeviceToHost, s));
    dfree(pos, s);
    TM_CUDA(cudaStreamSynchronize(s));
    return bytes;
}

void write_edge_list_device(const uint32_t* d_src, const uint32_t* d_dst, const int64_t* d_t, uint64_t m,
                            char* d_out, cudaStream_t s) {
    if (m == 0) return;
    uint64_t* pos = dalloc<uint64_t>(m + 1, s);
    exclusive_scan<uint64_t>(LineLenLoad{d_src, d_dst, d_t}, m, pos, s);
    TM_LAUNCH("write_lines", s, write_lines_kernel, grid_of(m), 256, 0, d_src, d_dst, d_t, pos, m, d_out);
    dfree(pos, s);
}

void free_parsed(ParsedEdges& P) {
    cudaStream_t s = P.stream;
    dfree(P.src, s);
    dfree(P.dst, s);
    dfree(P.t, s);
    dfree(P.node_off, s);
    dfree(P.node_len, s);
    dfree(P.text, s);
}

}  // namespace tmb
