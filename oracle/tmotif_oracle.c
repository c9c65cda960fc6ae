/*
 * tmotif_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's CPU algorithm for the hot path
 * (arXiv 2204.09236 FAST-Star / FAST-Tri / HARE, as implemented under
 * /root/reference/proj).  It is the parity checker for the CUDA path: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * it.  The product library (paper_2204_09236_b200/libtmotif_b200.so) never
 * links or calls this file.
 *
 * Parity pinned against: (1) the reference's frozen Fig.-1 toy census
 * (proj/tests/test_util.hpp:116-131), (2) censuses and raw counters produced
 * by the reference itself compiled from its own sources (oracle/_ref, see
 * oracle/Makefile) on seeded graphs, stored in tests/golden/.
 *
 * Every function cites the reference file:line it restates.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_ARG 1
#define ORC_ERR_OVERFLOW 3
#define ORC_ERR_CONSISTENCY 5

/* ------------------------------------------------------------------ */
/* saturating timestamp arithmetic: types.hpp:72-89                    */
static int64_t sat_add(int64_t a, int64_t b) {
    int64_t r;
    if (__builtin_add_overflow(a, b, &r)) return b > 0 ? INT64_MAX : INT64_MIN;
    return r;
}
static int64_t sat_sub(int64_t a, int64_t b) {
    int64_t r;
    if (__builtin_sub_overflow(a, b, &r)) return b < 0 ? INT64_MAX : INT64_MIN;
    return r;
}
static int g_overflow = 0;
/* checked_increment: types.hpp:65-70 */
static void inc(uint64_t* cell, uint64_t amount) {
    if (*cell > UINT64_MAX - amount) g_overflow = 1;
    *cell += amount;
}

/* ------------------------------------------------------------------ */
/* graph + indexes: graph.cpp:13-44 (build, (t, ordinal) sort),        */
/* indexes.cpp:7-26 (NodeSequenceIndex), indexes.cpp:28-58 (PairEdge)  */
typedef struct { uint32_t src, dst; int64_t t; uint64_t ord; } orc_edge;
typedef struct { int64_t t; uint64_t ord; uint32_t other; uint8_t dir; } orc_inc;
typedef struct { uint64_t key; int64_t t; uint64_t ord; uint8_t dir_rel_min; } orc_prec;

typedef struct {
    uint64_t n, m;
    orc_edge* edges;   /* (t, ordinal) sorted */
    uint64_t* off;     /* n+1 */
    orc_inc* inc;      /* 2m */
    orc_prec* prec;    /* m, sorted by (key, t, ord) */
} orc_graph;

static int cmp_edge(const void* a, const void* b) {
    const orc_edge* x = a; const orc_edge* y = b;
    if (x->t != y->t) return x->t < y->t ? -1 : 1;
    return x->ord < y->ord ? -1 : (x->ord > y->ord);
}
static int cmp_prec(const void* a, const void* b) {
    const orc_prec* x = a; const orc_prec* y = b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    if (x->t != y->t) return x->t < y->t ? -1 : 1;
    return x->ord < y->ord ? -1 : (x->ord > y->ord);
}

void orc_free(orc_graph* g) {
    if (!g) return;
    free(g->edges); free(g->off); free(g->inc); free(g->prec); free(g);
}

/* Edges given in ingestion order (ordinal = index). NULL on self-loop or
 * out-of-range endpoint (graph.cpp:24-33). */
orc_graph* orc_build(uint64_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                     const int64_t* t) {
    orc_graph* g = calloc(1, sizeof(orc_graph));
    g->n = n; g->m = m;
    g->edges = malloc(sizeof(orc_edge) * (m ? m : 1));
    for (uint64_t i = 0; i < m; ++i) {
        if (src[i] == dst[i] || src[i] >= n || dst[i] >= n) { orc_free(g); return NULL; }
        g->edges[i].src = src[i]; g->edges[i].dst = dst[i];
        g->edges[i].t = t[i]; g->edges[i].ord = i;
    }
    qsort(g->edges, m, sizeof(orc_edge), cmp_edge);

    g->off = calloc(n + 1, sizeof(uint64_t));
    for (uint64_t i = 0; i < m; ++i) { g->off[g->edges[i].src + 1]++; g->off[g->edges[i].dst + 1]++; }
    for (uint64_t u = 1; u <= n; ++u) g->off[u] += g->off[u - 1];
    g->inc = malloc(sizeof(orc_inc) * (2 * m ? 2 * m : 1));
    uint64_t* fill = malloc(sizeof(uint64_t) * (n ? n : 1));
    for (uint64_t u = 0; u < n; ++u) fill[u] = g->off[u];
    for (uint64_t i = 0; i < m; ++i) {
        const orc_edge* e = &g->edges[i];
        orc_inc a = {e->t, e->ord, e->dst, 0};
        orc_inc b = {e->t, e->ord, e->src, 1};
        g->inc[fill[e->src]++] = a;
        g->inc[fill[e->dst]++] = b;
    }
    free(fill);

    g->prec = malloc(sizeof(orc_prec) * (m ? m : 1));
    for (uint64_t i = 0; i < m; ++i) {
        const orc_edge* e = &g->edges[i];
        uint32_t lo = e->src < e->dst ? e->src : e->dst;
        uint32_t hi = e->src < e->dst ? e->dst : e->src;
        g->prec[i].key = ((uint64_t)lo << 32) | hi;
        g->prec[i].t = e->t; g->prec[i].ord = e->ord;
        g->prec[i].dir_rel_min = e->src == lo ? 0 : 1;
    }
    qsort(g->prec, m, sizeof(orc_prec), cmp_prec);
    return g;
}

uint64_t orc_degree(const orc_graph* g, uint32_t u) { return g->off[u + 1] - g->off[u]; }

/* NodeSequenceIndex::sequence (indexes.hpp:28-30) flattened for tests. */
uint64_t orc_sequence(const orc_graph* g, uint32_t u, int64_t* t, uint64_t* ord, uint32_t* other,
                      uint8_t* dir) {
    uint64_t s = orc_degree(g, u);
    for (uint64_t k = 0; k < s; ++k) {
        const orc_inc* r = &g->inc[g->off[u] + k];
        if (t) t[k] = r->t;
        if (ord) ord[k] = r->ord;
        if (other) other[k] = r->other;
        if (dir) dir[k] = r->dir;
    }
    return s;
}

/* PairEdgeIndex::window (indexes.cpp:60-73): records with lo <= t <= hi. */
static void pair_window(const orc_graph* g, uint32_t v, uint32_t w, int64_t lo, int64_t hi,
                        uint64_t* first, uint64_t* last, int* v_is_min) {
    uint32_t a = v < w ? v : w, b = v < w ? w : v;
    uint64_t key = ((uint64_t)a << 32) | b;
    *v_is_min = (v == a);
    /* lower_bound of (key, lo) */
    uint64_t L = 0, R = g->m;
    while (L < R) {
        uint64_t mid = (L + R) / 2;
        const orc_prec* p = &g->prec[mid];
        if (p->key < key || (p->key == key && p->t < lo)) L = mid + 1; else R = mid;
    }
    *first = L;
    R = g->m;
    uint64_t L2 = L;
    while (L2 < R) {
        uint64_t mid = (L2 + R) / 2;
        const orc_prec* p = &g->prec[mid];
        if (p->key < key || (p->key == key && p->t <= hi)) L2 = mid + 1; else R = mid;
    }
    *last = L2;
}

/* edges_in_window (indexes.cpp:75-85) flattened for tests. */
uint64_t orc_pair_window(const orc_graph* g, uint32_t v, uint32_t w, int64_t lo, int64_t hi,
                         int64_t* t, uint64_t* ord, uint8_t* dir_rel_v) {
    uint64_t f, l; int vmin;
    if (lo > hi) return 0;
    pair_window(g, v, w, lo, hi, &f, &l, &vmin);
    for (uint64_t k = f; k < l; ++k) {
        if (t) t[k - f] = g->prec[k].t;
        if (ord) ord[k - f] = g->prec[k].ord;
        if (dir_rel_v) dir_rel_v[k - f] = vmin ? g->prec[k].dir_rel_min : !g->prec[k].dir_rel_min;
    }
    return l - f;
}

/* Degree: graph.cpp:52-59 ; auto_degree_threshold: executor.cpp:15-21 */
static int cmp_desc_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x > y ? -1 : (x < y);
}
uint64_t orc_auto_degree_threshold(const orc_graph* g) {
    if (g->n == 0) return 0;
    uint64_t* d = malloc(sizeof(uint64_t) * g->n);
    for (uint64_t u = 0; u < g->n; ++u) d[u] = orc_degree(g, (uint32_t)u);
    qsort(d, g->n, sizeof(uint64_t), cmp_desc_u64);
    uint64_t r = g->n < 20 ? d[0] : d[19];
    free(d);
    return r;
}

/* ------------------------------------------------------------------ */
/* Counter layouts: motifs.hpp:78-83 (star), 103-106 (pair), 127-131    */
#define STAR_IDX(type, d1, d2, d3) ((((type) * 2 + (d1)) * 2 + (d2)) * 2 + (d3))
#define PAIR_IDX(d1, d2, d3) (((d1) * 2 + (d2)) * 2 + (d3))

/* FAST-Star, Algorithm 1: star_engine.cpp:64-127.  Neighbor count maps are
 * the epoch-stamped slot arrays of star_engine.cpp:14-60. */
int orc_star_pair_at_center(const orc_graph* g, uint32_t u, int64_t delta, uint64_t begin,
                            uint64_t end, uint64_t* star, uint64_t* pair) {
    g_overflow = 0;
    const orc_inc* seq = g->inc + g->off[u];
    uint64_t s = orc_degree(g, u);
    if (s < 3 || end <= begin) return ORC_OK;
    if (end > s - 2) end = s - 2;
    /* dense neighbor slots (slot_of) */
    uint32_t* slot_at = malloc(sizeof(uint32_t) * s);
    uint32_t* nbr_of_slot = malloc(sizeof(uint32_t) * s);
    uint32_t nslots = 0;
    for (uint64_t k = 0; k < s; ++k) {
        uint32_t sl = nslots;
        for (uint32_t q = 0; q < nslots; ++q) if (nbr_of_slot[q] == seq[k].other) { sl = q; break; }
        if (sl == nslots) nbr_of_slot[nslots++] = seq[k].other;
        slot_at[k] = sl;
    }
    uint64_t* cnt[2]; uint32_t* stamp[2];
    for (int d = 0; d < 2; ++d) { cnt[d] = calloc(nslots, 8); stamp[d] = calloc(nslots, 4); }
    uint32_t epoch = 0;
#define GET(d, sl) (stamp[d][sl] == epoch ? cnt[d][sl] : 0)
    for (uint64_t i = begin; i < end; ++i) {
        const orc_inc* first = &seq[i];
        uint32_t fs = slot_at[i];
        int64_t horizon = sat_add(first->t, delta);
        ++epoch;
        uint64_t tot[2] = {0, 0};
        for (uint64_t j = i + 1; j < s; ++j) {
            const orc_inc* third = &seq[j];
            if (third->t > horizon) break;
            uint32_t ts = slot_at[j];
            if (third->other == first->other) {
                uint64_t mid_in = GET(1, fs), mid_out = GET(0, fs);
                inc(&pair[PAIR_IDX(first->dir, 1, third->dir)], mid_in);
                inc(&pair[PAIR_IDX(first->dir, 0, third->dir)], mid_out);
                inc(&star[STAR_IDX(1, first->dir, 1, third->dir)], tot[1] - mid_in);
                inc(&star[STAR_IDX(1, first->dir, 0, third->dir)], tot[0] - mid_out);
            } else {
                inc(&star[STAR_IDX(0, first->dir, 1, third->dir)], GET(1, ts));
                inc(&star[STAR_IDX(0, first->dir, 0, third->dir)], GET(0, ts));
                inc(&star[STAR_IDX(2, first->dir, 1, third->dir)], GET(1, fs));
                inc(&star[STAR_IDX(2, first->dir, 0, third->dir)], GET(0, fs));
            }
            int d = third->dir;
            if (stamp[d][ts] != epoch) { stamp[d][ts] = epoch; cnt[d][ts] = 0; }
            cnt[d][ts]++;
            tot[d]++;
        }
    }
#undef GET
    for (int d = 0; d < 2; ++d) { free(cnt[d]); free(stamp[d]); }
    free(slot_at); free(nbr_of_slot);
    return g_overflow ? ORC_ERR_OVERFLOW : ORC_OK;
}

/* count_star_pair: star_engine.cpp:129-136 */
int orc_count_star_pair(const orc_graph* g, int64_t delta, uint64_t* star, uint64_t* pair) {
    memset(star, 0, 24 * 8); memset(pair, 0, 8 * 8);
    for (uint64_t u = 0; u < g->n; ++u) {
        uint64_t st[24] = {0}, pr[8] = {0};
        uint64_t s = orc_degree(g, (uint32_t)u);
        int rc = orc_star_pair_at_center(g, (uint32_t)u, delta, 0, s >= 3 ? s - 2 : 0, st, pr);
        if (rc) return rc;
        for (int k = 0; k < 24; ++k) inc(&star[k], st[k]);
        for (int k = 0; k < 8; ++k) inc(&pair[k], pr[k]);
        if (g_overflow) return ORC_ERR_OVERFLOW;
    }
    return ORC_OK;
}

/* FAST-Tri, Algorithm 2: triangle_engine.cpp:20-62.  (t, ordinal) total
 * order for boundary ties: triangle_engine.cpp:10-16. */
int orc_triangles_at_center(const orc_graph* g, uint32_t u, int64_t delta, uint64_t begin,
                            uint64_t end, const uint8_t* live, uint64_t* tri) {
    g_overflow = 0;
    const orc_inc* seq = g->inc + g->off[u];
    uint64_t s = orc_degree(g, u);
    if (s < 2 || end <= begin) return ORC_OK;
    if (end > s - 1) end = s - 1;
    for (uint64_t i = begin; i < end; ++i) {
        const orc_inc* ei = &seq[i];
        if (live && !live[ei->other]) continue;
        int64_t horizon = sat_add(ei->t, delta);
        for (uint64_t j = i + 1; j < s; ++j) {
            const orc_inc* ej = &seq[j];
            if (ej->t > horizon) break;
            if (ej->other == ei->other) continue;
            if (live && !live[ej->other]) continue;
            uint64_t f, l; int vmin;
            int64_t lo = sat_sub(ej->t, delta);
            if (lo > horizon) continue;
            pair_window(g, ei->other, ej->other, lo, horizon, &f, &l, &vmin);
            for (uint64_t k = f; k < l; ++k) {
                const orc_prec* r = &g->prec[k];
                int dk = vmin ? r->dir_rel_min : !r->dir_rel_min;
                int type;
                int before = r->t != ei->t ? r->t < ei->t : r->ord < ei->ord;
                int after = r->t != ej->t ? r->t > ej->t : r->ord > ej->ord;
                type = before ? 0 : (after ? 2 : 1);
                inc(&tri[STAR_IDX(type, ei->dir, ej->dir, dk)], 1);
            }
        }
    }
    return g_overflow ? ORC_ERR_OVERFLOW : ORC_OK;
}

/* count_triangles (count_all / removal): triangle_engine.cpp:64-84 */
int orc_count_triangles(const orc_graph* g, int64_t delta, int removal, uint64_t* tri) {
    memset(tri, 0, 24 * 8);
    uint8_t* alive = NULL;
    if (removal) { alive = malloc(g->n ? g->n : 1); memset(alive, 1, g->n); }
    for (uint64_t u = 0; u < g->n; ++u) {
        uint64_t tc[24] = {0};
        uint64_t s = orc_degree(g, (uint32_t)u);
        int rc = orc_triangles_at_center(g, (uint32_t)u, delta, 0, s >= 2 ? s - 1 : 0, alive, tc);
        if (rc) { free(alive); return rc; }
        for (int k = 0; k < 24; ++k) inc(&tri[k], tc[k]);
        if (alive) alive[u] = 0;
    }
    free(alive);
    return g_overflow ? ORC_ERR_OVERFLOW : ORC_OK;
}

/* ------------------------------------------------------------------ */
/* Signatures: motifs.cpp:49-77 (canonical_signature), 85-123 (cell     */
/* maps), 145-194 (universe sorted lexicographically)                  */
typedef struct { char s[9]; } sig_t;
static sig_t g_all[36];
static int g_star_sig[24], g_pair_sig[8], g_tri_sig[24];
static int g_universe_ready = 0;

static sig_t canonical(const uint32_t e[3][2]) {
    uint32_t seen[3]; int distinct = 0; sig_t out;
    for (int k = 0; k < 3; ++k)
        for (int side = 0; side < 2; ++side) {
            uint32_t node = e[k][side]; int lab = -1;
            for (int q = 0; q < distinct; ++q) if (seen[q] == node) lab = q + 1;
            if (lab < 0) { seen[distinct++] = node; lab = distinct; }
            out.s[3 * k + side] = (char)('0' + lab);
        }
    out.s[2] = '|'; out.s[5] = '|'; out.s[8] = 0;
    return out;
}
static void oriented(int d, uint32_t from, uint32_t to, uint32_t out[2]) {
    if (d == 0) { out[0] = from; out[1] = to; } else { out[0] = to; out[1] = from; }
}
static sig_t star_cell_sig(int type, int d1, int d2, int d3) {
    uint32_t e[3][2]; int d[3] = {d1, d2, d3};
    for (int p = 0; p < 3; ++p) oriented(d[p], 0, p == type ? 2 : 1, e[p]);
    return canonical(e);
}
static sig_t pair_cell_sig(int d1, int d2, int d3) {
    uint32_t e[3][2];
    oriented(d1, 0, 1, e[0]); oriented(d2, 0, 1, e[1]); oriented(d3, 0, 1, e[2]);
    return canonical(e);
}
static sig_t tri_cell_sig(int type, int di, int dj, int dk) {
    uint32_t ei[2], ej[2], ek[2], e[3][2];
    oriented(di, 0, 1, ei); oriented(dj, 0, 2, ej); oriented(dk, 1, 2, ek);
    const uint32_t* order[3];
    if (type == 0) { order[0] = ek; order[1] = ei; order[2] = ej; }
    else if (type == 1) { order[0] = ei; order[1] = ek; order[2] = ej; }
    else { order[0] = ei; order[1] = ej; order[2] = ek; }
    for (int k = 0; k < 3; ++k) { e[k][0] = order[k][0]; e[k][1] = order[k][1]; }
    return canonical(e);
}
static int cmp_sig(const void* a, const void* b) { return strcmp(((const sig_t*)a)->s, ((const sig_t*)b)->s); }
static int sig_index(const char* s) {
    for (int k = 0; k < 36; ++k) if (!strcmp(g_all[k].s, s)) return k;
    return -1;
}
static void universe(void) {
    if (g_universe_ready) return;
    sig_t pool[56]; int np = 0;
    for (int c = 0; c < 24; ++c) pool[np++] = star_cell_sig(c >> 3, (c >> 2) & 1, (c >> 1) & 1, c & 1);
    for (int c = 0; c < 8; ++c) pool[np++] = pair_cell_sig(c >> 2, (c >> 1) & 1, c & 1);
    for (int c = 0; c < 24; ++c) pool[np++] = tri_cell_sig(c >> 3, (c >> 2) & 1, (c >> 1) & 1, c & 1);
    qsort(pool, np, sizeof(sig_t), cmp_sig);
    int n = 0;
    for (int k = 0; k < np; ++k) if (n == 0 || strcmp(g_all[n - 1].s, pool[k].s)) g_all[n++] = pool[k];
    for (int c = 0; c < 24; ++c) g_star_sig[c] = sig_index(star_cell_sig(c >> 3, (c >> 2) & 1, (c >> 1) & 1, c & 1).s);
    for (int c = 0; c < 8; ++c) g_pair_sig[c] = sig_index(pair_cell_sig(c >> 2, (c >> 1) & 1, c & 1).s);
    for (int c = 0; c < 24; ++c) g_tri_sig[c] = sig_index(tri_cell_sig(c >> 3, (c >> 2) & 1, (c >> 1) & 1, c & 1).s);
    g_universe_ready = (n == 36);
}

int orc_signature(int idx, char* out) {
    universe();
    if (idx < 0 || idx >= 36) return ORC_ERR_ARG;
    memcpy(out, g_all[idx].s, 9);
    return ORC_OK;
}
/* cell -> signature index maps, for tests */
int orc_cell_signature(int kind, int cell) {
    universe();
    if (kind == 0) return g_star_sig[cell];
    if (kind == 1) return g_pair_sig[cell];
    return g_tri_sig[cell];
}

/* merge_census: motifs.cpp:233-281 */
int orc_merge_census(const uint64_t* star, const uint64_t* pair, const uint64_t* tri, int removal,
                     uint64_t* census) {
    universe();
    g_overflow = 0;
    memset(census, 0, 36 * 8);
    for (int c = 0; c < 24; ++c) inc(&census[g_star_sig[c]], star[c]);
    for (int c = 0; c < 4; ++c) {          /* d1 = outward cells 0..3 */
        uint64_t a = pair[c], b = pair[7 - c];  /* complement flips all three bits */
        if (a != b) return ORC_ERR_CONSISTENCY;
        inc(&census[g_pair_sig[c]], a);
    }
    uint64_t sums[36] = {0};
    for (int c = 0; c < 24; ++c) inc(&sums[g_tri_sig[c]], tri[c]);
    for (int k = 0; k < 36; ++k) {
        int is_tri = 0;
        for (int c = 0; c < 24; ++c) if (g_tri_sig[c] == k) is_tri = 1;
        if (!is_tri) continue;
        if (!removal) {
            if (sums[k] % 3) return ORC_ERR_CONSISTENCY;
            inc(&census[k], sums[k] / 3);
        } else {
            inc(&census[k], sums[k]);
        }
    }
    return g_overflow ? ORC_ERR_OVERFLOW : ORC_OK;
}

/* Brute-force enumeration: oracle.cpp:10-48 (classify, for_each_instance) */
int orc_census_bruteforce(const orc_graph* g, int64_t delta, uint64_t* census) {
    universe();
    g_overflow = 0;
    memset(census, 0, 36 * 8);
    const orc_edge* E = g->edges;
    uint64_t m = g->m;
    for (uint64_t i = 0; i + 2 < m; ++i) {
        int64_t horizon = sat_add(E[i].t, delta);
        for (uint64_t j = i + 1; j + 1 < m; ++j) {
            if (E[j].t > horizon) break;
            for (uint64_t k = j + 1; k < m; ++k) {
                if (E[k].t > horizon) break;
                uint32_t nodes[6] = {E[i].src, E[i].dst, E[j].src, E[j].dst, E[k].src, E[k].dst};
                uint32_t seen[3]; int distinct = 0, ok = 1;
                for (int q = 0; q < 6 && ok; ++q) {
                    int f = 0;
                    for (int z = 0; z < distinct; ++z) if (seen[z] == nodes[q]) f = 1;
                    if (!f) { if (distinct == 3) ok = 0; else seen[distinct++] = nodes[q]; }
                }
                if (!ok) continue;
                uint32_t e[3][2] = {{E[i].src, E[i].dst}, {E[j].src, E[j].dst}, {E[k].src, E[k].dst}};
                sig_t s = canonical(e);
                inc(&census[sig_index(s.s)], 1);
            }
        }
    }
    return g_overflow ? ORC_ERR_OVERFLOW : ORC_OK;
}

/* Brute force restricted to instances whose earliest edge has t < t_end
 * (time-slice partitions of the multi-GPU path); same enumeration as above. */
int orc_census_bruteforce_before(const orc_graph* g, int64_t delta, int64_t t_end, uint64_t* census) {
    universe();
    g_overflow = 0;
    memset(census, 0, 36 * 8);
    const orc_edge* E = g->edges;
    uint64_t m = g->m;
    for (uint64_t i = 0; i + 2 < m; ++i) {
        if (E[i].t >= t_end) break;
        int64_t horizon = sat_add(E[i].t, delta);
        for (uint64_t j = i + 1; j + 1 < m; ++j) {
            if (E[j].t > horizon) break;
            for (uint64_t k = j + 1; k < m; ++k) {
                if (E[k].t > horizon) break;
                uint32_t nodes[6] = {E[i].src, E[i].dst, E[j].src, E[j].dst, E[k].src, E[k].dst};
                uint32_t seen[3]; int distinct = 0, ok = 1;
                for (int q = 0; q < 6 && ok; ++q) {
                    int f = 0;
                    for (int z = 0; z < distinct; ++z) if (seen[z] == nodes[q]) f = 1;
                    if (!f) { if (distinct == 3) ok = 0; else seen[distinct++] = nodes[q]; }
                }
                if (!ok) continue;
                uint32_t e[3][2] = {{E[i].src, E[i].dst}, {E[j].src, E[j].dst}, {E[k].src, E[k].dst}};
                sig_t sg = canonical(e);
                inc(&census[sig_index(sg.s)], 1);
            }
        }
    }
    return g_overflow ? ORC_ERR_OVERFLOW : ORC_OK;
}

/* ------------------------------------------------------------------ */
/* generate_random_graph: graph.cpp:140-168 (mt19937_64, rejection      */
/* sampling bounded draws).  Output in ingestion (ordinal) order.      */
typedef struct { uint64_t mt[312]; int idx; } mt64;
static void mt64_seed(mt64* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}
static uint64_t mt64_next(mt64* r) {
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
static uint64_t bounded(mt64* r, uint64_t bound) {
    if (bound == 0) return 0;
    uint64_t limit = UINT64_MAX - UINT64_MAX % bound, x;
    do { x = mt64_next(r); } while (x >= limit);
    return x % bound;
}
int orc_generate_random_graph(uint64_t nodes, uint64_t m, int64_t t_max, uint64_t seed,
                              uint32_t* src, uint32_t* dst, int64_t* t) {
    if (m > 0 && nodes < 2) return ORC_ERR_ARG;
    if (t_max < 0) return ORC_ERR_ARG;
    mt64 r; mt64_seed(&r, seed);
    for (uint64_t i = 0; i < m; ++i) {
        uint32_t s = (uint32_t)bounded(&r, nodes);
        uint32_t o = (uint32_t)bounded(&r, nodes - 1);
        src[i] = s; dst[i] = o + (o >= s ? 1 : 0);
        t[i] = (int64_t)bounded(&r, (uint64_t)t_max + 1);
    }
    return ORC_OK;
}
