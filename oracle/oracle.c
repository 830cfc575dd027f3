/*
 * oracle.c — CPU restatement of the reference's Flash hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or as the reported CPU baseline — never as the product
 * path.  The product path (paper_2502_18113_b200) has no CPU fallback.
 *
 * Everything here is restated from the reference's behaviour, citing
 * /root/reference/pkg/src/flashann/... file:line:
 *   or_l2sq_f32      _kernels/_simd.h:44-51 (fp32 tree of the gcc -O3
 *                    -march=native -ffast-math build; pinned by golden vectors)
 *   or_quantize      _kernels/_simd.h:99-107
 *   or_encode_adt    _kernels/_simd.h:211-228
 *   or_batch_lanes   _kernels/_simd.h:111-121 (scalar semantic definition)
 *   or_sdt_sum       _kernels/_simd.h:87-95
 *   or_select        _kernels/_core.pyx:388-408
 *   or_layer_search  _pycore.py:246-283, the reference's semantic core for
 *                    _core.pyx:278-342 (ties by vertex id via tuple order)
 *   or_hill_climb    _kernels/_core.pyx:345-385
 *   or_reverse_add   _kernels/_core.pyx:441-477 (+ fa_sort_pairs :232-247)
 *   or_build         _kernels/_core.pyx:501-536 / :711-764 under the
 *                    deterministic insertion-batch schedule of the GPU build
 *                    (batch size 1 everywhere = the sequential reference)
 *   or_search        _kernels/_core.pyx:784-888
 *   kind 0 (exact)   asym_one / sym_one _core.pyx:167-191: fp32 L2 for every
 *                    distance, the same search / select / reverse rules; keys
 *                    carry the fp32 bit pattern (monotone for d >= 0)
 *
 * Compile: gcc -O2 -ffp-contract=off (explicit fmaf where the tree fuses).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- numerics ------------------------------------------------------------ */

double or_l2sq_f32(const float *a, const float *b, int d) {
    int i = 0;
    float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f, s;
    int have_v = 0;
    if (d >= 8) {
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (; i + 8 <= d; i += 8)
            for (int k = 0; k < 8; ++k) {
                float e = a[i + k] - b[i + k];
                float sq = e * e;
                acc[k] = acc[k] + sq;
            }
        v0 = acc[0] + acc[4];
        v1 = acc[1] + acc[5];
        v2 = acc[2] + acc[6];
        v3 = acc[3] + acc[7];
        have_v = 1;
    }
    if (d - i >= 4) {
        float e0 = a[i] - b[i], e1 = a[i + 1] - b[i + 1];
        float e2 = a[i + 2] - b[i + 2], e3 = a[i + 3] - b[i + 3];
        float w0 = fmaf(e0, e0, v0), w1 = fmaf(e1, e1, v1);
        float w2 = fmaf(e2, e2, v2), w3 = fmaf(e3, e3, v3);
        float t0 = w0 + w2, t1 = w1 + w3;
        s = t0 + t1;
        i += 4;
    } else if (have_v) {
        float t0 = v0 + v2, t1 = v1 + v3;
        s = t0 + t1;
    } else {
        s = 0.f;
    }
    for (; i < d; ++i) {
        float e = a[i] - b[i];
        s = fmaf(e, e, s);
    }
    return (double)s;
}

uint8_t or_quantize(double d, double dmin, double delta) {
    double dmax = dmin + delta;
    if (d >= dmax) return 255;
    if (d < dmin) d = dmin;
    double t = floor((d - dmin) / delta * 255.0);
    if (t >= 255.0) return 255;
    if (t <= 0.0) return 0;
    return (uint8_t)t;
}

void or_encode_adt(const float *red, const float *cent, const int32_t *dims, const int32_t *offs,
                   int m, int dmax, double dmin, double delta, uint8_t *code, uint8_t *adt) {
    for (int i = 0; i < m; ++i) {
        int best = 0;
        double bestd = INFINITY;
        for (int j = 0; j < 16; ++j) {
            double d = or_l2sq_f32(red + offs[i], cent + ((size_t)i * 16 + j) * dmax, dims[i]);
            if (adt) adt[i * 16 + j] = or_quantize(d, dmin, delta);
            if (d < bestd) {
                bestd = d;
                best = j;
            }
        }
        code[i] = (uint8_t)best;
    }
}

void or_batch_lanes(const uint8_t *adt, const uint8_t *codes, int m, int nb, uint8_t *out) {
    for (int b = 0; b < nb; ++b)
        for (int lane = 0; lane < 16; ++lane) {
            uint32_t acc = 0;
            for (int i = 0; i < m; ++i) {
                acc += adt[i * 16 + codes[(size_t)b * m * 16 + i * 16 + lane]];
                if (acc > 255u) acc = 255u;
            }
            out[b * 16 + lane] = (uint8_t)acc;
        }
}

int or_sdt_sum(const uint8_t *sdt, const uint8_t *ca, const uint8_t *cb, int m) {
    uint32_t acc = 0;
    for (int i = 0; i < m; ++i) {
        acc += sdt[((size_t)i * 16 + ca[i]) * 16 + cb[i]];
        if (acc > 255u) acc = 255u;
    }
    return (int)acc;
}

static int adt_sum(const uint8_t *adt, const uint8_t *code, int m) {
    uint32_t acc = 0;
    for (int i = 0; i < m; ++i) {
        acc += adt[i * 16 + code[i]];
        if (acc > 255u) acc = 255u;
    }
    return (int)acc;
}

int or_select(const uint8_t *sdt, int m, const uint8_t *codes, int cs, const int32_t *ids,
              const double *d, int n, int cap, int32_t *out, int64_t *sym) {
    int nk = 0;
    for (int j = 0; j < n && nk < cap; ++j) {
        int v = ids[j], ok = 1;
        for (int t = 0; t < nk; ++t) {
            if (sym) ++*sym;
            if ((double)or_sdt_sum(sdt, codes + (size_t)out[t] * cs, codes + (size_t)v * cs, m) <
                d[j]) {
                ok = 0;
                break;
            }
        }
        if (ok) out[nk++] = v;
    }
    return nk;
}

/* ---- distance context (kind 4 Flash: u8 tables; kind 0 exact: fp32 L2) ---- */

typedef struct {
    const uint8_t *adt; /* Flash: the query's table (m x 16)   */
    const float *vec;   /* exact: the query vector (dim)       */
} qctx;

static uint32_t fbits(double d) {
    float f = (float)d;
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}
static double bits_d(uint32_t u) {
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* distance query -> vertex u, as an order-preserving uint32 */
static uint32_t qdist(const or_graph *g, const qctx *q, int u) {
    if (g->kind == 0) return fbits(or_l2sq_f32(q->vec, g->vecs + (size_t)u * g->dim, g->dim));
    return (uint32_t)adt_sum(q->adt, g->codes + (size_t)u * g->cs, g->m);
}
/* distance vertex a -> vertex b (sym_one) */
static uint32_t pdist(const or_graph *g, const uint8_t *sdt, int a, int b) {
    if (g->kind == 0)
        return fbits(or_l2sq_f32(g->vecs + (size_t)a * g->dim, g->vecs + (size_t)b * g->dim,
                                 g->dim));
    return (uint32_t)or_sdt_sum(sdt, g->codes + (size_t)a * g->cs, g->codes + (size_t)b * g->cs,
                                g->m);
}
static double dist_value(const or_graph *g, uint32_t d) {
    return g->kind == 0 ? bits_d(d) : (double)d;
}

/* select_heur (_core.pyx:388-408) over uint32 distances */
static int select_g(const or_graph *g, const uint8_t *sdt, const int32_t *ids, const uint32_t *d,
                    int n, int cap, int32_t *out, int64_t *sym) {
    int nk = 0;
    for (int j = 0; j < n && nk < cap; ++j) {
        int v = ids[j], ok = 1;
        for (int t = 0; t < nk; ++t) {
            if (sym) ++*sym;
            if (pdist(g, sdt, out[t], v) < d[j]) {
                ok = 0;
                break;
            }
        }
        if (ok) out[nk++] = v;
    }
    return nk;
}

/* ---- graph ---------------------------------------------------------------- */

static int32_t *row_of(or_graph *g, int layer, int v) {
    if (layer == 0) return g->adj0 + (int64_t)v * g->cap0;
    return g->adjU + (g->uoff[v] + layer - 1) * g->capU;
}
static int32_t *cnt_of(or_graph *g, int layer, int v) {
    if (layer == 0) return g->cnt0 + v;
    return g->cntU + (g->uoff[v] + layer - 1);
}

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

typedef struct {
    uint32_t *visited; /* epoch per vertex */
    uint32_t epoch;
    uint64_t *fr;      /* frontier min-heap, key (d << 32 | u)                  */
    uint64_t *rs;      /* result max-heap, key (d << 32 | ~u): top = max d, min u */
    uint64_t *fresh;   /* (d << 32 | u) of one expansion                         */
    size_t fr_cap;
    uint32_t salt;     /* tie-order salt of the current search                   */
} scratch;

static void heap_push_min(uint64_t *h, int *n, uint64_t k) {
    int i = (*n)++;
    h[i] = k;
    while (i > 0) {
        int p = (i - 1) >> 1;
        if (h[p] <= h[i]) break;
        uint64_t t = h[p]; h[p] = h[i]; h[i] = t;
        i = p;
    }
}
static uint64_t heap_pop_min(uint64_t *h, int *n) {
    uint64_t top = h[0];
    int m = --(*n), i = 0;
    h[0] = h[m];
    for (;;) {
        int c = 2 * i + 1;
        if (c >= m) break;
        if (c + 1 < m && h[c + 1] < h[c]) ++c;
        if (h[i] <= h[c]) break;
        uint64_t t = h[i]; h[i] = h[c]; h[c] = t;
        i = c;
    }
    return top;
}
static void heap_push_max(uint64_t *h, int *n, uint64_t k) {
    int i = (*n)++;
    h[i] = k;
    while (i > 0) {
        int p = (i - 1) >> 1;
        if (h[p] >= h[i]) break;
        uint64_t t = h[p]; h[p] = h[i]; h[i] = t;
        i = p;
    }
}
static void heap_pop_max(uint64_t *h, int *n) {
    int m = --(*n), i = 0;
    h[0] = h[m];
    for (;;) {
        int c = 2 * i + 1;
        if (c >= m) break;
        if (c + 1 < m && h[c + 1] > h[c]) ++c;
        if (h[i] >= h[c]) break;
        uint64_t t = h[i]; h[i] = h[c]; h[c] = t;
        i = c;
    }
}
static uint64_t rkey(uint64_t d, uint32_t u) { return (d << 32) | (uint32_t)~u; }

/* Tie order among equal distances: vertex id (tie = 0, the reference's
 * semantic core) or a fixed bijective scramble of the id (tie = 1; a
 * deterministic stand-in for the compiled core's heap-order tie breaks). */
#define TIE_MUL 0x2545F491u
static uint32_t tie_inv(void) {
    uint32_t x = TIE_MUL; /* Newton iteration for the inverse mod 2^32 */
    for (int i = 0; i < 5; ++i) x *= 2u - TIE_MUL * x;
    return x;
}
/* tie = 2 salts the scramble per search (salt = hash of the inserted vertex
 * or query), so different insertions break ties differently, as the compiled
 * core's history-dependent heap order does.  tie = 3 / 4: modes 1 / 2 over
 * 32-bit tie ids (the GPU's wide-id kernels, n >= 2^24). */
static uint32_t tie_mask(int tie) { return tie >= 3 ? 0xffffffffu : 0xffffffu; }
static uint32_t tie_salt(int tie, uint32_t who) {
    return (tie == 2 || tie == 4) ? ((who + 1u) * 0x9E3779B1u) & tie_mask(tie) : 0u;
}
/* tie ids are 24-bit (32-bit) bijections of the vertex id */
static uint32_t tie_fwd(int tie, uint32_t salt, uint32_t u) {
    return tie ? ((u ^ salt) * TIE_MUL) & tie_mask(tie) : u;
}
static uint32_t tie_back(int tie, uint32_t salt, uint32_t t) {
    return tie ? ((t * tie_inv()) & tie_mask(tie)) ^ salt : t;
}

/* Best-first layer search with the semantics of the reference's semantic
 * core (flashann/_pycore.py:246-283): frontier popped in (d, id) order; stop
 * once the result set is full and the popped distance exceeds its worst
 * distance; a block's fresh neighbours are processed in ascending (d, id);
 * accept while the set is not full or d < worst distance (strict), evicting
 * the worst (largest d, smallest id on ties).  Returns |R|; out holds
 * (d << 32 | id) ascending. */
static int layer_search_impl(or_graph *g, scratch *s, const qctx *q, int layer, int entry,
                             uint32_t entry_d, int W, uint64_t *out, or_counters *c) {
    int cap = layer == 0 ? g->cap0 : g->capU;
    s->epoch++;
    if (s->epoch == 0) {
        memset(s->visited, 0, sizeof(uint32_t) * g->n);
        s->epoch = 1;
    }
    uint32_t ep = s->epoch;
    const int tie = g->tie;
    s->visited[entry] = ep;
    int nf = 0, nr = 0;
    heap_push_min(s->fr, &nf, ((uint64_t)entry_d << 32) | tie_fwd(tie, s->salt, (uint32_t)entry));
    heap_push_max(s->rs, &nr, rkey((uint64_t)entry_d, tie_fwd(tie, s->salt, (uint32_t)entry)));
    /* E > 1: pop up to E poppable frontier entries per step and expand them
     * together (a beam-search variant used for batched construction; E = 1 is
     * exactly the semantic core).  Poppable = d <= worst once the set is full. */
    const int E = g->expand > 1 ? g->expand : 1;
    while (nf > 0) {
        int pops[64];
        int npop = 0;
        while (npop < E && nf > 0) {
            uint64_t d = s->fr[0] >> 32;
            if (nr >= W && d > (s->rs[0] >> 32)) break;
            uint64_t top = heap_pop_min(s->fr, &nf);
            pops[npop++] = (int)tie_back(tie, s->salt, (uint32_t)top);
        }
        if (npop == 0) break;
        int nfresh = 0;
        for (int pi = 0; pi < npop; ++pi) {
            int v = pops[pi];
            if (c) c->visited++;
            int32_t *ids = row_of(g, layer, v);
            int cnt = *cnt_of(g, layer, v);
            if (cnt > cap) cnt = cap;
            if (c) c->kernel_calls += (cnt + 15) >> 4;
            for (int j = 0; j < cnt; ++j) {
                int u = ids[j];
                if (u < 0 || s->visited[u] == ep) continue;
                s->visited[u] = ep;
                uint64_t du = (uint64_t)qdist(g, q, u);
                s->fresh[nfresh++] = (du << 32) | tie_fwd(tie, s->salt, (uint32_t)u);
            }
        }
        if (c) c->dist_comps += nfresh;
        qsort(s->fresh, (size_t)nfresh, sizeof(uint64_t), cmp_u64);
        for (int j = 0; j < nfresh; ++j) {
            uint64_t du = s->fresh[j] >> 32;
            uint32_t u = (uint32_t)s->fresh[j];
            if (nr < W) {
                heap_push_max(s->rs, &nr, rkey(du, u));
            } else if (du < (s->rs[0] >> 32)) {
                heap_pop_max(s->rs, &nr);
                heap_push_max(s->rs, &nr, rkey(du, u));
            } else {
                break;  /* sorted: every later candidate is rejected too */
            }
            if ((size_t)nf >= s->fr_cap) return -1;
            heap_push_min(s->fr, &nf, s->fresh[j]);
        }
    }
    for (int i = 0; i < nr; ++i) {
        uint64_t k = s->rs[i];
        out[i] = (k & 0xffffffff00000000ull) | (uint32_t)~(uint32_t)k;
    }
    qsort(out, (size_t)nr, sizeof(uint64_t), cmp_u64);  /* (d, tie key) ascending */
    for (int i = 0; i < nr; ++i)
        out[i] = (out[i] & 0xffffffff00000000ull) | tie_back(tie, s->salt, (uint32_t)out[i]);
    return nr;
}

static void hill_climb_impl(or_graph *g, const qctx *q, int layer, int *cur, uint32_t *curd,
                            or_counters *c) {
    int cap = layer == 0 ? g->cap0 : g->capU;
    int improved = 1;
    while (improved) {
        improved = 0;
        int32_t *ids = row_of(g, layer, *cur);
        int cnt = *cnt_of(g, layer, *cur);
        if (cnt > cap) cnt = cap;
        if (c) c->kernel_calls += (cnt + 15) >> 4;
        int bu = -1;
        uint32_t bd = 0;
        for (int j = 0; j < cnt; ++j) {
            int u = ids[j];
            if (u < 0) continue;
            uint32_t du = qdist(g, q, u);
            if (c) c->dist_comps++;
            if (bu < 0 || du < bd) {
                bd = du;
                bu = u;
            }
        }
        if (bu >= 0 && bd < *curd) {
            *curd = bd;
            *cur = bu;
            improved = 1;
        }
    }
}

static int scratch_init(scratch *s, int64_t n, int W, int capmax) {
    s->visited = (uint32_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint32_t));
    s->fr_cap = (size_t)(n > 0 ? n : 1) + 2;  /* each vertex is pushed at most once */
    s->fr = (uint64_t *)malloc(sizeof(uint64_t) * s->fr_cap);
    s->rs = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(W + 2));
    s->fresh = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(64 * capmax + 8));
    s->epoch = 0;
    s->salt = 0;
    return (s->visited && s->fr && s->rs && s->fresh) ? 0 : -1;
}
static void scratch_free(scratch *s) {
    free(s->visited);
    free(s->fr);
    free(s->rs);
    free(s->fresh);
}

static int layer_search_q(or_graph *g, const qctx *q, int layer, int entry, int W,
                          int32_t *out_ids, int32_t *out_d, or_counters *c) {
    scratch s;
    int capmax = g->cap0 > g->capU ? g->cap0 : g->capU;
    if (scratch_init(&s, g->n, W, capmax)) return -1;
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(W + 1));
    uint32_t ed = qdist(g, q, entry);
    if (c) c->dist_comps++;
    int ts = layer_search_impl(g, &s, q, layer, entry, ed, W, keys, c);
    for (int i = 0; i < ts; ++i) {
        out_ids[i] = (int32_t)(keys[i] & 0xffffffffu);
        out_d[i] = (int32_t)(keys[i] >> 32);
    }
    free(keys);
    scratch_free(&s);
    return ts;
}

int or_layer_search(or_graph *g, const uint8_t *adt, int layer, int entry, int W, int32_t *out_ids,
                    int32_t *out_d, or_counters *c) {
    qctx q = {adt, NULL};
    return layer_search_q(g, &q, layer, entry, W, out_ids, out_d, c);
}

int or_layer_search_exact(or_graph *g, const float *qvec, int layer, int entry, int W,
                          int32_t *out_ids, int32_t *out_d, or_counters *c) {
    qctx q = {NULL, qvec};
    return layer_search_q(g, &q, layer, entry, W, out_ids, out_d, c);
}

int or_hill_climb(or_graph *g, const uint8_t *adt, int layer, int entry, int *out_d,
                  or_counters *c) {
    qctx q = {adt, NULL};
    int cur = entry;
    uint32_t curd = qdist(g, &q, entry);
    hill_climb_impl(g, &q, layer, &cur, &curd, c);
    if (out_d) *out_d = (int)curd;
    return cur;
}

/* reverse_add (_core.pyx:441-477) */
static void reverse_add(or_graph *g, const uint8_t *sdt, int y, int x, int layer, uint64_t *pairs,
                        int32_t *cid, uint32_t *cd, int32_t *sel, or_counters *c) {
    int cap = layer == 0 ? g->cap0 : g->capU;
    int32_t *ids = row_of(g, layer, y);
    int32_t *cntp = cnt_of(g, layer, y);
    int cnt = *cntp;
    if (cnt < cap) {
        ids[cnt] = x;
        *cntp = cnt + 1;
        if (c) c->reverse_appends++;
        return;
    }
    if (c) c->reverse_prunes++;
    for (int j = 0; j <= cnt; ++j) {
        int u = j < cnt ? ids[j] : x;
        uint64_t d = (uint64_t)pdist(g, sdt, y, u);
        pairs[j] = (d << 32) | (uint32_t)u; /* (d, id) order == fa_pair_cmp */
    }
    if (c) c->sym_comps += cnt + 1;
    qsort(pairs, (size_t)cnt + 1, sizeof(uint64_t), cmp_u64);
    for (int j = 0; j <= cnt; ++j) {
        cid[j] = (int32_t)(pairs[j] & 0xffffffffu);
        cd[j] = (uint32_t)(pairs[j] >> 32);
    }
    int nk = select_g(g, sdt, cid, cd, cnt + 1, cap, sel, c ? &c->sym_comps : NULL);
    for (int j = 0; j < cap; ++j) ids[j] = j < nk ? sel[j] : -1;
    *cntp = nk;
}

void or_reset(or_graph *g) {
    for (int64_t i = 0; i < g->n * g->cap0; ++i) g->adj0[i] = -1;
    for (int64_t i = 0; i < g->nU * g->capU; ++i) g->adjU[i] = -1;
    memset(g->cnt0, 0, sizeof(int32_t) * (size_t)g->n);
    if (g->nU) memset(g->cntU, 0, sizeof(int32_t) * (size_t)g->nU);
}

int or_schedule(const int32_t *levels, int64_t n, int batch_max, double batch_frac, int seq_prefix,
                int batch_min, int32_t *starts, int32_t *sizes) {
    if (n <= 1) return 0;
    /* batch_min < 0: auto, clamp(n / 256, 1, 4096) (the GPU build's rule) */
    if (batch_min < 0) batch_min = n / 256 < 1 ? 1 : (n / 256 > 4096 ? 4096 : (int)(n / 256));
    int ml = levels[0], nb = 0;
    int64_t x = 1;
    while (x < n) {
        int B;
        if (levels[x] > ml) B = 1;
        else if (x < seq_prefix) B = 1;
        else {
            double f = batch_frac * (double)x;
            B = (int)f;
            int bm = x < batch_min ? (int)x : batch_min;
            if (B < bm) B = bm;
            if (B > batch_max) B = batch_max;
            if (B < 1) B = 1;
        }
        int size = 0;
        starts[nb] = (int32_t)x;
        while (size < B && x < n) {
            int lv = levels[x];
            if (size > 0 && lv > ml) break;
            ++size;
            ++x;
            if (lv > ml) break;
        }
        sizes[nb] = size;
        int last = starts[nb] + size - 1;
        if (levels[last] > ml) ml = levels[last];
        ++nb;
    }
    return nb;
}

typedef struct {
    uint64_t key; /* row << 32 | x */
} req_t;

int or_build(or_graph *g, const float *proj, int dproj, const float *cent, const int32_t *dims,
             const int32_t *offs, int dmax, double dmin, double delta, const uint8_t *sdt, int C,
             int R, int batch_max, double batch_frac, int seq_prefix, int batch_min,
             or_build_result *res) {
    memset(res, 0, sizeof(*res));
    res->entry_point = -1;
    res->max_layer = -1;
    or_reset(g);
    if (g->n == 0) return 0;
    int m = g->m;
    const int exact = g->kind == 0;
    /* Flash: codes are the fp32-tree codes (prep_qctx overwrite,
     * _core.pyx:493-498); exact: proj holds the vectors themselves */
    int capmax = g->cap0 > g->capU ? g->cap0 : g->capU;
    if (!exact)
        for (int64_t v = 0; v < g->n; ++v)
            or_encode_adt(proj + (size_t)v * dproj, cent, dims, offs, m, dmax, dmin, delta,
                          g->codes + (size_t)v * g->cs, NULL);
    int32_t *starts = (int32_t *)malloc(sizeof(int32_t) * (size_t)g->n);
    int32_t *sizes = (int32_t *)malloc(sizeof(int32_t) * (size_t)g->n);
    int nb = or_schedule(g->levels, g->n, batch_max, batch_frac, seq_prefix, batch_min, starts,
                         sizes);
    int maxB = 1;
    for (int b = 0; b < nb; ++b)
        if (sizes[b] > maxB) maxB = sizes[b];
    /* per-thread workspaces: the searches of one batch read only the graph as
     * of the batch start (no vertex of the batch is reachable before the
     * reverse phase) and write only their own rows, so they run in parallel;
     * the requests are sorted afterwards, so the result is thread-count
     * independent */
    int nth = 1;
#ifdef _OPENMP
    nth = omp_get_max_threads();
#endif
    if (nth < 1) nth = 1;
    int maxlev = 0;
    for (int64_t v = 0; v < g->n; ++v)
        if (g->levels[v] > maxlev) maxlev = g->levels[v];
    size_t reqcap = (size_t)maxB * (size_t)(maxlev + 1) * (size_t)R + 1;
    uint64_t *req = (uint64_t *)malloc(sizeof(uint64_t) * reqcap);
    size_t *heads = (size_t *)malloc(sizeof(size_t) * reqcap);
    int32_t *cid = (int32_t *)malloc(sizeof(int32_t) * (size_t)(C + capmax + 2));
    uint32_t *cd = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(C + capmax + 2));
    int32_t *sel = (int32_t *)malloc(sizeof(int32_t) * (size_t)(C + capmax + 2));
    uint64_t *pairs = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(capmax + 2));
    int failed = 0;
    int ep = 0, ml = g->levels[0];
    or_counters *c = &res->counters;
    for (int b = 0; b < nb; ++b) {
        size_t nreq = 0;
        const int bep = ep, bml = ml;
        const int bsize = sizes[b], bstart = starts[b];
#pragma omp parallel num_threads(bsize > 64 ? nth : 1) reduction(|| : failed)
        {
            scratch s;
            or_counters lc;
            memset(&lc, 0, sizeof(lc));
            uint8_t *adt = (uint8_t *)malloc((size_t)(m > 0 ? m : 1) * 16);
            uint64_t *T = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(C + 1));
            int32_t *tid_ = (int32_t *)malloc(sizeof(int32_t) * (size_t)(C + capmax + 2));
            uint32_t *td = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(C + capmax + 2));
            int32_t *tsel = (int32_t *)malloc(sizeof(int32_t) * (size_t)(C + capmax + 2));
            if (scratch_init(&s, g->n, C, capmax) || !adt || !T || !tid_ || !td || !tsel) {
                failed = 1;
            } else {
#pragma omp for schedule(dynamic, 16)
                for (int p = 0; p < bsize; ++p) {
                    int x = bstart + p;
                    int level = g->levels[x];
                    qctx q = {adt, proj + (size_t)x * dproj};
                    if (!exact) {
                        uint8_t code_tmp[256];
                        or_encode_adt(proj + (size_t)x * dproj, cent, dims, offs, m, dmax, dmin,
                                      delta, code_tmp, adt);
                    }
                    int cur = bep;
                    uint32_t curd = qdist(g, &q, cur);
                    lc.dist_comps++;
                    for (int layer = bml; layer > level; --layer)
                        hill_climb_impl(g, &q, layer, &cur, &curd, &lc);
                    int top = bml < level ? bml : level;
                    for (int layer = top; layer >= 0; --layer) {
                        s.salt = tie_salt(g->tie, (uint32_t)x);
                        int ts = layer_search_impl(g, &s, &q, layer, cur, curd, C, T, &lc);
                        for (int j = 0; j < ts; ++j) {
                            tid_[j] = (int32_t)(T[j] & 0xffffffffu);
                            td[j] = (uint32_t)(T[j] >> 32);
                        }
                        int nsel = select_g(g, sdt, tid_, td, ts, R, tsel, &lc.sym_comps);
                        int cap = layer == 0 ? g->cap0 : g->capU;
                        int32_t *row = row_of(g, layer, x);
                        for (int j = 0; j < cap; ++j) row[j] = j < nsel ? tsel[j] : -1;
                        *cnt_of(g, layer, x) = nsel;
                        size_t pos;
#pragma omp atomic capture
                        { pos = nreq; nreq += (size_t)nsel; }
                        for (int j = 0; j < nsel; ++j) {
                            int y = tsel[j];
                            uint64_t rowg = layer == 0 ? (uint64_t)y
                                                       : (uint64_t)(g->n + g->uoff[y] + layer - 1);
                            req[pos + j] = (rowg << 32) | (uint32_t)x;
                        }
                        cur = (int)(T[0] & 0xffffffffu);
                        curd = (uint32_t)(T[0] >> 32);
                    }
                }
            }
#pragma omp critical
            {
                c->dist_comps += lc.dist_comps;
                c->sym_comps += lc.sym_comps;
                c->kernel_calls += lc.kernel_calls;
                c->visited += lc.visited;
            }
            scratch_free(&s);
            free(adt); free(T); free(tid_); free(td); free(tsel);
        }
        if (failed) break;
        for (int p = 0; p < bsize; ++p) {
            int level = g->levels[bstart + p];
            if (level > ml) {
                ep = bstart + p;
                ml = level;
            }
        }
        /* reverse edges grouped by row, ascending x (the sequential order) */
        qsort(req, nreq, sizeof(uint64_t), cmp_u64);
        /* rows are independent (a reverse update reads the immutable codes and
         * writes only its own row): groups of one row run in parallel, each in
         * ascending x */
        size_t ng = 0;
        for (size_t t = 0; t < nreq; ++t)
            if (t == 0 || (req[t] >> 32) != (req[t - 1] >> 32)) heads[ng++] = t;
        heads[ng] = nreq;
#pragma omp parallel num_threads(ng > 256 ? nth : 1)
        {
            or_counters lc;
            memset(&lc, 0, sizeof(lc));
            uint64_t *tp = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(capmax + 2));
            int32_t *tid_ = (int32_t *)malloc(sizeof(int32_t) * (size_t)(C + capmax + 2));
            uint32_t *td = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(C + capmax + 2));
            int32_t *tsel = (int32_t *)malloc(sizeof(int32_t) * (size_t)(C + capmax + 2));
#pragma omp for schedule(dynamic, 64)
            for (size_t gi = 0; gi < ng; ++gi) {
                for (size_t t = heads[gi]; t < heads[gi + 1]; ++t) {
                    uint64_t rowg = req[t] >> 32;
                    int x = (int)(req[t] & 0xffffffffu);
                    int layer, y;
                    if ((int64_t)rowg < g->n) {
                        layer = 0;
                        y = (int)rowg;
                    } else {
                        int64_t r = (int64_t)rowg - g->n;
                        y = g->upper_owner[r];
                        layer = (int)(r - g->uoff[y]) + 1;
                    }
                    reverse_add(g, sdt, y, x, layer, tp, tid_, td, tsel, &lc);
                }
            }
#pragma omp critical
            {
                c->sym_comps += lc.sym_comps;
                c->reverse_prunes += lc.reverse_prunes;
                c->reverse_appends += lc.reverse_appends;
            }
            free(tp); free(tid_); free(td); free(tsel);
        }
    }
    res->entry_point = ep;
    res->max_layer = ml;
    res->n_batches = nb;
    free(starts); free(sizes); free(cid); free(cd); free(sel);
    free(pairs); free(req); free(heads);
    return failed ? -1 : 0;
}

int or_search(or_graph *g, const float *vecs, int dim, const float *cent, const int32_t *dims,
              const int32_t *offs, int dmax, double dmin, double delta, int dproj, int entry,
              int max_layer, const float *queries, const float *qproj, int nq, int ef, int k,
              int rerank_depth, int64_t *out_ids, double *out_d, or_counters *c) {
    int m = g->m;
    int capmax = g->cap0 > g->capU ? g->cap0 : g->capU;
    typedef struct {
        double d;
        int32_t id;
    } pair;
    int failed = 0;
    /* queries are independent: one workspace per thread */
#pragma omp parallel reduction(|| : failed)
    {
    scratch s;
    or_counters lc;
    memset(&lc, 0, sizeof(lc));
    uint8_t *adt = (uint8_t *)malloc((size_t)(m > 0 ? m : 1) * 16);
    uint8_t code[256];
    uint64_t *T = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(ef + 1));
    pair *pr = (pair *)malloc(sizeof(pair) * (size_t)(ef + 1));
    if (scratch_init(&s, g->n, ef, capmax) || !adt || !T || !pr) failed = 1;
#pragma omp for schedule(dynamic, 8)
    for (int q = 0; q < nq; ++q) {
        if (failed) continue;
        qctx qc = {adt, queries + (size_t)q * dim};
        if (g->kind != 0)
            or_encode_adt(qproj + (size_t)q * dproj, cent, dims, offs, m, dmax, dmin, delta, code,
                          adt);
        int cur = entry;
        uint32_t curd = qdist(g, &qc, cur);
        lc.dist_comps++;
        for (int layer = max_layer; layer > 0; --layer)
            hill_climb_impl(g, &qc, layer, &cur, &curd, &lc);
        s.salt = tie_salt(g->tie, (uint32_t)q);
        int ts = layer_search_impl(g, &s, &qc, 0, cur, curd, ef, T, &lc);
        int64_t *oi = out_ids + (size_t)q * k;
        double *od = out_d + (size_t)q * k;
        if (rerank_depth > 0) {
            int rr = rerank_depth < ts ? rerank_depth : ts;
            for (int j = 0; j < rr; ++j) {
                int id = (int)(T[j] & 0xffffffffu);
                pr[j].d = or_l2sq_f32(queries + (size_t)q * dim, vecs + (size_t)id * dim, dim);
                pr[j].id = id;
            }
            /* insertion sort by (d, id) (fa_pair_cmp) */
            for (int a = 1; a < rr; ++a) {
                pair t = pr[a];
                int b = a - 1;
                while (b >= 0 && (pr[b].d > t.d || (pr[b].d == t.d && pr[b].id > t.id))) {
                    pr[b + 1] = pr[b];
                    --b;
                }
                pr[b + 1] = t;
            }
            for (int j = 0; j < k; ++j) {
                oi[j] = j < rr ? pr[j].id : -1;
                od[j] = j < rr ? pr[j].d : INFINITY;
            }
        } else {
            for (int j = 0; j < k; ++j) {
                oi[j] = j < ts ? (int64_t)(T[j] & 0xffffffffu) : -1;
                od[j] = j < ts ? dist_value(g, (uint32_t)(T[j] >> 32)) : INFINITY;
            }
        }
    }
    if (c) {
#pragma omp critical
        {
            c->dist_comps += lc.dist_comps;
            c->sym_comps += lc.sym_comps;
            c->kernel_calls += lc.kernel_calls;
            c->visited += lc.visited;
        }
    }
    free(adt); free(T); free(pr);
    scratch_free(&s);
    }
    return failed ? -1 : 0;
}
