/* oracle.h — CPU restatement of the Flash hot path (TEST INFRASTRUCTURE ONLY;
 * see oracle.c for the reference citations and the usage rule). */
#ifndef FLASHANN_ORACLE_H
#define FLASHANN_ORACLE_H

#include <stdint.h>

typedef struct {
    int64_t dist_comps, sym_comps, kernel_calls, visited;
    int64_t reverse_prunes, reverse_appends;
} or_counters;

/* Same logical layout as the device graph: ids rows of exactly cap int32
 * (-1 beyond the count) and counts; codes n x cs (cs >= m). */
typedef struct {
    int64_t n, nU;
    int m, cs;
    int cap0, capU;
    int32_t *adj0, *cnt0, *adjU, *cntU;
    uint8_t *codes;
    const int32_t *levels;
    const int64_t *uoff;
    const int32_t *upper_owner; /* nU: vertex owning each upper row */
    int tie;                    /* 0: ties by id; 1: by the scrambled id    */
    int expand;                 /* frontier entries expanded per step (<=1: 1) */
    int kind;                   /* 4 Flash (u8 table distances), 0 exact (fp32 L2) */
    const float *vecs;          /* exact: n x dim vectors                    */
    int dim;
} or_graph;

typedef struct {
    int64_t entry_point;
    int32_t max_layer;
    int32_t n_batches;
    or_counters counters;
} or_build_result;

double or_l2sq_f32(const float *a, const float *b, int d);
uint8_t or_quantize(double d, double dmin, double delta);
void or_encode_adt(const float *red, const float *cent, const int32_t *dims, const int32_t *offs,
                   int m, int dmax, double dmin, double delta, uint8_t *code, uint8_t *adt);
void or_batch_lanes(const uint8_t *adt, const uint8_t *codes, int m, int nb, uint8_t *out);
int or_sdt_sum(const uint8_t *sdt, const uint8_t *ca, const uint8_t *cb, int m);
int or_select(const uint8_t *sdt, int m, const uint8_t *codes, int cs, const int32_t *ids,
              const double *d, int n, int cap, int32_t *out, int64_t *sym);
void or_reset(or_graph *g);
int or_layer_search(or_graph *g, const uint8_t *adt, int layer, int entry, int W, int32_t *out_ids,
                    int32_t *out_d, or_counters *c);
/* exact kind: query vector instead of a table; out_d = fp32 distance bits */
int or_layer_search_exact(or_graph *g, const float *qvec, int layer, int entry, int W,
                          int32_t *out_ids, int32_t *out_d, or_counters *c);
int or_hill_climb(or_graph *g, const uint8_t *adt, int layer, int entry, int *out_d,
                  or_counters *c);
int or_schedule(const int32_t *levels, int64_t n, int batch_max, double batch_frac, int seq_prefix,
                int batch_min, int32_t *starts, int32_t *sizes);
int or_build(or_graph *g, const float *proj, int dproj, const float *cent, const int32_t *dims,
             const int32_t *offs, int dmax, double dmin, double delta, const uint8_t *sdt, int C,
             int R, int batch_max, double batch_frac, int seq_prefix, int batch_min,
             or_build_result *res);
int or_search(or_graph *g, const float *vecs, int dim, const float *cent, const int32_t *dims,
              const int32_t *offs, int dmax, double dmin, double delta, int dproj, int entry,
              int max_layer, const float *queries, const float *qproj, int nq, int ef, int k,
              int rerank_depth, int64_t *out_ids, double *out_d, or_counters *c);

#endif
