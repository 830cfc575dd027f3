/*
 * flashann_b200.h — C-ABI of the B200-native Flash HNSW-construction core.
 *
 * This is the drop-in boundary for the reference's "core module" contract
 * (flashann/core.py:16-26; the compiled core flashann/_kernels/_core.pyx).
 * Every entry point returns an int status (FA_OK = 0, negative on error) and
 * leaves a human-readable message in fa_last_error() (thread-local).  No
 * torch types cross this boundary: plain pointers, sizes and cudaStream_t
 * (passed as void*, NULL = legacy default stream).
 *
 * Pointer conventions
 *   - functions with the suffix _dev take DEVICE pointers and are
 *     stream-ordered (asynchronous; the caller synchronises);
 *   - functions with the suffix _host take HOST pointers (numpy buffers in the
 *     Python shim), stage H2D/D2H internally and return after the stream has
 *     synchronised, exactly like the reference's blocking Cython calls.
 *
 * Reference file:line anchors are relative to /root/reference/pkg/src/.
 */
#ifndef FLASHANN_B200_H
#define FLASHANN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------- */
#define FA_OK 0
#define FA_EINVAL -1   /* invalid argument (reference: ValueError/TypeError)   */
#define FA_ENOMEM -2   /* allocation failure (reference: MemoryError)          */
#define FA_ECUDA -3    /* CUDA runtime / launch failure                         */
#define FA_EOVERFLOW -4/* a fixed-capacity device structure overflowed          */
#define FA_EEMPTY -5   /* search on an empty graph (_core.pyx:821-822)          */

#define FA_KIND_FLASH 4 /* providers/base.py:23-29 KIND_IDS["flash"]             */

const char *fa_last_error(void);
int fa_version(void);

/* ---- table kernels (reference: flashann/_kernels/_simd.h) --------------- */

/* fa_batch_lanes over ncases independent cases (_core.pyx:977-994
 * flash_batch_distance_many; _simd.h:111-121 semantic definition).
 * adts: ncases x m x 16 u8, codes: ncases x m x 16 u8 -> out ncases x 16 u8. */
int fa_scan_cases_dev(const uint8_t *adts, const uint8_t *codes, int m, int64_t ncases,
                      uint8_t *out, void *stream);

/* nb consecutive 16-slot batches of one block (_core.pyx:997-1006
 * flash_batch_blocks; _simd.h:180-197 fa_batch_lanes).
 * adt: m x 16, codes: nb x m x 16 -> out nb*16.                              */
int fa_scan_blocks_dev(const uint8_t *adt, const uint8_t *codes, int m, int nb, uint8_t *out,
                       void *stream);

/* Standalone block scan (SURVEY §8(d) "standalone scan benchmark"): nq query
 * tables adt (nq x m x 16), each scanning nsel blocks of the padded device
 * block array (blocks, block_stride bytes per block: int32 count | pad |
 * int32 ids[cap] | codes nb x m x 16 at codes_off).  out[q] = min over the
 * live slots of (dist << 32 | neighbour id) — a running (d, id) minimum, no
 * per-lane writes.  sel: nq x nsel block indices.                                                            */
int fa_scan_select_dev(const uint8_t *adt, int nq, const uint8_t *blocks, int64_t nblocks,
                       int64_t block_stride, int64_t codes_off, int cap, int m,
                       const int32_t *sel, int nsel, uint64_t *out, void *stream);

/* Same scan with the blocks staged by 1-D TMA bulk copies (cp.async.bulk)
 * into a 2-deep shared-memory ring per warp; identical results.              */
int fa_scan_select_tma_dev(const uint8_t *adt, int nq, const uint8_t *blocks, int64_t nblocks,
                           int64_t block_stride, int64_t codes_off, int cap, int m,
                           const int32_t *sel, int nsel, uint64_t *out, void *stream);

/* fa_quantize (_simd.h:99-107) elementwise in IEEE double.                   */
int fa_quantize_dev(const double *d, int64_t n, double dist_min, double delta, uint8_t *out,
                    void *stream);

/* fa_l2sq_f32 (_simd.h:44-51) with the reference build's fp32 operation tree
 * (gcc -O3 -march=native -ffast-math), row-wise: out[i] = l2(a_i, b_i).
 * b_stride = 0 broadcasts one b row.                                          */
int fa_l2sq_rows_dev(const float *a, int64_t a_stride, const float *b, int64_t b_stride,
                     int64_t n, int d, double *out, void *stream);

/* fa_flash_encode_adt (_simd.h:211-228) for n rows of the reduced (projected)
 * matrix: codes_out n x code_stride (first m bytes written, rest zeroed up to
 * code_stride), adt_out (nullable) n x adt_rows x 16 (rows >= m zeroed).      */
int fa_encode_adt_dev(const float *red, int64_t n, int64_t red_stride, const float *cent,
                      const int32_t *dims, const int32_t *offs, int m, int dmax, double dist_min,
                      double delta, uint8_t *codes_out, int code_stride, uint8_t *adt_out,
                      int adt_rows, void *stream);

/* fa_sdt_sum_sat (_simd.h:87-95): out[i] = min(sum_s sdt[s][a_i[s]][b_i[s]],255)
 * for npairs pairs of code rows (row strides in bytes).                       */
int fa_sdt_sum_dev(const uint8_t *sdt, int m, const uint8_t *a, int64_t a_stride,
                   const uint8_t *b, int64_t b_stride, int64_t npairs, int32_t *out,
                   void *stream);

/* select_heur (_core.pyx:388-408) with Flash SDT distances, candidates given in
 * order; codes n x code_stride.  out: up to cap ids, *nout (device int).      */
int fa_select_dev(const uint8_t *sdt, int m, const uint8_t *codes, int code_stride,
                  const int32_t *cand_ids, const double *cand_d, int ncand, int cap,
                  int32_t *out, int32_t *nout, void *stream);

/* select_heur (_core.pyx:388-408) of the exact kind (kind 0; sym_one of
 * K_EXACT, _core.pyx:179-191): candidate v is kept iff every kept u has
 * (double) fa_l2sq_f32(u, v) >= cand_d[v]; vecs n x dim device f32.          */
int fa_select_exact_dev(const float *vecs, int dim, const int32_t *cand_ids,
                        const double *cand_d, int ncand, int cap, int32_t *out, int32_t *nout,
                        void *stream);

/* ---- coder training (flashann/kmeans.py, flashann/flash.py:63-107) ------- */

/* State of numpy's PCG64 bit generator (Generator.bit_generator.state). */
typedef struct {
    unsigned long long s_hi, s_lo, inc_hi, inc_lo;
    unsigned int has_uint32, uinteger;
} fa_pcg64_state;

/* k-means subsamples on the host: sel[i] = np.sort(rng_i.permutation(ns)[:cap])
 * for rng_i = default_rng(seed + i) given as its PCG64 state (kmeans.py:50-54);
 * states are advanced exactly as numpy advances them.  Host pointers; runs
 * the m subspaces on parallel threads; needs no device.                      */
int fa_kmeans_subsample(int64_t ns, int cap, int m, void *states, int32_t *sel);

/* Scratch bytes needed by fa_kmeans_subspaces_dev.                           */
size_t fa_kmeans_scratch_bytes(int m, int nsub);

/* kmeans(sub_i, 16, iters, seed+i) for every subspace i at once (one CTA per
 * subspace; kmeans.py:35-76).  xs: ns x ld f32 projected sample; sel: m x nsub
 * subsample rows (NULL = all rows, nsub = ns); states[i]: the PCG64 state of
 * default_rng(seed+i) after the host-drawn permutation.  cent_out m x 16 x
 * dmax f32 (zero padded), hist_out m x (iters+1) f64 inertia history.        */
int fa_kmeans_subspaces_dev(const float *xs, int64_t ns, int ld, const int32_t *dims,
                            const int32_t *offs, int m, const int32_t *sel, int nsub,
                            const void *states, int iters, float *cent_out, int dmax,
                            double *hist_out, void *scratch, void *stream);

/* Range statistics of flash_train (flash.py:86-98): raw_sdt m x 16 x 16 f64
 * (direct differences), range_out[0] = dist_min, range_out[1] = dist_max
 * (sum of per-subspace maxima).  scratch: >= 3*m*8 bytes.                    */
int fa_flash_range_dev(const float *xs, int64_t ns, int ld, const int32_t *dims,
                       const int32_t *offs, int m, const float *cent, int dmax, double *raw_sdt,
                       double *range_out, void *scratch, void *stream);

/* ---- PCA contractions on the tensor cores (providers/pca.py) ------------- */

#define FA_DTYPE_F32 0
#define FA_DTYPE_BF16 1

/* cov = (X - mean)^T (X - mean) / n as float64 (D x D, symmetric), X n x D
 * device rows of f32 or bf16 (x_dtype), mean D f32 (the reference's
 * float32-cast mean; pca.py:35-38).  3xTF32 tcgen05 GEMM, split over rows,
 * partials summed in float64 in a fixed order (deterministic).              */
int fa_pca_cov_dev(const void *x, int x_dtype, int64_t n, int D, const float *mean,
                   double *cov, void *stream);

/* out[i, j] = sum_k (X[i, k] - mean[k]) * basis[k, j] for j < d (pca.py:68-71
 * pca_project_all), X n x D f32 or bf16, basis D x dfull f32 row-major (the
 * rotation, columns by descending eigenvalue), out n x ldo f32.  3xTF32
 * tcgen05 GEMM fed by TMA; fp32-class accuracy.                              */
int fa_pca_project_dev(const void *x, int x_dtype, int64_t n, int D, const float *mean,
                       const float *basis, int dfull, int d, float *out, int64_t ldo,
                       void *stream);

/* pca_project (pca.py:57-65) of n vectors in float64: out[i, j] = sum_k
 * (x[i, k] - mean[k]) * basis[k, j], j < d; basis D x dfull row-major.       */
int fa_pca_project_f64_dev(const double *x, int64_t n, int D, const double *mean,
                           const double *basis, int dfull, int d, double *out, void *stream);

/* ---- graph index (build + search) --------------------------------------- */

typedef struct fa_index fa_index; /* opaque, device resident */

typedef struct {
    int64_t n;            /* vertices                                            */
    int m;                /* subspaces                                           */
    int R;                /* upper cap R, base cap 2R (_core.pyx:607-608)        */
    int dim;              /* original dimension (rerank), 0 if vecs absent       */
    int dproj;            /* reduced width d_F                                   */
    int dmax;             /* centroid padding width                              */
    double dist_min, delta;
    /* DEVICE pointers, borrowed for the index lifetime */
    const float *vecs;    /* n x dim f32 (nullable: no rerank)                   */
    const float *proj;    /* n x dproj f32 (nullable when codes are given)       */
    const float *cent;    /* m x 16 x dmax f32                                   */
    const int32_t *dims;  /* m                                                   */
    const int32_t *offs;  /* m                                                   */
    const uint8_t *sdt;   /* m x 16 x 16                                         */
    const int32_t *levels;/* n                                                   */
    const int64_t *uoff;  /* n, -1 when level 0 (graph.py:90-96)                 */
    int64_t n_upper_rows; /* sum(levels)                                         */
} fa_index_desc;

typedef struct {
    int C;                /* efConstruction width                                */
    int batch_max;        /* largest insertion batch (0 = default)               */
    double batch_frac;    /* batch <= frac * |inserted| (0 = default)            */
    int seq_prefix;       /* first vertices inserted one per batch (-1 default)  */
    int hash_log2;        /* shared visited table: 2^hash_log2 16-bit slots per
                             warp, >= 2^12 stored (0 = auto; 9..11 use only
                             2^hash_log2 / 512 slots per bucket)            */
    int profile;          /* 1: time every kernel class with CUDA events        */
    int tie;              /* order among equal distances in the searches:
                             0 vertex id (reference semantic core, _pycore.py),
                             1 fixed id scramble, 2 scramble salted per
                             inserted vertex (default of the Python layer)     */
    int expand;           /* frontier entries expanded per search step during
                             insertion (<= 1: one, the semantic core; max 8)  */
    int64_t *point_stats; /* optional DEVICE n x 8 per inserted vertex
                             (diagnostics): expansions, SM cycles, cycles in
                             pop / row+visited / distances / acceptance (0
                             unless built with FA_PHASE_PROFILE=1),
                             forward-selection cycles, distance evaluations   */
    int batch_min;        /* batches of at least min(inserted, batch_min) while
                             frac * inserted is smaller (fills the GPU sooner);
                             < 0 = auto: clamp(n / 256, 1, 4096); 0 = off    */
    int64_t start, end;   /* insert vertices [start, end) (end 0 = n).  start 0
                             resets the graph; start > 0 resumes a graph whose
                             vertices [0, start) were inserted by earlier
                             calls (the dynamic-rebuild workload: batches onto
                             an existing graph).  Batches never straddle
                             start or end.                                    */
} fa_build_opts;

typedef struct {
    int64_t entry_point;
    int32_t max_layer;
    int32_t n_batches;
    int64_t dist_comps, sym_comps, kernel_calls, visited; /* _core.pyx:695-704 */
    int64_t reverse_prunes, reverse_appends;
    int64_t reverse_full_prunes; /* prunes that could not take the fast path    */
    int64_t launches;     /* kernels of this library launched by the build      */
    double ms_encode, ms_search, ms_sort, ms_reverse; /* profile = 1 only       */
} fa_build_result;

/* Allocate the device graph (adjacency rows, counts, code table) for desc.   */
int fa_index_create(const fa_index_desc *desc, fa_index **out);
int fa_index_destroy(fa_index *idx);

/* Encode every vector (codes = fa_flash_encode_adt of proj rows), exactly as
 * the compiled core's prep_qctx overwrites codes[x] (_core.pyx:493-498).     */
int fa_index_encode(fa_index *idx, void *stream);
/* Use caller-provided device codes (n x m) instead of encoding.              */
int fa_index_set_codes(fa_index *idx, const uint8_t *codes, int code_stride, void *stream);

/* Batched insertion of all n vertices (reference build_graph,
 * _core.pyx:711-764): blocking; fills *res.                                   */
int fa_index_build(fa_index *idx, const fa_build_opts *opts, fa_build_result *res,
                   void *stream);

/* Query search (reference search_batch, _core.pyx:817-888).  qproj nq x dproj
 * device (reduced queries), queries nq x dim device (only for rerank).
 * out_ids nq x k int64 (-1 pad), out_d nq x k f64 (+inf pad).  counters[4]
 * (host) receives dist_comps, sym_comps, kernel_calls, visited.              */
int fa_index_search(fa_index *idx, const float *queries, const float *qproj, int nq, int ef,
                    int k, int rerank_depth, int64_t entry, int max_layer, int64_t *out_ids,
                    double *out_d, int64_t *counters, void *stream);

/* Tie order (fa_build_opts.tie modes) used by fa_index_search and
 * fa_index_search_layer; 0 (vertex id) by default.                            */
int fa_index_set_search_tie(fa_index *idx, int mode);

/* Single-layer candidate search from a given entry (greedy_search_layer,
 * _core.pyx:891-939) for nq queries; out_ids/out_d nq x width, out_n nq.     */
int fa_index_search_layer(fa_index *idx, const float *qproj, int nq, const int64_t *entries,
                          int width, int layer, int32_t *out_ids, double *out_d,
                          int32_t *out_n, int64_t *counters, void *stream);

/* Reference layout <-> device layout (flashann/layout.py:1-45).  The block
 * pointers are DEVICE pointers with the reference row strides.              */
int fa_index_export_blocks(fa_index *idx, uint8_t *base_blocks, int64_t base_stride,
                           uint8_t *upper_blocks, int64_t upper_stride, void *stream);
/* (count, ids) rows of every layer-0 / upper row: rows x (1 + cap) int32,
 * ids -1 beyond the count (device pointers; upper_rows may be NULL when the
 * graph has no upper rows).                                                  */
int fa_index_export_rows(fa_index *idx, int32_t *base_rows, int32_t *upper_rows, void *stream);
/* Reference blocks (layout.py:1-45) from (count, ids) rows and the n x m code
 * table, on the host cores (host pointers; no device needed).               */
int fa_assemble_blocks(uint8_t *blocks, int64_t rows, int64_t stride, int cap, int m,
                       const int32_t *id_rows, const uint8_t *codes, int64_t ncodes);
int fa_index_import_blocks(fa_index *idx, const uint8_t *base_blocks, int64_t base_stride,
                           const uint8_t *upper_blocks, int64_t upper_stride, void *stream);
/* Device code table (n x code_stride u8) of the index, for export.           */
const uint8_t *fa_index_codes(fa_index *idx, int *code_stride);
/* Raw device adjacency (for tests): ids rows and counts of a layer.         */
int fa_index_adjacency(fa_index *idx, int layer_kind, const int32_t **ids, const int32_t **cnt,
                       int *cap, int64_t *rows);

/* ---- host-pointer drop-ins (the reference core's Cython signatures) ------ */

/* build_graph(kind=4, prov, levels, base_blocks, upper_offsets, upper_blocks,
 * C, R, threads, kernel) (_core.pyx:711-764).  All pointers HOST; codes and
 * the two block arrays are mutated in place like the reference.             */
int fa_build_graph_host(int64_t n, int dim, const float *vecs, int dproj, const float *proj,
                        uint8_t *codes, int m, const float *cent, int dmax,
                        const int32_t *dims, const int32_t *offs, const uint8_t *sdt,
                        double dist_min, double delta, const int32_t *levels,
                        uint8_t *base_blocks, int64_t base_stride, const int64_t *uoff,
                        uint8_t *upper_blocks, int64_t n_upper_rows, int64_t upper_stride,
                        int C, int R, const fa_build_opts *opts, fa_build_result *res);

/* search_batch (_core.pyx:817-888) over reference-layout host blocks.       */
int fa_search_batch_host(int64_t n, int dim, const float *vecs, int dproj, const uint8_t *codes,
                         int m, const float *cent, int dmax, const int32_t *dims,
                         const int32_t *offs, const uint8_t *sdt, double dist_min, double delta,
                         const int32_t *levels, const uint8_t *base_blocks, int64_t base_stride,
                         const int64_t *uoff, const uint8_t *upper_blocks, int64_t n_upper_rows,
                         int64_t upper_stride, int R, int64_t entry, int max_layer,
                         const float *queries, const float *qproj, int nq, int ef, int k,
                         int rerank_depth, int64_t *out_ids, double *out_d, int64_t *counters);

/* The exact strategy (kind 0; asym_one / sym_one of K_EXACT, _core.pyx:
 * 167-191): every distance is the fp32 L2 of the vectors (fa_l2sq_f32 tree),
 * blocks carry no code region (code_subspaces = 0).  A device index created
 * with m = 0 (and vecs, dim) is an exact-kind index; these are its host
 * drop-ins for build_graph / search_batch with kind 0.  C, ef <= 512.        */
int fa_build_graph_exact_host(int64_t n, int dim, const float *vecs, const int32_t *levels,
                              uint8_t *base_blocks, int64_t base_stride, const int64_t *uoff,
                              uint8_t *upper_blocks, int64_t n_upper_rows, int64_t upper_stride,
                              int C, int R, const fa_build_opts *opts, fa_build_result *res);

int fa_search_batch_exact_host(int64_t n, int dim, const float *vecs, const int32_t *levels,
                               const uint8_t *base_blocks, int64_t base_stride,
                               const int64_t *uoff, const uint8_t *upper_blocks,
                               int64_t n_upper_rows, int64_t upper_stride, int R, int64_t entry,
                               int max_layer, const float *queries, int nq, int ef, int k,
                               int rerank_depth, int64_t *out_ids, double *out_d,
                               int64_t *counters);

#ifdef __cplusplus
}
#endif
#endif /* FLASHANN_B200_H */
