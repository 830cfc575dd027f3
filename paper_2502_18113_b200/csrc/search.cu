// Query search kernels: search with exact rerank (search_batch) and the
// single-layer hook (greedy_search_layer); the build search is build_search.cu.
#include "kernels.cuh"

namespace fa {

// Warp-cooperative fp32 L2 (fa_l2sq_f32 tree, common.cuh l2_tree) of four
// (query, vector) pairs at once: lane group g = lane/8 handles pair g and lane
// k = lane%8 owns accumulator k of the 8-wide main loop.
__device__ __forceinline__ float warp_l2_group(const float *q, const float *v, int d, int lane) {
    const int k = lane & 7;
    int nfull = d >= 8 ? d / 8 : 0;
    float acc = 0.f;
    if (q && v)
        for (int c = 0; c < nfull; ++c) {
            float e = __fsub_rn(__ldg(q + 8 * c + k), __ldg(v + 8 * c + k));
            acc = __fadd_rn(acc, __fmul_rn(e, e));
        }
    const unsigned full = 0xffffffffu;
    float hi = __shfl_down_sync(full, acc, 4);
    float vk = (k < 4) ? __fadd_rn(acc, hi) : 0.f;  // v[k] = acc[k] + acc[k+4]
    int i = 8 * nfull;
    bool four = (d - i) >= 4;
    float wk = vk;
    if (four && k < 4 && q && v) {
        float e = __fsub_rn(__ldg(q + i + k), __ldg(v + i + k));
        wk = __fmaf_rn(e, e, vk);
    }
    float w2 = __shfl_down_sync(full, wk, 2);
    float t = __fadd_rn(wk, w2);  // lane0: w0+w2, lane1: w1+w3
    float t1 = __shfl_down_sync(full, t, 1);
    float s = __fadd_rn(t, t1);   // lane k==0: (w0+w2)+(w1+w3)
    if (!four && nfull == 0) s = 0.f;
    if (four) i += 4;
    if (k == 0 && q && v)
        for (; i < d; ++i) {
            float e = __fsub_rn(__ldg(q + i), __ldg(v + i));
            s = __fmaf_rn(e, e, s);
        }
    return s;  // valid in lane k == 0 of the group
}

// search_one (_core.pyx:784-814): descent on layers ml..1, layer-0 search of
// width ef, optional exact rerank of the first rerank_depth results with
// (d, id) ordering (fa_sort_pairs), then the first k.
template <int J>
__global__ void __launch_bounds__(kSearchWarps * 32, 4) query_search_kernel(
    Graph g, const uint8_t *__restrict__ adt_q, int nq, int ep, int ml, int ef, int k,
    int rerank_depth, const float *__restrict__ vecs, int dim, const float *__restrict__ queries,
    WarpLayout L, int64_t *__restrict__ out_ids, double *__restrict__ out_d,
    unsigned long long *__restrict__ ctr, int *err) {
    extern __shared__ __align__(256) uint8_t smem[];
    const int lane = lane_id();
    const int wid = threadIdx.x >> 5;
    const int q = blockIdx.x * kSearchWarps + wid;
    if (q >= nq) return;
    WarpWS ws(smem, wid, kSearchWarps, L);
    const TieOrder to = TieOrder::make(g.tie, (uint32_t)q);
    load_adt_smem(ws.adt, adt_q + (size_t)q * g.mpad * 16, g.mpad, lane);
    __syncwarp();
    SearchCounters cnt = {};
    int cur = ep;
    uint32_t curd = adt_one(ws.adt, g.codes + (size_t)ep * g.mpad, g.mpad, lane);
    cnt.dist += 1;
    for (int layer = ml; layer > 0; --layer)
        hill_climb(g, layer, cur, curd, ws.adt, ws.fresh, ws.fdist, cnt, lane);
    int ts = 0;
    bool ok = layer_search<J, 1>(g, 0, cur, curd, ef, ws.adt, ws.T, ts, ws.S, ws.TQ, ws.fresh, ws.fdist,
                           ws.H, L.hash_log2, cnt, to, lane);
    int64_t *oid = out_ids + (size_t)q * k;
    double *od = out_d + (size_t)q * k;
    if (!ok) {
        if (lane == 0) atomicExch(err, 1);
        flush_counters(cnt, ctr, lane);
        return;
    }
    if (rerank_depth > 0) {
        const int rr = min(rerank_depth, ts);
        // exact distances (the visited hash is dead after the search)
        double *dd = reinterpret_cast<double *>(ws.H);
        const float *qv = queries + (size_t)q * dim;
        for (int base = 0; base < rr; base += 4) {
            int j = base + (lane >> 3);
            const float *vv =
                j < rr ? vecs + (size_t)to.back((uint32_t)key_id(ws.T[j])) * dim : nullptr;
            float s = warp_l2_group(j < rr ? qv : nullptr, vv, dim, lane);
            if ((lane & 7) == 0 && j < rr) dd[j] = (double)s;
        }
        __syncwarp();
        // rank sort by (d, id) (fa_pair_cmp, _simd.h:237-243)
        for (int j = lane; j < rr; j += 32) {
            double dj = dd[j];
            int idj = to.back((uint32_t)key_id(ws.T[j]));
            int rank = 0;
            for (int t = 0; t < rr; ++t) {
                double dt = dd[t];
                int idt = to.back((uint32_t)key_id(ws.T[t]));
                rank += (dt < dj) || (dt == dj && idt < idj);
            }
            if (rank < k) {
                oid[rank] = idj;
                od[rank] = dj;
            }
        }
        for (int j = rr + lane; j < k; j += 32) {
            oid[j] = -1;
            od[j] = __longlong_as_double(0x7ff0000000000000ll);
        }
    } else {
        for (int j = lane; j < k; j += 32) {
            if (j < ts) {
                oid[j] = to.back((uint32_t)key_id(ws.T[j]));
                od[j] = (double)key_d(ws.T[j]);
            } else {
                oid[j] = -1;
                od[j] = __longlong_as_double(0x7ff0000000000000ll);
            }
        }
    }
    flush_counters(cnt, ctr, lane);
}

// greedy_search_layer (_core.pyx:891-939): one layer from a given entry.
template <int J>
__global__ void __launch_bounds__(kSearchWarps * 32, 4) layer_search_kernel(
    Graph g, const uint8_t *__restrict__ adt_q, int nq, const int64_t *__restrict__ entries,
    int width, int layer, WarpLayout L, int32_t *__restrict__ out_ids, double *__restrict__ out_d,
    int32_t *__restrict__ out_n, unsigned long long *__restrict__ ctr, int *err) {
    extern __shared__ __align__(256) uint8_t smem[];
    const int lane = lane_id();
    const int wid = threadIdx.x >> 5;
    const int q = blockIdx.x * kSearchWarps + wid;
    if (q >= nq) return;
    WarpWS ws(smem, wid, kSearchWarps, L);
    const TieOrder to = TieOrder::make(g.tie, (uint32_t)q);
    load_adt_smem(ws.adt, adt_q + (size_t)q * g.mpad * 16, g.mpad, lane);
    __syncwarp();
    SearchCounters cnt = {};
    const int entry = (int)entries[q];
    uint32_t d0 = adt_one(ws.adt, g.codes + (size_t)entry * g.mpad, g.mpad, lane);
    cnt.dist += 1;
    int ts = 0;
    bool ok = layer_search<J, 1>(g, layer, entry, d0, width, ws.adt, ws.T, ts, ws.S, ws.TQ, ws.fresh,
                           ws.fdist, ws.H, L.hash_log2, cnt, to, lane);
    if (!ok) {
        if (lane == 0) atomicExch(err, 1);
        ts = 0;
    }
    for (int j = lane; j < width; j += 32) {
        out_ids[(size_t)q * width + j] = j < ts ? to.back((uint32_t)key_id(ws.T[j])) : -1;
        out_d[(size_t)q * width + j] = j < ts ? (double)key_d(ws.T[j]) : 0.0;
    }
    if (lane == 0) out_n[q] = ts;
    flush_counters(cnt, ctr, lane);
}

QuerySearchFn query_search_variant(int W) {
    switch (set_variant(W)) {
        case 2: return query_search_kernel<2>;
        case 4: return query_search_kernel<4>;
        case 7: return query_search_kernel<7>;
        case 8: return query_search_kernel<8>;
        case 10: return query_search_kernel<10>;
        case 16: return query_search_kernel<16>;
        default: return query_search_kernel<0>;
    }
}

LayerSearchFn layer_search_variant(int W) {
    switch (set_variant(W)) {
        case 2: return layer_search_kernel<2>;
        case 4: return layer_search_kernel<4>;
        case 7: return layer_search_kernel<7>;
        case 8: return layer_search_kernel<8>;
        case 10: return layer_search_kernel<10>;
        case 16: return layer_search_kernel<16>;
        default: return layer_search_kernel<0>;
    }
}

}  // namespace fa
