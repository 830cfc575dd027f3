// Query search kernels: search with exact rerank (search_batch) and the
// single-layer hook (greedy_search_layer); the build search is build_search.cu.
#include "kernels.cuh"

namespace fa {

// distance of a key in the caller's units: the u8 sum (Flash) or the fp32 L2
template <typename P>
__device__ __forceinline__ double key_value(unsigned long long k) {
    if constexpr (P::kExact) return (double)__uint_as_float(key_d(k));
    else return (double)key_d(k);
}

// the query context in the warp's ADT region: the query's table (Flash, from
// ctx rows of mpad x 16) or its vector (exact, from ctx rows of dim floats)
template <typename P>
__device__ __forceinline__ void load_query_ctx(const Graph &g, uint8_t *dst,
                                               const uint8_t *__restrict__ ctx, int q, int lane) {
    if constexpr (P::kExact) {
        const float *src = reinterpret_cast<const float *>(ctx) + (size_t)q * g.dim;
        float *qv = reinterpret_cast<float *>(dst);
        for (int i = lane; i < g.dim; i += 32) qv[i] = __ldg(src + i);
    } else {
        load_adt_smem(dst, ctx + (size_t)q * g.mpad * 16, g.mpad, lane);
    }
}

// search_one (_core.pyx:784-814): descent on layers ml..1, layer-0 search of
// width ef, optional exact rerank of the first rerank_depth results with
// (d, id) ordering (fa_sort_pairs), then the first k.
template <typename P, int J>
__global__ void __launch_bounds__(kSearchWarps * 32, 4) query_search_kernel(
    Graph g, const uint8_t *__restrict__ adt_q, int nq, int ep, int ml, int ef, int k,
    int rerank_depth, const float *__restrict__ vecs, int dim, const float *__restrict__ queries,
    WarpLayout L, int64_t *__restrict__ out_ids, double *__restrict__ out_d,
    unsigned long long *__restrict__ ctr, int *err) {
    extern __shared__ __align__(256) uint8_t smem[];
    const int lane = lane_id();
    const int wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;  // warps per CTA (fewer for wide searches)
    const int q = blockIdx.x * nw + wid;
    if (q >= nq) return;
    WarpWS ws(smem, wid, nw, L);
    const TieOrder to = TieOrder::make(g.tie, (uint32_t)q, P::kWide);
    load_query_ctx<P>(g, ws.adt, P::kExact ? reinterpret_cast<const uint8_t *>(queries) : adt_q,
                      q, lane);
    __syncwarp();
    SearchCounters cnt = {};
    int cur = ep;
    uint32_t curd = P::one(g, ws.adt, ep, lane);
    cnt.dist += 1;
    for (int layer = ml; layer > 0; --layer)
        hill_climb<P>(g, layer, cur, curd, ws.adt, ws.fresh, ws.fdist, cnt, lane);
    int ts = 0;
    GSlot gs = gslot_claim(g, lane);
    bool ok = layer_search<P, J, 1>(g, 0, cur, curd, ef, ws.adt, ws.T, ts, ws.S, ws.TQ, ws.fresh, ws.fdist,
                           ws.H, L.hash_log2, cnt, to, gs, lane);
    gslot_release(gs, lane);
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
            float s = warp_l2_group8(j < rr ? qv : nullptr, vv, dim, lane);
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
                od[j] = key_value<P>(ws.T[j]);
            } else {
                oid[j] = -1;
                od[j] = __longlong_as_double(0x7ff0000000000000ll);
            }
        }
    }
    flush_counters(cnt, ctr, lane);
}

// greedy_search_layer (_core.pyx:891-939): one layer from a given entry.
template <typename P, int J>
__global__ void __launch_bounds__(kSearchWarps * 32, 4) layer_search_kernel(
    Graph g, const uint8_t *__restrict__ adt_q, int nq, const int64_t *__restrict__ entries,
    int width, int layer, WarpLayout L, int32_t *__restrict__ out_ids, double *__restrict__ out_d,
    int32_t *__restrict__ out_n, unsigned long long *__restrict__ ctr, int *err) {
    extern __shared__ __align__(256) uint8_t smem[];
    const int lane = lane_id();
    const int wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;  // warps per CTA (fewer for wide searches)
    const int q = blockIdx.x * nw + wid;
    if (q >= nq) return;
    WarpWS ws(smem, wid, nw, L);
    const TieOrder to = TieOrder::make(g.tie, (uint32_t)q, P::kWide);
    load_query_ctx<P>(g, ws.adt, adt_q, q, lane);
    __syncwarp();
    SearchCounters cnt = {};
    const int entry = (int)entries[q];
    uint32_t d0 = P::one(g, ws.adt, entry, lane);
    cnt.dist += 1;
    int ts = 0;
    GSlot gs = gslot_claim(g, lane);
    bool ok = layer_search<P, J, 1>(g, layer, entry, d0, width, ws.adt, ws.T, ts, ws.S, ws.TQ, ws.fresh,
                           ws.fdist, ws.H, L.hash_log2, cnt, to, gs, lane);
    gslot_release(gs, lane);
    if (!ok) {
        if (lane == 0) atomicExch(err, 1);
        ts = 0;
    }
    for (int j = lane; j < width; j += 32) {
        out_ids[(size_t)q * width + j] = j < ts ? to.back((uint32_t)key_id(ws.T[j])) : -1;
        out_d[(size_t)q * width + j] = j < ts ? key_value<P>(ws.T[j]) : 0.0;
    }
    if (lane == 0) out_n[q] = ts;
    flush_counters(cnt, ctr, lane);
}

#define FA_VARIANTS(K, P)                \
    switch (set_variant(W)) {             \
        case 2: return K<P, 2>;           \
        case 4: return K<P, 4>;           \
        case 7: return K<P, 7>;           \
        case 8: return K<P, 8>;           \
        case 10: return K<P, 10>;         \
        case 16: return K<P, 16>;         \
        default: break;                   \
    }

QuerySearchFn query_search_variant(int W, bool exact, bool wide) {
    if (exact) {
        if (wide) {
            FA_VARIANTS(query_search_kernel, ExactDistW)
            return query_search_kernel<ExactDistW, 0>;
        }
        FA_VARIANTS(query_search_kernel, ExactDist)
        return query_search_kernel<ExactDist, 0>;
    }
    if (wide) {
        FA_VARIANTS(query_search_kernel, FlashDistW)
        return query_search_kernel<FlashDistW, 0>;
    }
    FA_VARIANTS(query_search_kernel, FlashDist)
    return query_search_kernel<FlashDist, 0>;
}

LayerSearchFn layer_search_variant(int W, bool exact, bool wide) {
    if (exact) {
        if (wide) {
            FA_VARIANTS(layer_search_kernel, ExactDistW)
            return layer_search_kernel<ExactDistW, 0>;
        }
        FA_VARIANTS(layer_search_kernel, ExactDist)
        return layer_search_kernel<ExactDist, 0>;
    }
    if (wide) {
        FA_VARIANTS(layer_search_kernel, FlashDistW)
        return layer_search_kernel<FlashDistW, 0>;
    }
    FA_VARIANTS(layer_search_kernel, FlashDist)
    return layer_search_kernel<FlashDist, 0>;
}
#undef FA_VARIANTS

}  // namespace fa
