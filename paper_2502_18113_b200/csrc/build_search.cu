// K4+K5: the batched-insertion search kernel (one warp per inserted vertex),
// instantiated per result-set variant and expansion width.
#include "kernels.cuh"

namespace fa {

// One warp inserts one vertex of the batch: descent, per-layer beam search of
// width C, forward selection (cap R), forward row write, reverse requests.
// Mirrors insert_one (_core.pyx:501-536) against the graph as of batch start.
// P = FlashDist: the per-insertion query tables come in adt_batch and forward
// selection uses the SDT (sdtT); P = ExactDist: the query is the inserted
// vertex's own vector and every distance is fp32 L2.
template <typename P, int J, int EM, int RC>
__global__ void __maxnreg__(96) build_search_kernel(
    Graph g, const uint8_t *__restrict__ sdtT, const uint8_t *__restrict__ adt_batch, int start,
    int size, int ep, int ml, int C, int R, WarpLayout L, const int64_t *__restrict__ req_off,
    const int32_t *__restrict__ order, unsigned long long *__restrict__ req, unsigned long long *__restrict__ ctr, int *err,
    int64_t *__restrict__ stats, int *__restrict__ work, const int *__restrict__ start_v,
    const uint32_t *__restrict__ start_d) {
    // sdtT: the transposed SDT in global memory (L1-resident; keeping it out of
    // shared memory leaves room for one more CTA per SM)
    extern __shared__ __align__(256) uint8_t smem[];
    const int lane = lane_id();
    const int wid = threadIdx.x >> 5;
    WarpWS ws(smem, wid, blockDim.x >> 5, L);  // fewer warps per CTA for wide searches
    CounterTotals total;
    GSlot gs = gslot_claim(g, lane);  // this warp's global visited table, for the launch
    // persistent warps pull vertices from the batch; a slow search never holds
    // its CTA siblings' slots idle
    for (;;) {
        int p = 0;
        if (lane == 0) p = atomicAdd(work, 1);
        p = __shfl_sync(0xffffffffu, p, 0);
        if (p >= size) break;
        // the batch's vertices in the host's processing order (upper-layer
        // vertices, the longest searches, first: a shorter tail)
        const int q = __ldg(order + p);
        const int x = start + q;
        const long long t_begin = clock64();
        const TieOrder to = TieOrder::make(g.tie, (uint32_t)x, P::kWide);
        __syncwarp();
        if constexpr (P::kExact) {
            float *qv = reinterpret_cast<float *>(ws.adt);
            for (int i = lane; i < g.dim; i += 32) qv[i] = __ldg(g.vecs + (size_t)x * g.dim + i);
        } else {
            load_adt_smem(ws.adt, adt_batch + (size_t)q * g.mpad * 16, g.mpad, lane);
        }
        __syncwarp();
        SearchCounters cnt = {};
        const int level = __ldg(g.levels + x);
        int cur = ep;
        uint32_t curd;
        if (start_v) {  // the descent ran in batch_descend_kernel
            cur = __ldg(start_v + q);
            curd = __ldg(start_d + q);
        } else {
            curd = P::one(g, ws.adt, ep, lane);
            cnt.dist += 1;
            for (int layer = ml; layer > level; --layer)
                hill_climb<P>(g, layer, cur, curd, ws.adt, ws.fresh, ws.fdist, cnt, lane);
        }
        const int top = min(ml, level);
        unsigned long long *myreq = req + __ldg(req_off + q);
        long long sel_cycles = 0;
        for (int layer = top; layer >= 0; --layer) {
            int ts = 0;
            bool ok = layer_search<P, J, EM, RC, 9>(g, layer, cur, curd, C, ws.adt, ws.T, ts, ws.S, ws.TQ, ws.fresh,
                                   ws.fdist, ws.H, L.hash_log2, cnt, to, gs, lane);
            if (!ok) {
                if (lane == 0) atomicExch(err, 1);
                for (int l = layer; l >= 0; --l)
                    for (int j = lane; j < R; j += 32) myreq[(size_t)(top - l) * R + j] = KEY_MAX;
                break;
            }
            unsigned long long sym = 0;
            const unsigned long long *T = ws.T;
            const long long t_sel = clock64();
            int32_t *kept;
            int nsel;
            if constexpr (P::kExact) {
                // kept ids, their distances to the candidate, the candidate's
                // vector: the start of the (dead) visited table
                kept = reinterpret_cast<int32_t *>(ws.H);
                uint32_t *kd = reinterpret_cast<uint32_t *>(ws.H) + round_up(R, 4);
                float *cv = reinterpret_cast<float *>(kd + round_up(R, 4));
                nsel = warp_select_exact(
                    g, ts, R,
                    [&](int j, int &v, uint32_t &dv) {
                        unsigned long long k = T[j];
                        v = to.back((uint32_t)key_id(k));
                        dv = key_d(k);
                    },
                    kept, cv, kd, lane, &sym);
            } else {
                nsel = warp_select_tv(
                    sdtT, g.m, g.mpad, g.codes, g.mpad, ts, R,
                    [&](int j, int &v, uint32_t &dv) {
                        unsigned long long k = T[j];
                        v = to.back((uint32_t)key_id(k));
                        dv = key_d(k);
                    },
                    reinterpret_cast<uint8_t *>(ws.H), lane, &sym, kept);
            }
            cnt.sym += sym;
            sel_cycles += clock64() - t_sel;
            // forward row of x (write_forward, _core.pyx:424-438); rows past the
            // live count keep -1 so readers need only the id row
            int32_t *row = const_cast<int32_t *>(row_ids(g, layer, x));
            const int cap = layer_cap(g, layer);
            for (int j = lane; j < cap; j += 32) row[j] = j < nsel ? kept[j] : -1;
            if (lane == 0) {
                if (layer == 0) {
                    g.cnt0[x] = nsel;
                    g.cons0[x] = 0;
                } else {
                    int64_t r = __ldg(g.uoff + x) + layer - 1;
                    g.cntU[r] = nsel;
                    g.consU[r] = 0;
                }
            }
            // reverse requests (row << 32 | x), counted per target row; the
            // batch's touched rows are listed for the bucketing (reverse.cu)
            unsigned long long *lreq = myreq + (size_t)(top - layer) * R;
            for (int j0 = 0; j0 < R; j0 += 32) {
                const int j = j0 + lane;
                unsigned long long key = KEY_MAX;
                bool first = false;
                int64_t rg = 0;
                if (j < nsel) {
                    rg = row_global(g, layer, kept[j]);
                    key = ((unsigned long long)rg << 32) | (uint32_t)x;
                    first = atomicAdd(g.rowcnt + rg, 1) == 0;
                }
                if (j < R) lreq[j] = key;
                const unsigned fb = __ballot_sync(0xffffffffu, first);
                if (fb) {
                    int tb = 0;
                    if (lane == 0) tb = atomicAdd(g.ntouched, __popc(fb));
                    tb = __shfl_sync(0xffffffffu, tb, 0);
                    if (first) g.touched[tb + __popc(fb & ((1u << lane) - 1u))] = (int32_t)rg;
                }
            }
            cur = to.back((uint32_t)key_id(ws.T[0]));
            curd = key_d(ws.T[0]);
            __syncwarp();
        }
        if (stats && lane == 0) {
            int64_t *st = stats + 8 * (int64_t)x;
            st[0] = (int64_t)cnt.visited;
            st[1] = clock64() - t_begin;
#if FA_PHASE_PROFILE
            for (int k = 0; k < 4; ++k) st[2 + k] = (int64_t)cnt.ph[k];
#endif
            st[6] = sel_cycles;
            st[7] = (int64_t)cnt.dist;
        }
        total.add(cnt);
    }
    gslot_release(gs, lane);
    flush_counters(total, ctr, lane);
}

// The batch's greedy descents (hill_climb through the layers above each
// vertex's level, _core.pyx:345-385, from the batch's entry point), ahead of
// the beam searches: their end points and distances seed build_search_kernel,
// and the distance orders the batch.  The length of a vertex's layer-0 search
// correlates with how far its descent ends from it (0.64 at config 2), so
// processing the far ones first leaves a shorter tail of long searches at the
// end of the batch (a simulated 5.7 % off the makespan of the 65,536-vertex
// batches).  Any processing order builds the same graph.  hist gets the
// count of every (level, distance) key, key_of below.
__device__ __forceinline__ int descend_key(int level, int maxlv, uint32_t d) {
    return (maxlv - min(level, maxlv)) * 256 + (255 - (int)min(d, 255u));
}

template <typename P>
__global__ void __launch_bounds__(kSearchWarps * 32) batch_descend_kernel(
    Graph g, const uint8_t *__restrict__ adt_batch, int start, int size, int ep, int ml,
    int maxlv, int ctx_bytes, int cand, int *__restrict__ start_v, uint32_t *__restrict__ start_d,
    int *__restrict__ hist, unsigned long long *__restrict__ ctr, int *__restrict__ work) {
    extern __shared__ __align__(256) uint8_t smem[];
    const int lane = lane_id();
    const int wid = threadIdx.x >> 5;
    // (per-warp stride a multiple of 256: the ADT's PRMT-merged addresses)
    uint8_t *ctx = smem + (size_t)wid * round_up(ctx_bytes + 8 * cand, 256);
    int32_t *ids_s = reinterpret_cast<int32_t *>(ctx + ctx_bytes);
    uint32_t *d_s = reinterpret_cast<uint32_t *>(ids_s + cand);
    CounterTotals total;
    for (;;) {
        int q = 0;
        if (lane == 0) q = atomicAdd(work, 1);
        q = __shfl_sync(0xffffffffu, q, 0);
        if (q >= size) break;
        const int x = start + q;
        load_adt_smem(ctx, adt_batch + (size_t)q * g.mpad * 16, g.mpad, lane);
        __syncwarp();
        SearchCounters cnt = {};
        const int level = __ldg(g.levels + x);
        int cur = ep;
        uint32_t curd = P::one(g, ctx, ep, lane);
        cnt.dist += 1;
        for (int layer = ml; layer > level; --layer)
            hill_climb<P>(g, layer, cur, curd, ctx, ids_s, d_s, cnt, lane);
        if (lane == 0) {
            start_v[q] = cur;
            start_d[q] = curd;
            atomicAdd(hist + descend_key(level, maxlv, curd), 1);
        }
        total.add(cnt);
        __syncwarp();
    }
    flush_counters(total, ctr, lane);
}
template __global__ void batch_descend_kernel<FlashDist>(Graph, const uint8_t *, int, int, int, int,
                                                         int, int, int, int *, uint32_t *, int *,
                                                         unsigned long long *, int *);
template __global__ void batch_descend_kernel<FlashDistW>(Graph, const uint8_t *, int, int, int, int,
                                                          int, int, int, int *, uint32_t *, int *,
                                                          unsigned long long *, int *);

// hist -> exclusive offsets (one CTA; nkeys <= a few thousand)
__global__ void __launch_bounds__(1024) descend_scan_kernel(int *__restrict__ hist, int nkeys) {
    __shared__ int part[1024];
    const int per = (nkeys + 1023) / 1024;
    const int k0 = threadIdx.x * per, k1 = min(nkeys, k0 + per);
    int sum = 0;
    for (int k = k0; k < k1; ++k) sum += hist[k];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    int run = part[threadIdx.x] - sum;
    for (int k = k0; k < k1; ++k) {
        const int c = hist[k];
        hist[k] = run;
        run += c;
    }
}

// the batch's processing order: vertices by key (higher levels first, then
// the farthest descents first); within a key in any order
__global__ void descend_order_kernel(const int32_t *__restrict__ levels, int start, int size,
                                     int maxlv, const uint32_t *__restrict__ start_d,
                                     int *__restrict__ offs, int32_t *__restrict__ order) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < size; q += gridDim.x * blockDim.x) {
        const int key = descend_key(__ldg(levels + start + q), maxlv, __ldg(start_d + q));
        order[atomicAdd(offs + key, 1)] = q;
    }
}

// RC: id-row chunks compiled into the hot loop (2 when the base rows hold
// <= 64 slots: the common R <= 32; else 4)
#define FA_BUILD_J(P, EM, RC)                                 \
    switch (v) {                                              \
        case 2: return build_search_kernel<P, 2, EM, RC>;     \
        case 4: return build_search_kernel<P, 4, EM, RC>;     \
        case 7: return build_search_kernel<P, 7, EM, RC>;     \
        case 8: return build_search_kernel<P, 8, EM, RC>;     \
        case 10: return build_search_kernel<P, 10, EM, RC>;   \
        case 16: return build_search_kernel<P, 16, EM, RC>;   \
        default: break;                                       \
    }

BuildSearchFn build_search_variant(int W, int expand, int cap0, bool wide) {
    const int v = set_variant(W);
    if (wide) {  // 32-bit ids (n >= 2^24): one expansion per step, any row size
        FA_BUILD_J(FlashDistW, 1, kRowChunks)
        return build_search_kernel<FlashDistW, 0, 1, kRowChunks>;
    }
    if (expand > 1) {
        if (v == 0) return build_search_kernel<FlashDist, 0, 1, kRowChunks>;
        return v <= 8 ? build_search_kernel<FlashDist, 8, kMaxExpand, kRowChunks>
                      : build_search_kernel<FlashDist, 16, kMaxExpand, kRowChunks>;
    }
    if (cap0 <= 64) {
        FA_BUILD_J(FlashDist, 1, 2)
    } else {
        FA_BUILD_J(FlashDist, 1, kRowChunks)
    }
    return build_search_kernel<FlashDist, 0, 1, kRowChunks>;
}

BuildSearchFn build_search_exact_variant(int W, int cap0, bool wide) {
    const int v = set_variant(W);
    if (wide) {
        FA_BUILD_J(ExactDistW, 1, kRowChunks)
        return build_search_kernel<ExactDistW, 0, 1, kRowChunks>;
    }
    if (cap0 <= 64) {
        FA_BUILD_J(ExactDist, 1, 2)
    } else {
        FA_BUILD_J(ExactDist, 1, kRowChunks)
    }
    return build_search_kernel<ExactDist, 0, 1, kRowChunks>;  // W > kRegSetMax
}
#undef FA_BUILD_J

}  // namespace fa
