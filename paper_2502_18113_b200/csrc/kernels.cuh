// Kernel declarations shared between the translation units of the core.
#pragma once

#include "search.cuh"

namespace fa {

constexpr int kSearchWarps = 4;   // warps (points) per CTA in the search kernels
// The build's search kernel: CTAs of up to this many warps (the host picks the
// width that keeps the most warps resident); __maxnreg__(96) keeps 5 warps
// per scheduler whatever the width
constexpr int kBuildWarpsMax = 7;
constexpr int kReverseWarps = 4;  // warps per CTA in the reverse-edge kernel

__device__ __forceinline__ int64_t row_global(const Graph &g, int layer, int y) {
    return layer == 0 ? (int64_t)y : g.n + __ldg(g.uoff + y) + layer - 1;
}

// Per-warp workspace pointers (WarpLayout): warp `wid` of a CTA of `warps`.
struct WarpWS {
    uint8_t *adt;
    unsigned long long *T, *S;
    int32_t *TQ;
    int32_t *fresh;
    uint32_t *fdist;
    uint32_t *H;
    __device__ WarpWS(uint8_t *smem, int wid, int warps, const WarpLayout &L) {
        uint8_t *bg = smem + wid * L.big;
        uint8_t *sm = smem + warps * L.big + wid * L.small;
        adt = bg + L.adt;
        H = reinterpret_cast<uint32_t *>(bg + L.hash);
        T = reinterpret_cast<unsigned long long *>((L.t_big ? bg : sm) + L.T);
        S = reinterpret_cast<unsigned long long *>(sm + L.S);
        TQ = reinterpret_cast<int32_t *>(sm + L.TQ);
        fresh = reinterpret_cast<int32_t *>(sm + L.fresh);
        fdist = reinterpret_cast<uint32_t *>(sm + L.fdist);
    }
};

// 64-bit running totals of SearchCounters over the searches of one warp
struct CounterTotals {
    unsigned long long dist = 0, kcalls = 0, visited = 0, sym = 0;
    __device__ void add(const SearchCounters &c) {
        dist += c.dist;
        kcalls += c.kcalls;
        visited += c.visited;
        sym += c.sym;
    }
};

__device__ __forceinline__ void flush_counters(const CounterTotals &c, unsigned long long *ctr,
                                               int lane) {
    if (lane == 0) {
        atomicAdd(ctr + 0, c.dist);
        atomicAdd(ctr + 1, c.sym);
        atomicAdd(ctr + 2, c.kcalls);
        atomicAdd(ctr + 3, c.visited);
    }
}
__device__ __forceinline__ void flush_counters(const SearchCounters &c, unsigned long long *ctr,
                                               int lane) {
    CounterTotals t;
    t.add(c);
    flush_counters(t, ctr, lane);
}

using BuildSearchFn = void (*)(Graph, const uint8_t *, const uint8_t *, int, int, int, int, int,
                               int, WarpLayout, const int64_t *, const int32_t *,
                               unsigned long long *, unsigned long long *, int *, int64_t *, int *,
                               const int *, const uint32_t *);
// the Flash build's batch descents and processing order (build_search.cu)
template <typename P>
__global__ void batch_descend_kernel(Graph g, const uint8_t *__restrict__ adt_batch, int start,
                                     int size, int ep, int ml, int maxlv, int ctx_bytes, int cand,
                                     int *__restrict__ start_v, uint32_t *__restrict__ start_d,
                                     int *__restrict__ hist, unsigned long long *__restrict__ ctr,
                                     int *__restrict__ work);
__global__ void descend_scan_kernel(int *__restrict__ hist, int nkeys);
__global__ void descend_order_kernel(const int32_t *__restrict__ levels, int start, int size,
                                     int maxlv, const uint32_t *__restrict__ start_d,
                                     int *__restrict__ offs, int32_t *__restrict__ order);
using QuerySearchFn = void (*)(Graph, const uint8_t *, int, int, int, int, int, int, const float *,
                               int, const float *, WarpLayout, int64_t *, double *,
                               unsigned long long *, int *);
using LayerSearchFn = void (*)(Graph, const uint8_t *, int, const int64_t *, int, int, WarpLayout,
                               int32_t *, double *, int32_t *, unsigned long long *, int *);

// Kernel instantiations per result-set variant (set_variant(W)) and, for the
// build, per expansion width (1 or kMaxExpand).
// wide: 32-bit vertex ids (n >= 2^24; 64-bit keys, FlashDistW / ExactDistW)
BuildSearchFn build_search_variant(int W, int expand, int cap0, bool wide);
BuildSearchFn build_search_exact_variant(int W, int cap0, bool wide);
// exact = true: the exact-kind instantiations
QuerySearchFn query_search_variant(int W, bool exact, bool wide);
LayerSearchFn layer_search_variant(int W, bool exact, bool wide);

struct ReverseLayout {
    int tdom, tkeep, row, rowd, keptd, cand, sel, total;
    int qv, cv, cid, cd, kd;  // exact kind: y's and a candidate's vectors, ids, distances
    int rowd32, keptd32, kflag;  // exact kind: the row's cached fp32 distances, survivors
    __host__ __device__ void init(int capmax, int m, int mpad, int dim = 0) {
        int o = 0;
        tdom = o; o += round_up(mpad * 16, 256);   // x's row tables (256-aligned)
        tkeep = o; o += round_up(mpad * 16, 256);
        row = o; o += round_up(capmax, 32) * 4;
        rowd = o; o += round_up(capmax, 32);
        keptd = o; o += round_up(capmax, 32);
        cand = o; o += 128 * 8;
        o = round_up(o, 256);
        // kept ids (the rare full prune's select workspace lives in global
        // scratch: reverse_kernel's sel_scratch)
        sel = o; o += round_up(capmax * 4, 256);
        qv = cv = cid = cd = kd = rowd32 = keptd32 = kflag = 0;
        if (dim > 0) {
            qv = o; o += round_up(dim * 4, 16);
            cv = o; o += round_up(dim * 4, 16);
            cid = o; o += round_up(capmax + 1, 32) * 4;
            cd = o; o += round_up(capmax + 1, 32) * 4;
            kd = o; o += round_up(capmax, 32) * 4;
            rowd32 = o; o += round_up(capmax, 32) * 4;
            keptd32 = o; o += round_up(capmax, 32) * 4;
            kflag = o; o += round_up(capmax, 32);
        }
        total = round_up(o, 256);
    }
};

__global__ void bucket_place_kernel(const int32_t *touched, const int *ntouched, int32_t *rowcnt,
                                    int32_t *rowoff, int64_t *heads, int *cursor);
__global__ void bucket_scatter_kernel(const unsigned long long *req, int64_t N, int32_t *fill,
                                      const int32_t *rowoff, const int *cursor,
                                      unsigned long long *out);

template <int RC>
__global__ void reverse_kernel(Graph g, const uint8_t *__restrict__ sdt,
                               const uint8_t *__restrict__ sdtT,
                               const unsigned long long *__restrict__ keys, int64_t N,
                               const int64_t *__restrict__ heads, const int *__restrict__ nheads,
                               int *__restrict__ next, const int32_t *__restrict__ upper_owner,
                               ReverseLayout L, unsigned long long *__restrict__ ctr,
                               uint8_t *__restrict__ sel_scratch, int sel_bytes);

__global__ void reverse_exact_kernel(Graph g, const unsigned long long *__restrict__ keys,
                                     int64_t N, const int64_t *__restrict__ heads,
                                     const int *__restrict__ nheads, int *__restrict__ next,
                                     const int32_t *__restrict__ upper_owner, ReverseLayout L,
                                     unsigned long long *__restrict__ ctr);

int launch_encode_adt(const float *red, int64_t n, int64_t red_stride, const float *cent,
                      const int32_t *dims, const int32_t *offs, int m, int dmax, double dmin,
                      double delta, uint8_t *codes, int code_stride, uint8_t *adt, int adt_rows,
                      cudaStream_t st);

}  // namespace fa
