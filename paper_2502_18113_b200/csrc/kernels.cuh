// Kernel declarations shared between the translation units of the core.
#pragma once

#include "search.cuh"

namespace fa {

constexpr int kSearchWarps = 4;   // warps (points) per CTA in the search kernels
constexpr int kReverseWarps = 4;  // warps per CTA in the reverse-edge kernel

__global__ void build_search_kernel(Graph g, const uint8_t *__restrict__ sdt,
                                    const uint8_t *__restrict__ adt_batch, int start, int size,
                                    int ep, int ml, int C, int R, WarpLayout L,
                                    const int64_t *__restrict__ req_off,
                                    unsigned long long *__restrict__ req,
                                    unsigned long long *__restrict__ ctr, int *err,
                                    int64_t *__restrict__ stats, int *__restrict__ work);

__global__ void query_search_kernel(Graph g, const uint8_t *__restrict__ adt_q, int nq, int ep,
                                    int ml, int ef, int k, int rerank_depth,
                                    const float *__restrict__ vecs, int dim,
                                    const float *__restrict__ queries, WarpLayout L,
                                    int64_t *__restrict__ out_ids, double *__restrict__ out_d,
                                    unsigned long long *__restrict__ ctr, int *err);

__global__ void layer_search_kernel(Graph g, const uint8_t *__restrict__ adt_q, int nq,
                                    const int64_t *__restrict__ entries, int width, int layer,
                                    WarpLayout L, int32_t *__restrict__ out_ids,
                                    double *__restrict__ out_d, int32_t *__restrict__ out_n,
                                    unsigned long long *__restrict__ ctr, int *err);

struct ReverseLayout {
    int row, cand, kept, kcodes, total;
    __host__ __device__ void init(int capmax, int mpad) {
        int o = 0;
        row = o; o += round_up(capmax, 32) * 4;
        cand = o; o += 128 * 8;
        kept = o; o += round_up(capmax, 32) * 4;
        kcodes = o; o += round_up(capmax * kept_stride(mpad), 16);
        total = round_up(o, 128);
    }
};

__global__ void reverse_heads_kernel(const unsigned long long *__restrict__ keys, int64_t N,
                                     int64_t *__restrict__ heads, int *__restrict__ nheads,
                                     int *__restrict__ next);

__global__ void reverse_kernel(Graph g, const uint8_t *__restrict__ sdt,
                               const unsigned long long *__restrict__ keys, int64_t N,
                               const int64_t *__restrict__ heads, const int *__restrict__ nheads,
                               int *__restrict__ next, const int32_t *__restrict__ upper_owner,
                               ReverseLayout L, unsigned long long *__restrict__ ctr);

int launch_encode_adt(const float *red, int64_t n, int64_t red_stride, const float *cent,
                      const int32_t *dims, const int32_t *offs, int m, int dmax, double dmin,
                      double delta, uint8_t *codes, int code_stride, uint8_t *adt, int adt_rows,
                      cudaStream_t st);

}  // namespace fa
