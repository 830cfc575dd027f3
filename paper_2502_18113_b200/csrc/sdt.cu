// SDT sums (fa_sdt_sum_sat, _simd.h:87-95) and the select_neighbors hook
// (_core.pyx:942-959) on the warp selection of select.cuh.
#include "select.cuh"

namespace fa {

__global__ void sdt_sum_kernel(const uint8_t *__restrict__ sdt, int m, const uint8_t *__restrict__ a,
                               int64_t as, const uint8_t *__restrict__ b, int64_t bs, int64_t npairs,
                               int32_t *__restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npairs;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t *ca = a + p * as;
        const uint8_t *cb = b + p * bs;
        uint32_t acc = 0;
        for (int i = 0; i < m; ++i) acc += __ldg(sdt + ((size_t)i * 16 + ca[i]) * 16 + cb[i]);
        out[p] = (int32_t)(acc > 255u ? 255u : acc);
    }
}

__global__ void transpose_sdt_kernel(const uint8_t *__restrict__ sdt, int m,
                                     uint8_t *__restrict__ sdtT) {
    stage_sdt_T(sdt, m, sdtT, threadIdx.x, blockDim.x);
}

// One warp: the whole candidate list of a select_neighbors call.
__global__ void select_hook_kernel(const uint8_t *__restrict__ sdt, int m, int mpad,
                                   const uint8_t *__restrict__ codes, int cs,
                                   const int32_t *__restrict__ cand_ids,
                                   const double *__restrict__ cand_d, int ncand, int cap,
                                   int32_t *__restrict__ out, int32_t *__restrict__ nout) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t *sdtT = smem;
    int32_t *kept = reinterpret_cast<int32_t *>(smem + round_up(m * 256, 16));
    uint8_t *kcodes = reinterpret_cast<uint8_t *>(kept) + round_up(cap * 4, 16);
    const int lane = threadIdx.x;
    stage_sdt_T(sdt, m, sdtT, lane, 32);
    __syncwarp();
    int nk = warp_select_heur(
        sdtT, m, mpad, codes, cs, ncand, cap,
        [&](int j, int &v, double &dv) {
            v = __ldg(cand_ids + j);
            dv = __ldg(cand_d + j);
        },
        kept, kcodes, lane, nullptr);
    for (int t = lane; t < nk; t += 32) out[t] = kept[t];
    if (lane == 0) *nout = nk;
}

// select_heur of the exact kind for the select_neighbors hook: candidate v
// (distance dv, f64 as given) is kept iff no kept u has (double) fp32 L2(u, v)
// < dv (_core.pyx:388-408 with sym_one of K_EXACT, _core.pyx:179-191).  One
// warp; lanes test the kept set in parallel, each with the fa_l2sq_f32 tree.
__global__ void select_exact_hook_kernel(const float *__restrict__ vecs, int dim,
                                         const int32_t *__restrict__ cand_ids,
                                         const double *__restrict__ cand_d, int ncand, int cap,
                                         int32_t *__restrict__ out, int32_t *__restrict__ nout) {
    extern __shared__ __align__(16) int32_t kept[];
    const int lane = threadIdx.x;
    int nk = 0;
    for (int j = 0; j < ncand && nk < cap; ++j) {
        const int v = __ldg(cand_ids + j);
        const double dv = __ldg(cand_d + j);
        const float *b = vecs + (size_t)v * dim;
        bool bad = false;
        for (int t = lane; t < nk; t += 32) {
            const float *a = vecs + (size_t)kept[t] * dim;
            const float s = l2_tree(dim, [&](int i) { return __fsub_rn(__ldg(a + i), __ldg(b + i)); });
            bad |= (double)s < dv;
        }
        if (!__any_sync(0xffffffffu, bad)) {
            if (lane == 0) kept[nk] = v;
            ++nk;
        }
        __syncwarp();
    }
    for (int t = lane; t < nk; t += 32) out[t] = kept[t];
    if (lane == 0) *nout = nk;
}

}  // namespace fa

using namespace fa;

extern "C" int fa_select_exact_dev(const float *vecs, int dim, const int32_t *cand_ids,
                                   const double *cand_d, int ncand, int cap, int32_t *out,
                                   int32_t *nout, void *stream) {
    FA_CHECK_ARG(dim >= 1, "dim must be >= 1");
    FA_CHECK_ARG(ncand >= 0 && cap >= 0, "negative sizes");
    cudaStream_t st = as_stream(stream);
    if (ncand == 0 || cap == 0) {
        FA_CUDA(cudaMemsetAsync(nout, 0, sizeof(int32_t), st));
        return FA_OK;
    }
    const size_t smem = (size_t)round_up(cap, 4) * 4;
    FA_CHECK_ARG(smem <= 220 * 1024, "cap too large for one select call");
    if (smem > 48 * 1024)
        FA_CUDA(cudaFuncSetAttribute(select_exact_hook_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    select_exact_hook_kernel<<<1, 32, smem, st>>>(vecs, dim, cand_ids, cand_d, ncand, cap, out,
                                                  nout);
    FA_LAUNCH_CHECK();
    return FA_OK;
}

extern "C" int fa_sdt_sum_dev(const uint8_t *sdt, int m, const uint8_t *a, int64_t a_stride,
                              const uint8_t *b, int64_t b_stride, int64_t npairs, int32_t *out,
                              void *stream) {
    FA_CHECK_ARG(m >= 1 && npairs >= 0, "bad sizes");
    if (npairs == 0) return FA_OK;
    int64_t want = (npairs + 127) / 128;
    int grid = (int)(want < 148 * 16 ? want : 148 * 16);
    sdt_sum_kernel<<<grid, 128, 0, as_stream(stream)>>>(sdt, m, a, a_stride, b, b_stride, npairs,
                                                         out);
    FA_LAUNCH_CHECK();
    return FA_OK;
}

extern "C" int fa_select_dev(const uint8_t *sdt, int m, const uint8_t *codes, int code_stride,
                             const int32_t *cand_ids, const double *cand_d, int ncand, int cap,
                             int32_t *out, int32_t *nout, void *stream) {
    FA_CHECK_ARG(m >= 1, "m must be >= 1");
    FA_CHECK_ARG(code_stride % 16 == 0 && code_stride >= m,
                 "code_stride must be a multiple of 16 and >= m (zero padded)");
    FA_CHECK_ARG(ncand >= 0 && cap >= 0, "negative sizes");
    cudaStream_t st = as_stream(stream);
    if (ncand == 0 || cap == 0) {
        FA_CUDA(cudaMemsetAsync(nout, 0, sizeof(int32_t), st));
        return FA_OK;
    }
    int mpad = code_stride;
    size_t smem = round_up(m * 256, 16) + round_up(cap * 4, 16) + (size_t)cap * kept_stride(mpad);
    FA_CHECK_ARG(smem <= 220 * 1024, "cap too large for one select call");
    if (smem > 48 * 1024)
        FA_CUDA(cudaFuncSetAttribute(select_hook_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    select_hook_kernel<<<1, 32, smem, st>>>(sdt, m, mpad, codes, code_stride, cand_ids, cand_d,
                                            ncand, cap, out, nout);
    FA_LAUNCH_CHECK();
    return FA_OK;
}
