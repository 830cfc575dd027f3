// K2: batched encode + uint8 query table (fa_flash_encode_adt, _simd.h:211-228),
// the uint8 quantiser (fa_quantize, _simd.h:99-107) and row-wise fp32 L2
// (fa_l2sq_f32, _simd.h:44-51) with the reference build's operation tree.
#include "common.cuh"

namespace fa {

__global__ void quantize_kernel(const double *__restrict__ d, int64_t n, double dmin, double delta,
                                uint8_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = quantize_dev(d[i], dmin, delta);
}

__global__ void l2_rows_kernel(const float *__restrict__ a, int64_t as, const float *__restrict__ b,
                               int64_t bs, int64_t n, int d, double *__restrict__ out) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const float *x = a + r * as;
        const float *y = b + r * bs;
        float s = l2_tree(d, [&](int k) { return __fsub_rn(__ldg(x + k), __ldg(y + k)); });
        out[r] = (double)s;
    }
}

// One thread per (row, subspace slot).  Centroids are staged in shared memory
// transposed to [j][k][i] (subspace fastest) so consecutive threads (= consecutive
// subspaces of one row) read consecutive words: conflict-free.
__global__ void __launch_bounds__(256) encode_adt_kernel(
    const float *__restrict__ red, int64_t n, int64_t red_stride, const float *__restrict__ cent,
    const int32_t *__restrict__ dims, const int32_t *__restrict__ offs, int m, int dmax,
    double dmin, double delta, uint8_t *__restrict__ codes, int code_stride,
    uint8_t *__restrict__ adt, int adt_rows, int P) {
    extern __shared__ float cs[];  // [16][dmax][m]
    for (int t = threadIdx.x; t < m * 16 * dmax; t += blockDim.x) {
        int i = t / (16 * dmax);
        int rem = t % (16 * dmax);  // j * dmax + k
        cs[rem * m + i] = cent[t];
    }
    __syncthreads();
    const int64_t total = n * P;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
         w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = w / P;
        const int i = (int)(w % P);
        if (i < m) {
            const int di = __ldg(dims + i);
            const float *x = red + row * red_stride + __ldg(offs + i);
            float xr[64];
#pragma unroll 8
            for (int k = 0; k < di; ++k) xr[k] = __ldg(x + k);
            int best = 0;
            double bestd = __longlong_as_double(0x7ff0000000000000ll);  // +inf
            uint32_t q[4] = {0, 0, 0, 0};
#pragma unroll 4
            for (int j = 0; j < 16; ++j) {
                const float *c = cs + (size_t)j * dmax * m + i;
                float s = l2_tree(di, [&](int k) { return __fsub_rn(xr[k], c[(size_t)k * m]); });
                double dd = (double)s;
                uint32_t qb = quantize_dev(dd, dmin, delta);
                q[j >> 2] |= qb << (8 * (j & 3));
                if (dd < bestd) {
                    bestd = dd;
                    best = j;
                }
            }
            if (codes && i < code_stride) codes[row * code_stride + i] = (uint8_t)best;
            if (adt && i < adt_rows)
                *reinterpret_cast<uint4 *>(adt + (row * adt_rows + i) * 16) =
                    make_uint4(q[0], q[1], q[2], q[3]);
        } else {
            if (codes && i < code_stride) codes[row * code_stride + i] = 0;
            if (adt && i < adt_rows)
                *reinterpret_cast<uint4 *>(adt + (row * adt_rows + i) * 16) = make_uint4(0, 0, 0, 0);
        }
    }
}

int launch_encode_adt(const float *red, int64_t n, int64_t red_stride, const float *cent,
                      const int32_t *dims, const int32_t *offs, int m, int dmax, double dmin,
                      double delta, uint8_t *codes, int code_stride, uint8_t *adt, int adt_rows,
                      cudaStream_t st) {
    FA_CHECK_ARG(m >= 1, "m must be >= 1");
    FA_CHECK_ARG(dmax >= 1 && dmax <= 64, "dmax=%d outside [1,64]", dmax);
    FA_CHECK_ARG(code_stride >= m, "code_stride < m");
    FA_CHECK_ARG(!adt || adt_rows >= m, "adt_rows < m");
    FA_CHECK_ARG(delta > 0.0, "degenerate quantization range");
    if (n == 0) return FA_OK;
    int P = m;
    if (adt && adt_rows > P) P = adt_rows;
    if (code_stride > P) P = code_stride;
    size_t smem = sizeof(float) * (size_t)m * 16 * dmax;
    FA_CHECK_ARG(smem <= 200 * 1024, "centroid table too large for shared memory");
    if (smem > 48 * 1024)
        FA_CUDA(cudaFuncSetAttribute(encode_adt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    int64_t total = n * P;
    int64_t want = (total + 255) / 256;
    int grid = (int)(want < 148 * 8 ? want : 148 * 8);
    encode_adt_kernel<<<grid, 256, smem, st>>>(red, n, red_stride, cent, dims, offs, m, dmax, dmin,
                                               delta, codes, code_stride, adt, adt_rows, P);
    FA_LAUNCH_CHECK();
    return FA_OK;
}

}  // namespace fa

using namespace fa;

extern "C" int fa_quantize_dev(const double *d, int64_t n, double dist_min, double delta,
                               uint8_t *out, void *stream) {
    FA_CHECK_ARG(n >= 0, "n < 0");
    if (n == 0) return FA_OK;
    int64_t want = (n + 255) / 256;
    int grid = (int)(want < 148 * 16 ? want : 148 * 16);
    quantize_kernel<<<grid, 256, 0, as_stream(stream)>>>(d, n, dist_min, delta, out);
    FA_LAUNCH_CHECK();
    return FA_OK;
}

extern "C" int fa_l2sq_rows_dev(const float *a, int64_t a_stride, const float *b, int64_t b_stride,
                                int64_t n, int d, double *out, void *stream) {
    FA_CHECK_ARG(n >= 0 && d >= 0, "negative sizes");
    if (n == 0) return FA_OK;
    int64_t want = (n + 127) / 128;
    int grid = (int)(want < 148 * 16 ? want : 148 * 16);
    l2_rows_kernel<<<grid, 128, 0, as_stream(stream)>>>(a, a_stride, b, b_stride, n, d, out);
    FA_LAUNCH_CHECK();
    return FA_OK;
}

extern "C" int fa_encode_adt_dev(const float *red, int64_t n, int64_t red_stride, const float *cent,
                                 const int32_t *dims, const int32_t *offs, int m, int dmax,
                                 double dist_min, double delta, uint8_t *codes_out, int code_stride,
                                 uint8_t *adt_out, int adt_rows, void *stream) {
    return launch_encode_adt(red, n, red_stride, cent, dims, offs, m, dmax, dist_min, delta,
                             codes_out, code_stride, adt_out, adt_rows, as_stream(stream));
}
