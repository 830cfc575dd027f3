// K2: batched encode + uint8 query table (fa_flash_encode_adt, _simd.h:211-228),
// the uint8 quantiser (fa_quantize, _simd.h:99-107) and row-wise fp32 L2
// (fa_l2sq_f32, _simd.h:44-51) with the reference build's operation tree.
#include <mutex>
#include <vector>

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

// The quantiser as thresholds.  fa_quantize (IEEE double: subtract, divide,
// multiply, floor, clamp) is a non-decreasing function of its input, and K2
// feeds it fp32 distances (widened exactly), so q(s) = #{k >= 1 : s >= T[k]}
// with T[k] the smallest non-negative float whose quantised value reaches k,
// found once per (dist_min, delta) by bisection over float bit patterns with
// the exact double formula.  The encoder then replaces a double division per
// (row, subspace, centroid) by a float estimate corrected against T: the same
// bytes (bit-exact by construction; the golden 1-ulp grids check it).
__global__ void quant_thresholds_kernel(double dmin, double delta, float *__restrict__ T) {
    const int k = threadIdx.x;
    if (k == 0) {
        T[0] = -__int_as_float(0x7f800000);  // every value quantises to >= 0
        return;
    }
    uint32_t lo = 0u, hi = 0x7f800000u;  // q(+inf) = 255 >= k
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        if (quantize_dev((double)__uint_as_float(mid), dmin, delta) >= k)
            hi = mid;
        else
            lo = mid + 1u;
    }
    T[k] = __uint_as_float(lo);
}

// q(s) from the thresholds Ts (shared): an estimate from the float formula,
// corrected to the exact count (at most a step or two either way)
__device__ __forceinline__ uint32_t quantize_thr(float s, const float *Ts, float dminf,
                                                 float scalef) {
    const float est = __fmul_rn(__fsub_rn(s, dminf), scalef);
    int g = est >= 255.f ? 255 : (est > 0.f ? (int)est : 0);
    while (g < 255 && s >= Ts[g + 1]) ++g;
    while (g > 0 && s < Ts[g]) --g;
    return (uint32_t)g;
}

// One thread per (row, subspace slot).  Centroids are staged in shared memory
// transposed to [j][k][i] (subspace fastest) so consecutive threads (= consecutive
// subspaces of one row) read consecutive words: conflict-free.  qthr: the
// quantiser's thresholds (null = codes only, no table).  DT > 0: subspaces of
// exactly DT dimensions (every one of them when d_F is a multiple of m) take
// a fully unrolled path whose row slice stays in registers; others take the
// generic loop (its slice in local memory).
template <int DT>
__global__ void __launch_bounds__(256) encode_adt_kernel(
    const float *__restrict__ red, int64_t n, int64_t red_stride, const float *__restrict__ cent,
    const int32_t *__restrict__ dims, const int32_t *__restrict__ offs, int m, int dmax,
    double dmin, double delta, const float *__restrict__ qthr, uint8_t *__restrict__ codes,
    int code_stride, uint8_t *__restrict__ adt, int adt_rows, int P) {
    extern __shared__ float cs[];  // [16][dmax][m], then the 256 thresholds
    float *Ts = cs + m * 16 * dmax;
    for (int t = threadIdx.x; t < m * 16 * dmax; t += blockDim.x) {
        int i = t / (16 * dmax);
        int rem = t % (16 * dmax);  // j * dmax + k
        cs[rem * m + i] = cent[t];
    }
    if (qthr)
        for (int t = threadIdx.x; t < 256; t += blockDim.x) Ts[t] = qthr[t];
    const float dminf = (float)dmin, scalef = (float)(255.0 / delta);
    __syncthreads();
    const int64_t total = n * P;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
         w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = w / P;
        const int i = (int)(w % P);
        if (i < m) {
            const int di = __ldg(dims + i);
            const float *x = red + row * red_stride + __ldg(offs + i);
            float sd[16];  // distances to the 16 centroids
            if (DT > 0 && di == DT) {
                float xr[DT > 0 ? DT : 1];
#pragma unroll
                for (int k = 0; k < DT; ++k) xr[k] = __ldg(x + k);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float *c = cs + (size_t)j * dmax * m + i;
                    sd[j] = l2_tree(DT, [&](int k) { return __fsub_rn(xr[k], c[(size_t)k * m]); });
                }
            } else {
                float xr[64];
#pragma unroll 8
                for (int k = 0; k < di; ++k) xr[k] = __ldg(x + k);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float *c = cs + (size_t)j * dmax * m + i;
                    sd[j] = l2_tree(di, [&](int k) { return __fsub_rn(xr[k], c[(size_t)k * m]); });
                }
            }
            int best = 0;
            float bests = __int_as_float(0x7f800000);  // +inf
            uint32_t q[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float s = sd[j];
                if (qthr) q[j >> 2] |= quantize_thr(s, Ts, dminf, scalef) << (8 * (j & 3));
                // (the reference compares the widened doubles: the same order)
                if (s < bests) {
                    bests = s;
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

// Thresholds of one quantiser (dist_min, delta), computed once and kept for
// the process (1 KB per coder; never freed, so no stream can still be reading
// a table that goes away).
static int quant_thresholds(double dmin, double delta, const float **out) {
    struct Entry {
        int dev;
        double dmin, delta;
        float *T;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    int dev = 0;
    FA_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    for (const Entry &e : cache)
        if (e.dev == dev && e.dmin == dmin && e.delta == delta) {
            *out = e.T;
            return FA_OK;
        }
    float *T = nullptr;
    FA_TRY(pool_alloc((void **)&T, 256 * sizeof(float)));
    quant_thresholds_kernel<<<1, 256>>>(dmin, delta, T);
    FA_CUDA(cudaGetLastError());
    FA_CUDA(cudaStreamSynchronize(0));  // ready for every stream that uses it
    cache.push_back({dev, dmin, delta, T});
    *out = T;
    return FA_OK;
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
    const float *qthr = nullptr;
    if (adt) FA_TRY(quant_thresholds(dmin, delta, &qthr));
    size_t smem = sizeof(float) * ((size_t)m * 16 * dmax + 256);
    FA_CHECK_ARG(smem <= 200 * 1024, "centroid table too large for shared memory");
    // the widest subspaces (dmax dimensions: all of them when d_F % m == 0)
    // get the unrolled path
    decltype(&encode_adt_kernel<0>) fn = encode_adt_kernel<0>;
    switch (dmax) {
        case 1: fn = encode_adt_kernel<1>; break;
        case 2: fn = encode_adt_kernel<2>; break;
        case 3: fn = encode_adt_kernel<3>; break;
        case 4: fn = encode_adt_kernel<4>; break;
        case 5: fn = encode_adt_kernel<5>; break;
        case 6: fn = encode_adt_kernel<6>; break;
        case 8: fn = encode_adt_kernel<8>; break;
        case 12: fn = encode_adt_kernel<12>; break;
        case 16: fn = encode_adt_kernel<16>; break;
        default: break;
    }
    if (smem > 48 * 1024)
        FA_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int64_t total = n * P;
    int64_t want = (total + 255) / 256;
    int grid = (int)(want < 148 * 8 ? want : 148 * 8);
    fn<<<grid, 256, smem, st>>>(red, n, red_stride, cent, dims, offs, m, dmax, dmin, delta, qthr,
                                codes, code_stride, adt, adt_rows, P);
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
