// K3: coder training on the device — one CTA per subspace.
//
//   kmeans (flashann/kmeans.py:16-76): k-means++ seeding + `iters` Lloyd steps
//     in float64 on the (sub)sample; argmin first index; empty clusters
//     reseeded to the farthest point.  The random stream is numpy's PCG64
//     (Generator.integers / Generator.random) continued on the device from the
//     host-drawn permutation state, so the draws are the reference's draws.
//   range statistics (flashann/flash.py:86-98): raw SDT (direct differences),
//     sample-to-centroid distances (||x||^2 + ||c||^2 - 2 x.c, clamped >= 0),
//     per-subspace min/max, dist_min = min, dist_max = sum of maxima.
//
// numpy's float64 summation order is reproduced where it decides a value:
// np.sum is pairwise (n < 8 sequential from 0; 8..128 eight strided
// accumulators; recursive halving above), which `pw_sum` restates.
#include <algorithm>
#include <thread>
#include <vector>

#include "common.cuh"

namespace fa {

struct Pcg64State {
    unsigned long long s_hi, s_lo, inc_hi, inc_lo;
    unsigned int has_uint32, uinteger;
};

struct Pcg64 {
    unsigned __int128 s, inc;
    bool has;
    uint32_t u;
    __host__ __device__ explicit Pcg64(const Pcg64State &st) {
        s = ((unsigned __int128)st.s_hi << 64) | st.s_lo;
        inc = ((unsigned __int128)st.inc_hi << 64) | st.inc_lo;
        has = st.has_uint32 != 0;
        u = st.uinteger;
    }
    __host__ __device__ uint64_t next64() {
        const unsigned __int128 mult =
            ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
        s = s * mult + inc;
        uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
        unsigned rot = (unsigned)(s >> 122);
        return (x >> rot) | (x << ((64 - rot) & 63));
    }
    __host__ __device__ uint32_t next32() {
        if (has) {
            has = false;
            return u;
        }
        uint64_t v = next64();
        has = true;
        u = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
    __host__ void store(Pcg64State &st) const {
        st.s_hi = (unsigned long long)(s >> 64);
        st.s_lo = (unsigned long long)s;
        st.inc_hi = (unsigned long long)(inc >> 64);
        st.inc_lo = (unsigned long long)inc;
        st.has_uint32 = has ? 1u : 0u;
        st.uinteger = u;
    }
    // random_interval (numpy distributions.c): a draw in [0, mx] by masked
    // rejection, 32-bit draws while mx fits
    __host__ uint64_t interval(uint64_t mx) {
        if (mx == 0) return 0;
        uint64_t mask = mx;
        for (int k = 1; k < 64; k <<= 1) mask |= mask >> k;
        uint64_t v;
        if (mx <= 0xffffffffull) {
            do v = next32() & mask; while (v > mx);
        } else {
            do v = next64() & mask; while (v > mx);
        }
        return v;
    }
    // Generator.random(): 53-bit double
    __device__ double random() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
    // Generator.integers(n) for 1 <= n <= 2^32 (Lemire, buffered 32-bit draws)
    __device__ int64_t integers(int64_t n) {
        uint32_t rng = (uint32_t)(n - 1);
        if (rng == 0) return 0;
        uint32_t ex = rng + 1u;
        uint64_t m = (uint64_t)next32() * ex;
        uint32_t lo = (uint32_t)m;
        if (lo < ex) {
            uint32_t th = (0xFFFFFFFFu - rng) % ex;
            while (lo < th) {
                m = (uint64_t)next32() * ex;
                lo = (uint32_t)m;
            }
        }
        return (int64_t)(m >> 32);
    }
};

// numpy pairwise_sum leaf (n <= 128)
__device__ double pw_leaf(const double *a, int64_t n, int64_t stride) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i * stride]);
        return r;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j * stride];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[(i + j) * stride]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i * stride]);
    return res;
}

// numpy pairwise_sum (loops_utils.h) over a[0..n): recursive halving at
// multiples of 8 above 128 elements, restated with an explicit stack.
__device__ double pw_sum(const double *a, int64_t n, int64_t stride) {
    if (n <= 128) return pw_leaf(a, n, stride);
    struct Frame {
        int64_t off, n;
        int state;
    };
    Frame fr[64];
    double vals[64];
    int fp = 0, vp = 0;
    fr[fp++] = {0, n, 0};
    while (fp) {
        Frame &f = fr[fp - 1];
        if (f.n <= 128) {
            vals[vp++] = pw_leaf(a + f.off * stride, f.n, stride);
            --fp;
            continue;
        }
        int64_t n2 = f.n / 2;
        n2 -= n2 % 8;
        if (f.state == 0) {
            f.state = 1;
            fr[fp++] = {f.off, n2, 0};
        } else if (f.state == 1) {
            f.state = 2;
            fr[fp++] = {f.off + n2, f.n - n2, 0};
        } else {
            double rgt = vals[--vp];
            double lft = vals[--vp];
            vals[vp++] = __dadd_rn(lft, rgt);
            --fp;
        }
    }
    return vals[0];
}

// row sum of (x_k - c_k)^2 over k < d, numpy order (pairwise over a tiny row)
template <class F>
__device__ __forceinline__ double row_pw(int d, F term) {
    if (d < 8) {
        double r = 0.0;
        for (int k = 0; k < d; ++k) r = __dadd_rn(r, term(k));
        return r;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = term(j);
    int i = 8;
    for (; i < d - (d % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], term(i + j));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < d; ++i) res = __dadd_rn(res, term(i));
    return res;
}

// BLAS-style dot (x @ c.T with a tiny K): fused multiply-add chain in k order
__device__ __forceinline__ double dot_fma(const double *x, const double *c, int d) {
    double acc = 0.0;
    for (int k = 0; k < d; ++k) acc = __fma_rn(x[k], c[k], acc);
    return acc;
}

constexpr int KM_K = 16;
constexpr int KM_MAXD = 32;

__global__ void __launch_bounds__(256) kmeans_kernel(
    const float *__restrict__ xs, int64_t ns, int ld, const int32_t *__restrict__ dims,
    const int32_t *__restrict__ offs, const int32_t *__restrict__ sel, int nsub,
    const Pcg64State *__restrict__ states, int iters, double *__restrict__ xbuf,
    double *__restrict__ d2buf, int32_t *__restrict__ abuf, float *__restrict__ cent_out, int dmax,
    double *__restrict__ hist_out) {
    const int i = blockIdx.x;
    const int d = dims[i];
    const int off = offs[i];
    const int n = nsub;
    double *x = xbuf + (size_t)i * nsub * KM_MAXD;  // row stride KM_MAXD
    double *d2 = d2buf + (size_t)i * nsub;
    int32_t *asg = abuf + (size_t)i * nsub;
    __shared__ double c[KM_K][KM_MAXD];
    __shared__ double csq[KM_K];
    __shared__ double sums[KM_K][KM_MAXD];
    __shared__ int64_t counts[KM_K];
    __shared__ int pick;
    const int tid = threadIdx.x;
    for (int t = tid; t < n; t += blockDim.x) {
        int64_t row = sel ? sel[(size_t)i * nsub + t] : t;
        for (int k = 0; k < d; ++k) x[(size_t)t * KM_MAXD + k] = (double)xs[row * ld + off + k];
    }
    __syncthreads();
    Pcg64 rng(states[i]);  // meaningful in thread 0 only
    // ---- k-means++ seeding (kmeans.py:16-32) ----
    if (tid == 0) pick = (int)rng.integers(n);
    __syncthreads();
    for (int k = tid; k < d; k += blockDim.x) c[0][k] = x[(size_t)pick * KM_MAXD + k];
    __syncthreads();
    for (int t = tid; t < n; t += blockDim.x) {
        const double *xt = x + (size_t)t * KM_MAXD;
        d2[t] = row_pw(d, [&](int k) {
            double e = __dsub_rn(xt[k], c[0][k]);
            return __dmul_rn(e, e);
        });
    }
    for (int j = 1; j < KM_K; ++j) {
        __syncthreads();
        if (tid == 0) {
            double total = pw_sum(d2, n, 1);
            if (total <= 0.0) {
                pick = -1 - (int)rng.integers(n);  // negative: no d2 update
            } else {
                double r = __dmul_rn(rng.random(), total);
                double cs = 0.0;
                int idx = n;
                for (int t = 0; t < n; ++t) {  // searchsorted(cumsum(d2), r), side=left
                    cs = __dadd_rn(cs, d2[t]);
                    if (cs >= r) {
                        idx = t;
                        break;
                    }
                }
                pick = idx < n - 1 ? idx : n - 1;
            }
        }
        __syncthreads();
        const int p = pick >= 0 ? pick : -1 - pick;
        for (int k = tid; k < d; k += blockDim.x) c[j][k] = x[(size_t)p * KM_MAXD + k];
        __syncthreads();
        if (pick >= 0) {
            for (int t = tid; t < n; t += blockDim.x) {
                const double *xt = x + (size_t)t * KM_MAXD;
                double nd = row_pw(d, [&](int k) {
                    double e = __dsub_rn(xt[k], c[j][k]);
                    return __dmul_rn(e, e);
                });
                d2[t] = fmin(d2[t], nd);
            }
        }
    }
    __syncthreads();
    // ---- Lloyd iterations (kmeans.py:57-75) ----
    double *xsq = d2;  // seeding distances are dead: reuse the buffer for ||x||^2
    for (int t = tid; t < n; t += blockDim.x) {
        const double *xt = x + (size_t)t * KM_MAXD;
        xsq[t] = row_pw(d, [&](int k) { return __dmul_rn(xt[k], xt[k]); });
    }
    extern __shared__ double bv[];  // clamped best distance per point (n doubles)
    for (int it = 0; it <= iters; ++it) {
        __syncthreads();
        if (tid < KM_K) csq[tid] = row_pw(d, [&](int k) { return __dmul_rn(c[tid][k], c[tid][k]); });
        __syncthreads();
        for (int t = tid; t < n; t += blockDim.x) {
            const double *xt = x + (size_t)t * KM_MAXD;
            int bj = 0;
            double bd = 0.0;
            for (int j = 0; j < KM_K; ++j) {
                double v = __dsub_rn(__dadd_rn(xsq[t], csq[j]), __dmul_rn(2.0, dot_fma(xt, c[j], d)));
                if (j == 0 || v < bd) {
                    bd = v;
                    bj = j;
                }
            }
            asg[t] = bj;
            bv[t] = bd > 0.0 ? bd : 0.0;
        }
        __syncthreads();
        if (tid == 0) hist_out[(size_t)i * (iters + 1) + it] = pw_sum(bv, n, 1);
        if (it == iters) break;
        // counts + sums in index order (np.bincount / np.add.at)
        for (int q = tid; q < KM_K * (d + 1); q += blockDim.x) {
            int j = q / (d + 1), k = q % (d + 1);
            if (k == d) {
                int64_t cnt = 0;
                for (int t = 0; t < n; ++t) cnt += (asg[t] == j);
                counts[j] = cnt;
            } else {
                double s = 0.0;
                for (int t = 0; t < n; ++t)
                    if (asg[t] == j) s = __dadd_rn(s, x[(size_t)t * KM_MAXD + k]);
                sums[j][k] = s;
            }
        }
        __syncthreads();
        for (int q = tid; q < KM_K * d; q += blockDim.x) {
            int j = q / d, k = q % d;
            if (counts[j] > 0) c[j][k] = __ddiv_rn(sums[j][k], (double)counts[j]);
        }
        __syncthreads();
        if (tid == 0) {
            for (int j = 0; j < KM_K; ++j) {
                if (counts[j] > 0) continue;
                int far = 0;
                double fv = bv[0];
                for (int t = 1; t < n; ++t)
                    if (bv[t] > fv) {
                        fv = bv[t];
                        far = t;
                    }
                for (int k = 0; k < d; ++k) c[j][k] = x[(size_t)far * KM_MAXD + k];
                bv[far] = 0.0;
            }
        }
        __syncthreads();
    }
    __syncthreads();
    for (int q = tid; q < KM_K * dmax; q += blockDim.x) {
        int j = q / dmax, k = q % dmax;
        cent_out[((size_t)i * KM_K + j) * dmax + k] = k < d ? __double2float_rn(c[j][k]) : 0.f;
    }
}

// Range statistics over the FULL training sample (flash.py:86-96): per
// subspace min/max of the raw SDT and of the clamped sample-to-centroid
// distances.  Non-negative doubles order like their int64 bit patterns.
__global__ void range_kernel(const float *__restrict__ xs, int64_t ns, int ld,
                             const int32_t *__restrict__ dims, const int32_t *__restrict__ offs,
                             const float *__restrict__ cent, int dmax,
                             unsigned long long *__restrict__ mn, unsigned long long *__restrict__ mx,
                             double *__restrict__ raw_sdt) {
    const int i = blockIdx.y;
    const int d = dims[i];
    const int off = offs[i];
    __shared__ double c[KM_K][KM_MAXD];
    __shared__ double cc[KM_K];
    for (int q = threadIdx.x; q < KM_K * d; q += blockDim.x)
        c[q / d][q % d] = (double)cent[((size_t)i * KM_K + q / d) * dmax + q % d];
    __syncthreads();
    if (threadIdx.x < KM_K)
        cc[threadIdx.x] = row_pw(d, [&](int k) {
            return __dmul_rn(c[threadIdx.x][k], c[threadIdx.x][k]);
        });
    __syncthreads();
    double lmin = 1.0 / 0.0, lmax = 0.0;
    if (blockIdx.x == 0) {  // raw SDT: ((c_a - c_b)^2).sum(2)
        for (int q = threadIdx.x; q < KM_K * KM_K; q += blockDim.x) {
            int a = q / KM_K, b = q % KM_K;
            double v = row_pw(d, [&](int k) {
                double e = __dsub_rn(c[a][k], c[b][k]);
                return __dmul_rn(e, e);
            });
            raw_sdt[(size_t)i * 256 + q] = v;
            lmin = fmin(lmin, v);
            lmax = fmax(lmax, v);
        }
    }
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ns;
         t += (int64_t)gridDim.x * blockDim.x) {
        double s[KM_MAXD];
        for (int k = 0; k < d; ++k) s[k] = (double)xs[t * ld + off + k];
        double ss = row_pw(d, [&](int k) { return __dmul_rn(s[k], s[k]); });
        for (int j = 0; j < KM_K; ++j) {
            double v = __dsub_rn(__dadd_rn(ss, cc[j]), __dmul_rn(2.0, dot_fma(s, c[j], d)));
            v = v > 0.0 ? v : 0.0;
            lmin = fmin(lmin, v);
            lmax = fmax(lmax, v);
        }
    }
    for (int o = 16; o; o >>= 1) {
        lmin = fmin(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
        lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mn + i, (unsigned long long)__double_as_longlong(lmin));
        atomicMax(mx + i, (unsigned long long)__double_as_longlong(lmax));
    }
}

// dist_min = min_i sub_min; dist_max = np.sum(sub_max) (pairwise order)
__global__ void range_final_kernel(const unsigned long long *mn, const unsigned long long *mx,
                                   int m, double *sub_max_scratch, double *out) {
    if (threadIdx.x != 0) return;
    double dmin = 1.0 / 0.0;
    for (int i = 0; i < m; ++i) {
        dmin = fmin(dmin, __longlong_as_double((long long)mn[i]));
        sub_max_scratch[i] = __longlong_as_double((long long)mx[i]);
    }
    out[0] = dmin;
    out[1] = pw_sum(sub_max_scratch, m, 1);
}

}  // namespace fa

using namespace fa;

extern "C" int fa_kmeans_subspaces_dev(const float *xs, int64_t ns, int ld, const int32_t *dims,
                                       const int32_t *offs, int m, const int32_t *sel, int nsub,
                                       const void *states, int iters, float *cent_out, int dmax,
                                       double *hist_out, void *scratch, void *stream) {
    FA_CHECK_ARG(m >= 1 && nsub >= KM_K && dmax >= 1 && dmax <= KM_MAXD && iters >= 0,
                 "bad k-means arguments");
    cudaStream_t st = as_stream(stream);
    double *xbuf = reinterpret_cast<double *>(scratch);
    double *d2 = xbuf + (size_t)m * nsub * KM_MAXD;
    int32_t *asg = reinterpret_cast<int32_t *>(d2 + (size_t)m * nsub);
    size_t smem = sizeof(double) * (size_t)nsub;
    FA_CHECK_ARG(smem <= 160 * 1024, "k-means sample too large");
    if (smem > 48 * 1024)
        FA_CUDA(cudaFuncSetAttribute(kmeans_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    kmeans_kernel<<<m, 256, smem, st>>>(xs, ns, ld, dims, offs, sel, nsub,
                                         reinterpret_cast<const Pcg64State *>(states), iters, xbuf,
                                         d2, asg, cent_out, dmax, hist_out);
    FA_LAUNCH_CHECK();
    return FA_OK;
}

// k-means subsample rows of every subspace on the host cores:
// np.sort(default_rng(seed + i).permutation(ns)[:cap]) (kmeans.py:50-54) —
// numpy's shuffle of arange(ns) (Fisher-Yates from the top, j =
// random_interval(i)) replayed from the generator's state, which is left as
// numpy leaves it.  The subspaces run on parallel threads.
extern "C" int fa_kmeans_subsample(int64_t ns, int cap, int m, void *states, int32_t *sel) {
    FA_CHECK_ARG(ns >= 1 && cap >= 1 && cap <= ns && m >= 1 && states && sel,
                 "bad subsample arguments");
    FA_CHECK_ARG(ns <= 0x7fffffffll, "sample of %lld rows too large", (long long)ns);
    Pcg64State *st = reinterpret_cast<Pcg64State *>(states);
    const int T = std::max(1, std::min<int>(m, (int)std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([=]() {
            std::vector<int32_t> a((size_t)ns);
            for (int i = t; i < m; i += T) {
                Pcg64 rng(st[i]);
                for (int64_t k = 0; k < ns; ++k) a[k] = (int32_t)k;
                for (int64_t k = ns - 1; k > 0; --k) std::swap(a[k], a[rng.interval((uint64_t)k)]);
                int32_t *out = sel + (size_t)i * cap;
                std::copy(a.begin(), a.begin() + cap, out);
                std::sort(out, out + cap);
                rng.store(st[i]);
            }
        });
    for (auto &x : th) x.join();
    return FA_OK;
}

extern "C" size_t fa_kmeans_scratch_bytes(int m, int nsub) {
    return sizeof(double) * (size_t)m * nsub * (KM_MAXD + 1) + sizeof(int32_t) * (size_t)m * nsub;
}

extern "C" int fa_flash_range_dev(const float *xs, int64_t ns, int ld, const int32_t *dims,
                                  const int32_t *offs, int m, const float *cent, int dmax,
                                  double *raw_sdt, double *range_out, void *scratch, void *stream) {
    FA_CHECK_ARG(m >= 1 && dmax <= KM_MAXD, "bad range arguments");
    cudaStream_t st = as_stream(stream);
    unsigned long long *mn = reinterpret_cast<unsigned long long *>(scratch);
    unsigned long long *mx = mn + m;
    double *tmp = reinterpret_cast<double *>(mx + m);
    FA_CUDA(cudaMemsetAsync(mn, 0x7f, sizeof(unsigned long long) * m, st));
    FA_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned long long) * m, st));
    int gx = (int)((ns + 255) / 256);
    if (gx > 64) gx = 64;
    if (gx < 1) gx = 1;
    range_kernel<<<dim3(gx, m), 256, 0, st>>>(xs, ns, ld, dims, offs, cent, dmax, mn, mx, raw_sdt);
    FA_LAUNCH_CHECK();
    range_final_kernel<<<1, 32, 0, st>>>(mn, mx, m, tmp, range_out);
    FA_LAUNCH_CHECK();
    return FA_OK;
}
