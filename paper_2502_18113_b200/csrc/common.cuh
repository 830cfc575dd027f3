// Shared device/host helpers for the sm_100a Flash core.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <functional>
#include <string>

#include "../../include/flashann_b200.h"

namespace fa {

// ---- error plumbing (fa_last_error) ---------------------------------------
void set_error(const char *fmt, ...);

#define FA_CHECK_ARG(cond, ...)            \
    do {                                   \
        if (!(cond)) {                     \
            ::fa::set_error(__VA_ARGS__);  \
            return FA_EINVAL;              \
        }                                  \
    } while (0)

#define FA_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t _e = (call);                                                        \
        if (_e != cudaSuccess) {                                                        \
            ::fa::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,                  \
                            cudaGetErrorString(_e));                                    \
            return FA_ECUDA;                                                            \
        }                                                                               \
    } while (0)

#define FA_LAUNCH_CHECK() FA_CUDA(cudaGetLastError())

#define FA_TRY(call)                 \
    do {                             \
        int _rc = (call);            \
        if (_rc != FA_OK) return _rc; \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kWarp = 32;
constexpr int kNumSMs = 148;  // B200; grids use num_sms() (the device's own count)

// ---- device memory from the stream-ordered pool -----------------------------
// The core's device buffers (index arrays, host drop-in staging targets,
// build scratch) come from the device's default memory pool with its release
// threshold raised (to a quarter of the device), so the repeated create/free of the host drop-ins reuses
// mapped memory instead of paying cudaMalloc / cudaFree (which unmap and
// synchronise) on every call.  Allocation and free are ordered on the legacy
// default stream; pool_alloc waits for that stream so the buffer is usable on
// any stream.
inline void keep_pool() {
    static unsigned long long done = 0;  // one bit per device ordinal < 64
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64 || ((done >> dev) & 1ull)) return;
    cudaMemPool_t pool;
    size_t free_b = 0, total_b = 0;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess &&
        cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
        // keep up to a quarter of the device mapped between calls; anything
        // above goes back at the next synchronisation (other allocators, e.g.
        // PyTorch's, cannot use memory parked in this pool)
        uint64_t keep = (uint64_t)total_b / 4;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done |= 1ull << dev;
}
inline int pool_alloc(void **p, size_t bytes) {
    keep_pool();
    cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 16, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    if (e != cudaSuccess) {
        *p = nullptr;
        set_error("device allocation of %zu bytes: %s", bytes, cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? FA_ENOMEM : FA_ECUDA;
    }
    return FA_OK;
}
inline void pool_free(void *p) {
    if (p) cudaFreeAsync(p, 0);
}

// Internal (C++) hooks of the index for the host drop-ins (csrc/index.cu).
int index_encode_rows(fa_index *ix, int64_t r0, int64_t r1, cudaStream_t st);
void index_set_late_rows(fa_index *ix, int64_t from, std::function<int(cudaStream_t)> hook);

// SM count of the current device (cached per process; B200: 148)
inline int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
            n = v;
        else
            n = kNumSMs;
    }
    return n;
}

__host__ __device__ inline int round_up(int x, int a) { return (x + a - 1) / a * a; }
__host__ __device__ inline int64_t round_up64(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// ---- numerics pinned to the reference build -------------------------------

// fa_quantize (_simd.h:99-107): IEEE double, divide then multiply, floor.
__device__ __forceinline__ uint8_t quantize_dev(double d, double dmin, double delta) {
    double dmax = __dadd_rn(dmin, delta);
    if (d >= dmax) return 255;
    if (d < dmin) d = dmin;
    double t = floor(__dmul_rn(__ddiv_rn(__dsub_rn(d, dmin), delta), 255.0));
    if (t >= 255.0) return 255;
    if (t <= 0.0) return 0;
    return (uint8_t)t;
}

// fa_l2sq_f32 (_simd.h:44-51) exactly as gcc -O3 -march=native -ffast-math
// lowers it on the reference host (AVX2 256-bit vectors):
//   d >= 8 : 8 lane accumulators acc[k] += fl(e*e) (mul then add, no FMA) over
//            full chunks; v[k] = acc[k] + acc[k+4]; if a 4-wide remainder
//            exists, w[k] = fma(e,e,v[k]) and s = (w0+w2)+(w1+w3), else
//            s = (v0+v2)+(v1+v3); scalar tail s = fma(e,e,s).
//   d <  8 : 4-wide block w[k] = fl(e*e) when d >= 4, s = (w0+w2)+(w1+w3);
//            scalar tail s = fma(e,e,s) starting from 0.
// Pinned bit-for-bit against the compiled reference (tests/golden).
template <typename Load>
__device__ __forceinline__ float l2_tree(int d, Load ld) {
    int i = 0;
    float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;
    float s;
    bool have_v = false;
    if (d >= 8) {
        float a[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = 0.f;
#pragma unroll
        for (; i + 8 <= d; i += 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                float e = ld(i + k);
                a[k] = __fadd_rn(a[k], __fmul_rn(e, e));
            }
        }
        v0 = __fadd_rn(a[0], a[4]);
        v1 = __fadd_rn(a[1], a[5]);
        v2 = __fadd_rn(a[2], a[6]);
        v3 = __fadd_rn(a[3], a[7]);
        have_v = true;
    }
    if (d - i >= 4) {
        float e0 = ld(i), e1 = ld(i + 1), e2 = ld(i + 2), e3 = ld(i + 3);
        float w0 = __fmaf_rn(e0, e0, v0), w1 = __fmaf_rn(e1, e1, v1);
        float w2 = __fmaf_rn(e2, e2, v2), w3 = __fmaf_rn(e3, e3, v3);
        s = __fadd_rn(__fadd_rn(w0, w2), __fadd_rn(w1, w3));
        i += 4;
    } else if (have_v) {
        s = __fadd_rn(__fadd_rn(v0, v2), __fadd_rn(v1, v3));
    } else {
        s = 0.f;
    }
#pragma unroll
    for (; i < d; ++i) {
        float e = ld(i);
        s = __fmaf_rn(e, e, s);
    }
    return s;
}

// ---- warp helpers ----------------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

// 16-entry byte table (t0..t3 = bytes 0..15) looked up by the four 4-bit codes
// held in the bytes of w (each byte < 16): returns the four table bytes.
__device__ __forceinline__ uint32_t lut16x4(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3,
                                            uint32_t w) {
    uint32_t y = w | (w >> 4);               // byte0 = c0|c1<<4, byte2 = c2|c3<<4
    uint32_t sel = prmt(y, 0u, 0x3320u);     // nibbles c0,c1,c2,c3 (bit 3 ignored below)
    uint32_t sel7 = sel & 0x7777u;           // plain byte select mode
    uint32_t lo = prmt(t0, t1, sel7);        // table[c & 7]
    uint32_t hi = prmt(t2, t3, sel7);        // table[8 + (c & 7)]
    uint32_t msk = prmt(w << 4, 0u, 0xBA98u);// 0xFF where code bit 3 set (sign replicate)
    return (lo & ~msk) | (hi & msk);
}

}  // namespace fa
