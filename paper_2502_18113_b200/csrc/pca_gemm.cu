// K9: the PCA contractions on the 5th-generation tensor cores.
//
//   covariance  cov = (X - mean)^T (X - mean) / n      (providers/pca.py:36-38)
//   projection  Y   = (X - mean) @ basis[:, :d]         (providers/pca.py:68-71)
//
// The reference computes both in fp32 (numpy sgemm over the float32-centred
// rows).  Here they run as 3xTF32 on tcgen05: every fp32 operand x is split
// into hi = rna_tf32(x) and lo = x - hi (exact in fp32), and each stage's
// product is hi*hi + (lo*hi + hi*lo) — fp32-class accuracy (the dropped lo*lo
// term is 2^-22 relative) at tensor-core rate.
//
// Accumulation: the tensor core's fp32 accumulator does not round to nearest
// (it truncates after aligning to the largest term), so a long chain of MMAs
// into one TMEM tile drifts (4.6e-6 relative over 375 MMAs, measured, against
// 3e-7 for the reference's sgemm).  The hi*hi term of each stage (K = 32, 4
// MMAs) therefore goes into a fresh TMEM accumulator, which the epilogue warps
// add into fp32 running sums in registers with round-to-nearest FADDs; two
// such accumulators alternate, so the epilogue drains one while the tensor
// core fills the other.  The two cross terms (lo*hi, hi*lo) are 2^-11 smaller,
// so their truncation drift is ~2^-11 smaller too: they accumulate over the
// whole tile in a third accumulator (double-buffered across tiles) drained
// once at the end.
//
// One persistent CTA per SM, warp-specialised (448 threads):
//   warp 0      TMA producer: raw X tiles (and, for the projection, the
//               pre-split basis tiles hi/lo, already in the UMMA K-major
//               128-byte-swizzled layout) into a 2-stage shared-memory ring;
//   warp 1      TMEM allocator and MMA issuer: one thread issues
//               tcgen05.mma.kind::tf32 (M = 128, N = 128, K = 8), 12 per stage;
//   warps 2-5   converters: raw tile -> centred (x - mean, the reference's
//               fp32 subtraction; bf16 inputs are widened exactly) -> hi/lo
//               written in the K-major SW128 layout (transposed for the
//               covariance, whose contraction runs over the rows of X);
//   warps 6-13  epilogue: tcgen05.ld of the accumulators (lane quarter =
//               warp % 4, column half = (warp - 6) / 4) -> register sums ->
//               global fp32 at the end of the tile.
// Barriers: full (TMA -> converters, transaction bytes), conv (converters ->
// MMA), empty (MMA commit -> TMA), tfull / tempty (MMA <-> epilogue, per
// stage, the hi*hi accumulators), sfull / sempty (per tile, the cross-term
// accumulators).
//
// The covariance is symmetric: only tiles with n-block >= m-block are
// computed, split over K (rows of X) into per-split fp32 partials that a
// second kernel sums in float64 in a fixed order (deterministic) and mirrors.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace fa {
namespace pg {

constexpr int BM = 128;   // tile rows (MMA M, TMEM lanes)
constexpr int BK = 32;    // fp32 elements per 128-byte swizzle row = one stage's K
// 14 warps (4 converter warps: the conversion is on the critical path); with
// 4 warps on some SM sub-partitions a thread holds at most 128 registers, so
// the epilogue drains TMEM 16 columns at a time
constexpr int kConvWarps = 4, kEpiWarps = 8;
constexpr int kConvThreads = 32 * kConvWarps;
constexpr int kThreads = 32 * (2 + kConvWarps + kEpiWarps);
constexpr int kConvWarp0 = 2, kEpiWarp0 = kConvWarp0 + kConvWarps;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_2d(void *dst, const CUtensorMap *map, int c0, int c1,
                                       uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32, both operands K-major
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row atoms of
// 1024 B (SBO), version 1 (sm_100), LBO unused for swizzled K-major (1)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;
    d |= (uint64_t)(1024u >> 4) << 32;
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)2u << 61;
    return d;
}
// instruction descriptor: D f32, A/B tf32, K-major both, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(BM >> 4) << 24);
}
// 16 consecutive fp32 columns of this thread's TMEM lane (32x32b.x16)
__device__ __forceinline__ void tmem_ld16(uint32_t ta, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,"
        "%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(ta));
}
__device__ __forceinline__ float rna_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
// byte offset of (row, 16-byte chunk) in a K-major SW128 tile
__device__ __forceinline__ uint32_t sw128(int row, int chunk) {
    return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((chunk ^ (row & 7)) << 4));
}
__device__ __forceinline__ void split_store(uint8_t *hi, uint8_t *lo, uint32_t off, float4 a) {
    float4 h, l;
    h.x = rna_tf32(a.x); l.x = a.x - h.x;
    h.y = rna_tf32(a.y); l.y = a.y - h.y;
    h.z = rna_tf32(a.z); l.z = a.z - h.z;
    h.w = rna_tf32(a.w); l.w = a.w - h.w;
    *reinterpret_cast<float4 *>(hi + off) = h;
    *reinterpret_cast<float4 *>(lo + off) = l;
}
__device__ __forceinline__ float widen(float x) { return x; }
__device__ __forceinline__ float widen(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
struct Tile {
    // raw tile bytes (TMA box) and converted operand tiles
    static constexpr int raw_bytes = BM * BK * (int)sizeof(T);
    static constexpr int op_bytes = BM * BK * 4;  // 16 KB per hi / lo tile of 128 rows
};

// Shared memory: three rings with their own depths, so the TMA loads run
// ahead of the conversion and of the MMAs instead of waiting for a whole
// stage to retire:
//   raw ring  (RS stages, freed by the converters once read): raw X tiles
//             (COV: the A and the B column blocks);
//   B ring    (BS stages, freed by the MMA commit; projection only): the
//             pre-split basis tiles hi / lo, TMA'd straight into UMMA layout;
//   op ring   (2 stages, freed by the MMA commit): the converted hi / lo
//             tiles (COV: A and B).
template <bool COV, int BN, typename T>
struct Layout {
    static constexpr int raw = Tile<T>::raw_bytes;
    static constexpr int raw_pad = (raw + 1023) / 1024 * 1024;
    static constexpr int a_op = Tile<T>::op_bytes;
    static constexpr int b_op = BN * BK * 4;
    static constexpr int RS = COV ? (sizeof(T) == 4 ? 2 : 3) : (sizeof(T) == 4 ? 3 : 4);
    static constexpr int BS = COV ? 0 : 3;
    static constexpr int OS = 2;
    static constexpr int raw_stage = raw_pad * (COV ? 2 : 1);
    static constexpr int b_stage = 2 * b_op;                      // hi, lo
    static constexpr int op_stage = 2 * a_op + (COV ? 2 * b_op : 0);  // A hi, lo (+ B hi, lo)
    static constexpr int off_raw = 0;
    static constexpr int off_b = off_raw + RS * raw_stage;
    static constexpr int off_op = off_b + BS * b_stage;
    static constexpr int bars = off_op + OS * op_stage;  // barrier block after the rings
    static constexpr int total = bars + 512 + 1024;      // + barriers + alignment slack
    static_assert(total <= 227 * 1024, "shared memory");
    // raw stage: rawA at 0, rawB at raw_pad; op stage: Ahi, Alo, Bhi, Blo
    static constexpr int off_ahi = 0, off_alo = a_op, off_bhi = 2 * a_op,
                         off_blo = 2 * a_op + b_op;
};

struct Params {
    int64_t n;        // rows of X
    int D;            // columns of X (logical)
    int d;            // PROJ: output columns
    const float *mean;  // D fp32 (the reference's float32-cast mean)
    float *out;         // PROJ: n x ldo; COV: nsplit x D x D partials
    int64_t ldo;
    int nm, nn;         // PROJ: m-tiles, n-tiles
    int nb;             // COV: 128-blocks along D
    int nsplit;         // COV: K splits
    int nk;             // k-blocks per work item (PROJ) / in total (COV)
    int64_t nwork;
};

// COV work item w -> (mb, nb, split): triangle index t = w / nsplit over
// pairs mb <= nb (row-major), split = w % nsplit
__device__ __forceinline__ void cov_item(const Params &p, int64_t w, int &mb, int &nb, int &sp) {
    sp = (int)(w % p.nsplit);
    int t = (int)(w / p.nsplit);
    mb = 0;
    while (t >= p.nb - mb) {
        t -= p.nb - mb;
        ++mb;
    }
    nb = mb + t;
}
__device__ __forceinline__ void cov_krange(const Params &p, int sp, int &k0, int &k1) {
    const int per = (p.nk + p.nsplit - 1) / p.nsplit;
    k0 = sp * per;
    k1 = min(p.nk, k0 + per);
}

template <bool COV, int BN, typename T>
__global__ void __launch_bounds__(kThreads, 1)
    pca_gemm_kernel(const __grid_constant__ CUtensorMap mapX,
                    const __grid_constant__ CUtensorMap mapBhi,
                    const __grid_constant__ CUtensorMap mapBlo, Params p) {
    using L = Layout<COV, BN, T>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem =
        reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    uint64_t *raw_full = reinterpret_cast<uint64_t *>(smem + L::bars);
    uint64_t *raw_empty = raw_full + L::RS;
    uint64_t *b_full = raw_empty + L::RS;
    uint64_t *b_empty = b_full + 4;
    uint64_t *op_full = b_empty + 4;
    uint64_t *op_empty = op_full + L::OS;
    uint64_t *tfull = op_empty + L::OS;
    uint64_t *tempty = tfull + 2;
    uint64_t *sfull = tempty + 2;
    uint64_t *sempty = sfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sempty + 2);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // TMEM: hi*hi accumulators of stages (2 x BN columns), then the cross-term
    // accumulators of tiles (2 x BN)
    constexpr uint32_t kTmemCols = 4 * BN;
    static_assert(4 * BN <= 512, "TMEM holds 512 fp32 columns");

    if (threadIdx.x == 0) {
        for (int s = 0; s < L::RS; ++s) {
            mbar_init(raw_full + s, 1);
            mbar_init(raw_empty + s, kConvThreads);
        }
        for (int s = 0; s < L::BS; ++s) {
            mbar_init(b_full + s, 1);
            mbar_init(b_empty + s, 1);
        }
        for (int s = 0; s < L::OS; ++s) {
            mbar_init(op_full + s, kConvThreads);
            mbar_init(op_empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, 256);
            mbar_init(sfull + a, 1);
            mbar_init(sempty + a, 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===== TMA producer: raw tiles run up to RS stages ahead of the
        // converters, basis tiles up to BS stages ahead of the MMAs =====
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapX)));
            int rs = 0, bs = 0;
            uint32_t rph = 0, bph = 0;
            for (int64_t w = blockIdx.x; w < p.nwork; w += gridDim.x) {
                int k0, k1, m0, n0;
                bool diag = false;
                if constexpr (COV) {
                    int mb, nb, sp;
                    cov_item(p, w, mb, nb, sp);
                    cov_krange(p, sp, k0, k1);
                    m0 = mb * BM;
                    n0 = nb * BM;
                    diag = mb == nb;
                } else {
                    m0 = (int)(w / p.nn) * BM;
                    n0 = (int)(w % p.nn) * BN;
                    k0 = 0;
                    k1 = p.nk;
                }
                for (int kb = k0; kb < k1; ++kb) {
                    mbar_wait(raw_empty + rs, rph ^ 1);
                    uint8_t *rst = smem + L::off_raw + rs * L::raw_stage;
                    if constexpr (COV) {
                        // X[k rows, m / n column blocks]: box {BM cols, BK rows}
                        mbar_expect_tx(raw_full + rs, (diag ? 1 : 2) * L::raw);
                        tma_2d(rst, &mapX, m0, kb * BK, raw_full + rs);
                        if (!diag) tma_2d(rst + L::raw_pad, &mapX, n0, kb * BK, raw_full + rs);
                    } else {
                        mbar_expect_tx(raw_full + rs, L::raw);
                        tma_2d(rst, &mapX, kb * BK, m0, raw_full + rs);
                    }
                    if (++rs == L::RS) {
                        rs = 0;
                        rph ^= 1;
                    }
                    if constexpr (!COV) {
                        mbar_wait(b_empty + bs, bph ^ 1);
                        uint8_t *bst = smem + L::off_b + bs * L::b_stage;
                        mbar_expect_tx(b_full + bs, L::b_stage);
                        tma_2d(bst, &mapBhi, kb * BK, n0, b_full + bs);
                        tma_2d(bst + L::b_op, &mapBlo, kb * BK, n0, b_full + bs);
                        if (++bs == L::BS) {
                            bs = 0;
                            bph ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer: every stage into a fresh accumulator pair =====
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(BN);
            int s = 0, bs = 0;  // op ring, B ring
            uint32_t ph = 0, bph = 0;
            uint32_t fl = 0;  // stages flushed so far (hi*hi accumulator = fl & 1)
            uint32_t it = 0;  // tiles so far (cross-term accumulator = it & 1)
            for (int64_t w = blockIdx.x; w < p.nwork; w += gridDim.x, ++it) {
                int k0, k1;
                bool diag = false;
                if constexpr (COV) {
                    int mb, nb, sp;
                    cov_item(p, w, mb, nb, sp);
                    cov_krange(p, sp, k0, k1);
                    diag = mb == nb;
                } else {
                    k0 = 0;
                    k1 = p.nk;
                }
                const uint32_t sa = it & 1u;
                mbar_wait(sempty + sa, ((it >> 1) & 1u) ^ 1u);
                const uint32_t d_small = tmem_base + 2 * BN + sa * BN;
                for (int kb = k0; kb < k1; ++kb, ++fl) {
                    const uint32_t acc = fl & 1u;
                    mbar_wait(tempty + acc, ((fl >> 1) & 1u) ^ 1u);
                    mbar_wait(op_full + s, ph);
                    if constexpr (!COV) mbar_wait(b_full + bs, bph);
                    tc_fence_after();
                    const uint32_t d_big = tmem_base + acc * BN;
                    uint8_t *ost = smem + L::off_op + s * L::op_stage;
                    const uint32_t ahi = smem_u32(ost + L::off_ahi), alo = smem_u32(ost + L::off_alo);
                    uint32_t bhi, blo;
                    if constexpr (COV) {
                        bhi = diag ? ahi : smem_u32(ost + L::off_bhi);
                        blo = diag ? alo : smem_u32(ost + L::off_blo);
                    } else {
                        uint8_t *bst = smem + L::off_b + bs * L::b_stage;
                        bhi = smem_u32(bst);
                        blo = smem_u32(bst + L::b_op);
                    }
#pragma unroll
                    for (int k = 0; k < BK / 8; ++k) {
                        const uint32_t o = (uint32_t)k * 32u;  // 8 tf32 = 32 bytes along K
                        const uint32_t more = k > 0 ? 1u : 0u;
                        const uint32_t smore = (kb > k0 || k > 0) ? 1u : 0u;
                        mma_tf32(d_big, sdesc(ahi + o), sdesc(bhi + o), idesc, more);
                        mma_tf32(d_small, sdesc(alo + o), sdesc(bhi + o), idesc, smore);
                        mma_tf32(d_small, sdesc(ahi + o), sdesc(blo + o), idesc, 1u);
                    }
                    tc_commit(op_empty + s);  // the converted tiles are free once these retire
                    if constexpr (!COV) {
                        tc_commit(b_empty + bs);  // and the basis tiles
                        if (++bs == L::BS) {
                            bs = 0;
                            bph ^= 1;
                        }
                    }
                    tc_commit(tfull + acc);  // the hi*hi sums are ready to drain
                    if (++s == L::OS) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                tc_commit(sfull + sa);  // the tile's cross terms are complete
            }
        }
    } else if (warp >= kConvWarp0 && warp < kEpiWarp0) {
        // ===== converters: raw -> centred -> hi / lo, K-major SW128 =====
        const int t = threadIdx.x - kConvWarp0 * 32;  // 0 .. kConvThreads - 1
        int rs = 0, s = 0;  // raw ring, op ring
        uint32_t rph = 0, ph = 0;
        for (int64_t w = blockIdx.x; w < p.nwork; w += gridDim.x) {
            int k0, k1, m0 = 0, n0 = 0;
            bool diag = false;
            if constexpr (COV) {
                int mb, nb, sp;
                cov_item(p, w, mb, nb, sp);
                cov_krange(p, sp, k0, k1);
                m0 = mb * BM;
                n0 = nb * BM;
                diag = mb == nb;
            } else {
                k0 = 0;
                k1 = p.nk;
            }
            for (int kb = k0; kb < k1; ++kb) {
                mbar_wait(raw_full + rs, rph);
                mbar_wait(op_empty + s, ph ^ 1);
                const uint8_t *rst = smem + L::off_raw + rs * L::raw_stage;
                uint8_t *st = smem + L::off_op + s * L::op_stage;
                if constexpr (COV) {
                    // thread t owns columns t, t + kConvThreads, ... of the
                    // block: rows k of the raw tile become the K of operand
                    // row t (a transpose)
                    for (int op = 0; op < (diag ? 1 : 2); ++op)
                    for (int tc = t; tc < BM; tc += kConvThreads) {
                        const int col = (op ? n0 : m0) + tc;
                        const bool cin = col < p.D;
                        const float mu = cin ? __ldg(p.mean + col) : 0.f;
                        const T *raw = reinterpret_cast<const T *>(rst + (op ? L::raw_pad : 0));
                        uint8_t *hi = st + (op ? L::off_bhi : L::off_ahi);
                        uint8_t *lo = st + (op ? L::off_blo : L::off_alo);
                        const int64_t kr0 = (int64_t)kb * BK;
#pragma unroll
                        for (int c = 0; c < BK / 4; ++c) {
                            float4 a;
                            float *av = reinterpret_cast<float *>(&a);
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const int kr = 4 * c + j;
                                const bool in = cin && kr0 + kr < p.n;
                                av[j] = in ? widen(raw[kr * BM + tc]) - mu : 0.f;
                            }
                            split_store(hi, lo, sw128(tc, c), a);
                        }
                    }
                } else {
                    const T *raw = reinterpret_cast<const T *>(rst);
                    uint8_t *hi = st + L::off_ahi;
                    uint8_t *lo = st + L::off_alo;
                    constexpr int per16 = 16 / (int)sizeof(T);  // elements per 16-byte chunk
                    constexpr int cpr = BK / per16;             // chunks per raw row
                    constexpr int iters = BM * cpr / kConvThreads;
                    const int ch = t % cpr;  // fixed per thread
                    float mu[per16];
#pragma unroll
                    for (int j = 0; j < per16; ++j) {
                        const int k = kb * BK + ch * per16 + j;
                        mu[j] = k < p.D ? __ldg(p.mean + k) : 0.f;
                    }
#pragma unroll
                    for (int i = 0; i < iters; ++i) {
                        const int idx = t + kConvThreads * i;
                        const int row = idx / cpr;
                        const uint4 v = *reinterpret_cast<const uint4 *>(raw + row * BK + ch * per16);
                        const T *e = reinterpret_cast<const T *>(&v);
                        float f[per16];
#pragma unroll
                        for (int j = 0; j < per16; ++j) {
                            const int k = kb * BK + ch * per16 + j;
                            f[j] = k < p.D ? widen(e[j]) - mu[j] : 0.f;
                        }
#pragma unroll
                        for (int q = 0; q < per16 / 4; ++q)
                            split_store(hi, lo, sw128(row, ch * (per16 / 4) + q),
                                        make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]));
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(raw_empty + rs);  // the raw tile is consumed
                mbar_arrive(op_full + s);     // the converted tiles are ready
                if (++rs == L::RS) {
                    rs = 0;
                    rph ^= 1;
                }
                if (++s == L::OS) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp >= kEpiWarp0) {
        // ===== epilogue: per stage TMEM -> register sums; per tile -> global =====
        constexpr int HC = BN / 2;  // columns per epilogue warp (its half)
        const int q = warp & 3;     // TMEM lane quarter this warp may access
        const int h = (warp - kEpiWarp0) >> 2;
        const int r = 32 * q + lane;
        uint32_t fl = 0, it = 0;
        for (int64_t w = blockIdx.x; w < p.nwork; w += gridDim.x, ++it) {
            int m0, n0, k0, k1;
            float *dst;
            int64_t ld;
            int ncol;
            if constexpr (COV) {
                int mb, nb, sp;
                cov_item(p, w, mb, nb, sp);
                cov_krange(p, sp, k0, k1);
                m0 = mb * BM;
                n0 = nb * BM;
                dst = p.out + (size_t)sp * p.D * p.D;
                ld = p.D;
                ncol = p.D;
            } else {
                m0 = (int)(w / p.nn) * BM;
                n0 = (int)(w % p.nn) * BN;
                k0 = 0;
                k1 = p.nk;
                dst = p.out;
                ld = p.ldo;
                ncol = p.d;
            }
            const int64_t nrow = COV ? (int64_t)p.D : p.n;
            float sum[HC];
#pragma unroll
            for (int j = 0; j < HC; ++j) sum[j] = 0.f;
            const uint32_t lanebase = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(h * HC);
            for (int kb = k0; kb < k1; ++kb, ++fl) {
                const uint32_t acc = fl & 1u;
                mbar_wait(tfull + acc, (fl >> 1) & 1u);
                tc_fence_after();
                const uint32_t tb = lanebase + acc * BN;
#pragma unroll
                for (int c = 0; c < HC / 16; ++c) {
                    uint32_t vb[16];
                    tmem_ld16(tb + 16 * c, vb);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 16; ++j) sum[16 * c + j] += __uint_as_float(vb[j]);
                }
                tc_fence_before();
                mbar_arrive(tempty + acc);
            }
            {  // the tile's cross terms, once
                const uint32_t sa = it & 1u;
                mbar_wait(sfull + sa, (it >> 1) & 1u);
                tc_fence_after();
                const uint32_t tb = lanebase + 2 * BN + sa * BN;
#pragma unroll
                for (int c = 0; c < HC / 16; ++c) {
                    uint32_t vs[16];
                    tmem_ld16(tb + 16 * c, vs);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 16; ++j) sum[16 * c + j] += __uint_as_float(vs[j]);
                }
                tc_fence_before();
                mbar_arrive(sempty + sa);
            }
            const int64_t row = (int64_t)m0 + r;
            const int col0 = n0 + h * HC;
            if (row < nrow) {
                float *orow = dst + row * ld;
                if (col0 + HC <= ncol && (ld & 3) == 0) {
#pragma unroll
                    for (int j = 0; j < HC; j += 4)
                        *reinterpret_cast<float4 *>(orow + col0 + j) =
                            make_float4(sum[j], sum[j + 1], sum[j + 2], sum[j + 3]);
                } else {
#pragma unroll
                    for (int j = 0; j < HC; ++j)
                        if (col0 + j < ncol) orow[col0 + j] = sum[j];
                }
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(kTmemCols)
                     : "memory");
    }
}

// hi / lo split of the transposed basis: bt (d x ldb) -> bhi, blo (d x ldb)
__global__ void split_basis_kernel(const float *__restrict__ basis, int D, int dfull, int d,
                                   int ldb, float *__restrict__ bhi, float *__restrict__ blo) {
    // basis: D x dfull row-major (columns by descending eigenvalue); output
    // row j = column j of basis[:, :d], zero padded to ldb
    const int64_t total = (int64_t)d * ldb;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(i / ldb), k = (int)(i % ldb);
        const float x = k < D ? basis[(int64_t)k * dfull + j] : 0.f;
        const float h = rna_tf32(x);
        bhi[i] = h;
        blo[i] = x - h;
    }
}

// cov[i][j] = sum_s part[s][min(i,j)][max(i,j)] / n in float64 (exactly symmetric)
__global__ void cov_reduce_kernel(const float *__restrict__ part, int nsplit, int D, double inv_n,
                                  double *__restrict__ cov) {
    const int64_t total = (int64_t)D * D;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        int i = (int)(e / D), j = (int)(e % D);
        if (i > j) {  // lower triangle: the mirrored (computed) element -> exact symmetry
            const int t = i;
            i = j;
            j = t;
        }
        double s = 0.0;
        for (int k = 0; k < nsplit; ++k) s += (double)part[(size_t)k * D * D + (size_t)i * D + j];
        cov[e] = s * inv_n;
    }
}

// ---- host side ---------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 2-D row-major map: inner dim `cols` (contiguous), outer `rows`, row pitch
// `pitch` bytes, box {bcols, brows}
static int make_map(CUtensorMap *m, const void *base, bool bf16, uint64_t cols, uint64_t rows,
                    uint64_t pitch, uint32_t bcols, uint32_t brows, bool swizzle128) {
    auto fn = encode_fn();
    if (!fn) {
        set_error("cuTensorMapEncodeTiled is unavailable from the driver");
        return FA_ECUDA;
    }
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {pitch};
    cuuint32_t box[2] = {bcols, brows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                    const_cast<void *>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d): dims %llu x %llu pitch %llu box %u x %u",
                  (int)r, (unsigned long long)cols, (unsigned long long)rows,
                  (unsigned long long)pitch, bcols, brows);
        return FA_ECUDA;
    }
    return FA_OK;
}

template <bool COV, int BN, typename T>
static int launch(const CUtensorMap &mx, const CUtensorMap &mbh, const CUtensorMap &mbl,
                  const Params &p, cudaStream_t st) {
    using L = Layout<COV, BN, T>;
    auto k = pca_gemm_kernel<COV, BN, T>;
    FA_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L::total));
    const int grid = (int)std::min<int64_t>(p.nwork, num_sms());
    k<<<grid, kThreads, L::total, st>>>(mx, mbh, mbl, p);
    FA_LAUNCH_CHECK();
    return FA_OK;
}

// X rows must satisfy the TMA pitch rule (a multiple of 16 bytes); a narrow
// or odd-width X is first copied into a zero-padded buffer (zero columns
// contribute nothing once centred with a zero mean entry).
struct Padded {
    const void *x = nullptr;
    const float *mean = nullptr;
    int ldx = 0;
    void *own_x = nullptr;
    float *own_mean = nullptr;
    cudaStream_t st = nullptr;
    ~Padded() {  // stream-ordered: the kernels that read the copies run first
        if (own_x) cudaFreeAsync(own_x, st);
        if (own_mean) cudaFreeAsync(own_mean, st);
    }
};
static int pad_input(const void *x, bool bf16, int64_t n, int D, const float *mean, int min_cols,
                     cudaStream_t st, Padded &P) {
    const int es = bf16 ? 2 : 4;
    const int align = 16 / es;
    int ld = (D + align - 1) / align * align;
    if (ld < min_cols) ld = min_cols;
    if (ld == D && ((uintptr_t)x & 15) == 0) {
        P.x = x;
        P.mean = mean;
        P.ldx = D;
        return FA_OK;
    }
    P.st = st;
    FA_TRY(pool_alloc(&P.own_x, (size_t)n * ld * es));
    FA_TRY(pool_alloc((void **)&P.own_mean, (size_t)ld * 4));
    FA_CUDA(cudaMemsetAsync(P.own_x, 0, (size_t)n * ld * es, st));
    FA_CUDA(cudaMemsetAsync(P.own_mean, 0, (size_t)ld * 4, st));
    FA_CUDA(cudaMemcpy2DAsync(P.own_x, (size_t)ld * es, x, (size_t)D * es, (size_t)D * es, n,
                              cudaMemcpyDeviceToDevice, st));
    FA_CUDA(cudaMemcpyAsync(P.own_mean, mean, (size_t)D * 4, cudaMemcpyDeviceToDevice, st));
    P.x = P.own_x;
    P.mean = P.own_mean;
    P.ldx = ld;
    return FA_OK;
}

}  // namespace pg
}  // namespace fa

using namespace fa;
using namespace fa::pg;

extern "C" int fa_pca_cov_dev(const void *x, int x_dtype, int64_t n, int D, const float *mean,
                              double *cov, void *stream) {
    FA_CHECK_ARG(x && mean && cov, "null argument");
    FA_CHECK_ARG(x_dtype == FA_DTYPE_F32 || x_dtype == FA_DTYPE_BF16, "x_dtype must be f32 or bf16");
    FA_CHECK_ARG(n >= 1 && D >= 1, "need n >= 1 and D >= 1");
    FA_CHECK_ARG(n < (1ll << 31) - BK, "n too large");
    cudaStream_t st = as_stream(stream);
    const bool bf = x_dtype == FA_DTYPE_BF16;
    Padded P;
    // the covariance box spans 128 columns: narrower X is padded to 128
    FA_TRY(pad_input(x, bf, n, D, mean, BM, st, P));
    Params p{};
    p.n = n;
    p.D = D;
    p.mean = P.mean;
    p.nb = (D + BM - 1) / BM;
    p.nk = (int)((n + BK - 1) / BK);
    const int64_t ntri = (int64_t)p.nb * (p.nb + 1) / 2;
    // K splits: enough work items for every SM, at least 16 k-blocks each
    int ns = (int)std::max<int64_t>(1, (2 * num_sms() + ntri - 1) / ntri);
    ns = std::min(ns, std::max(1, p.nk / 16));
    // every split must own at least one k-block: an empty split issues no MMA,
    // and its epilogue would drain whatever an earlier kernel left in TMEM
    // into the partial sums (cov_krange gives split sp blocks [sp * per, ...))
    const int per = (p.nk + ns - 1) / ns;
    ns = (p.nk + per - 1) / per;
    p.nsplit = ns;
    p.nwork = ntri * ns;
    float *part = nullptr;
    FA_TRY(pool_alloc((void **)&part, sizeof(float) * (size_t)ns * D * D));
    p.out = part;
    CUtensorMap mx;
    int rc = make_map(&mx, P.x, bf, (uint64_t)P.ldx, (uint64_t)n, (uint64_t)P.ldx * (bf ? 2 : 4),
                      BM, BK, false);
    if (!rc)
        rc = bf ? launch<true, BM, __nv_bfloat16>(mx, mx, mx, p, st)
                : launch<true, BM, float>(mx, mx, mx, p, st);
    if (!rc) {
        cov_reduce_kernel<<<num_sms() * 4, 256, 0, st>>>(part, ns, D, 1.0 / (double)n, cov);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            set_error("cov_reduce_kernel: %s", cudaGetErrorString(e));
            rc = FA_ECUDA;
        }
    }
    // the partials must outlive the kernels: free in stream order
    cudaFreeAsync(part, st);
    return rc;
}

extern "C" int fa_pca_project_dev(const void *x, int x_dtype, int64_t n, int D,
                                  const float *mean, const float *basis, int dfull, int d,
                                  float *out, int64_t ldo, void *stream) {
    FA_CHECK_ARG(x && mean && basis && out, "null argument");
    FA_CHECK_ARG(x_dtype == FA_DTYPE_F32 || x_dtype == FA_DTYPE_BF16, "x_dtype must be f32 or bf16");
    FA_CHECK_ARG(D >= 1 && d >= 1 && d <= dfull && dfull <= D && ldo >= d, "bad sizes");
    FA_CHECK_ARG(n >= 0 && n < (1ll << 31) - BM, "n out of range");
    if (n == 0) return FA_OK;
    cudaStream_t st = as_stream(stream);
    const bool bf = x_dtype == FA_DTYPE_BF16;
    Padded P;
    FA_TRY(pad_input(x, bf, n, D, mean, BK, st, P));
    constexpr int BN = 128;
    const int ldb = (P.ldx + 3) / 4 * 4;
    float *bsplit = nullptr;
    FA_TRY(pool_alloc((void **)&bsplit, sizeof(float) * 2 * (size_t)d * ldb));
    float *bhi = bsplit, *blo = bsplit + (size_t)d * ldb;
    split_basis_kernel<<<num_sms(), 256, 0, st>>>(basis, D, dfull, d, ldb, bhi, blo);
    int rc = FA_OK;
    if (cudaGetLastError() != cudaSuccess) {
        set_error("split_basis_kernel launch failed");
        rc = FA_ECUDA;
    }
    Params p{};
    p.n = n;
    p.D = D;
    p.d = d;
    p.mean = P.mean;
    p.out = out;
    p.ldo = ldo;
    p.nm = (int)((n + BM - 1) / BM);
    p.nn = (d + BN - 1) / BN;
    p.nk = (P.ldx + BK - 1) / BK;
    p.nwork = (int64_t)p.nm * p.nn;
    CUtensorMap mx, mbh, mbl;
    if (!rc)
        rc = make_map(&mx, P.x, bf, (uint64_t)P.ldx, (uint64_t)n, (uint64_t)P.ldx * (bf ? 2 : 4),
                      BK, BM, false);
    if (!rc) rc = make_map(&mbh, bhi, false, (uint64_t)ldb, (uint64_t)d, (uint64_t)ldb * 4, BK, BN, true);
    if (!rc) rc = make_map(&mbl, blo, false, (uint64_t)ldb, (uint64_t)d, (uint64_t)ldb * 4, BK, BN, true);
    if (!rc) {
        rc = bf ? launch<false, BN, __nv_bfloat16>(mx, mbh, mbl, p, st)
                : launch<false, BN, float>(mx, mbh, mbl, p, st);
    }
    cudaFreeAsync(bsplit, st);
    return rc;
}

// pca_project of single vectors in float64 (providers/pca.py:57-65: the
// reference's exact-frame projection of queries and inserted vectors): one
// thread per output element, k ascending.
__global__ void pca_project_f64_kernel(const double *__restrict__ x, int64_t n, int D,
                                       const double *__restrict__ mean,
                                       const double *__restrict__ basis, int dfull, int d,
                                       double *__restrict__ out) {
    const int64_t total = n * d;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / d;
        const int j = (int)(e % d);
        double s = 0.0;
        for (int k = 0; k < D; ++k) s = fma(x[i * D + k] - mean[k], basis[(int64_t)k * dfull + j], s);
        out[e] = s;
    }
}

extern "C" int fa_pca_project_f64_dev(const double *x, int64_t n, int D, const double *mean,
                                      const double *basis, int dfull, int d, double *out,
                                      void *stream) {
    FA_CHECK_ARG(x && mean && basis && out, "null argument");
    FA_CHECK_ARG(n >= 0 && D >= 1 && d >= 1 && d <= dfull, "bad sizes");
    if (n == 0) return FA_OK;
    const int64_t total = n * d;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 4 * num_sms());
    pca_project_f64_kernel<<<grid, 256, 0, as_stream(stream)>>>(x, n, D, mean, basis, dfull, d,
                                                                 out);
    FA_LAUNCH_CHECK();
    return FA_OK;
}
