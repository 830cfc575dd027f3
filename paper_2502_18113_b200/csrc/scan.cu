// K1 entry points: parity hooks (flash_batch_distance_many / _blocks) and the
// standalone HBM-bound block scan.
#include "scan.cuh"

namespace fa {

// One warp per case: the case's own table + one 16-slot batch.
template <int NR>
__global__ void __launch_bounds__(256) scan_cases_kernel(const uint8_t *__restrict__ adts,
                                                         const uint8_t *__restrict__ codes, int m,
                                                         int64_t ncases, uint8_t *__restrict__ out) {
    const int lane = lane_id();
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t c = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); c < ncases;
         c += warps) {
        WarpTable<NR> tab;
        tab.load(adts + c * m * 16, m, lane);
        uint32_t v = scan_batch<NR>(tab, codes + c * m * 16, m, lane);
        if ((lane & 2) == 0) out[c * 16 + slot_of_lane(lane)] = (uint8_t)v;
    }
}

// One warp per batch of a block.
template <int NR>
__global__ void scan_blocks_kernel(const uint8_t *__restrict__ adt, const uint8_t *__restrict__ codes,
                                   int m, int nb, uint8_t *__restrict__ out) {
    const int lane = lane_id();
    const int b = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (b >= nb) return;
    WarpTable<NR> tab;
    tab.load(adt, m, lane);
    uint32_t v = scan_batch<NR>(tab, codes + (size_t)b * m * 16, m, lane);
    if ((lane & 2) == 0) out[b * 16 + slot_of_lane(lane)] = (uint8_t)v;
}

// Standalone scan: warp per (query, slice of its block list).  Each block is
// [int32 count | pad | int32 ids[cap] | codes nb x m x 16] in the padded
// device layout.  out[q] = min over live slots of (d << 32 | id); several
// warps of one query combine with atomicMin.
template <int NR>
__global__ void __launch_bounds__(256) scan_select_kernel(
    const uint8_t *__restrict__ adt, int nq, const uint8_t *__restrict__ blocks,
    int64_t block_stride, int64_t codes_off, int cap, int m, const int32_t *__restrict__ sel,
    int nsel, int slices, unsigned long long *__restrict__ out) {
    const int lane = lane_id();
    const int gw = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int q = gw / slices;
    const int slice = gw % slices;
    if (q >= nq) return;
    WarpTable<NR> tab;
    tab.load(adt + (size_t)q * m * 16, m, lane);
    const int nb = (cap + 15) >> 4;
    const int per = (nsel + slices - 1) / slices;
    const int lo = slice * per;
    const int hi = min(nsel, lo + per);
    unsigned long long best = ~0ull;
    const int32_t *qsel = sel + (size_t)q * nsel;
    for (int s = lo; s < hi; ++s) {
        const uint8_t *blk = blocks + (int64_t)__ldg(qsel + s) * block_stride;
        int cnt = __ldg(reinterpret_cast<const int32_t *>(blk));
        cnt = min(cnt, cap);
        const int32_t *ids = reinterpret_cast<const int32_t *>(blk + 16);
        const uint8_t *cod = blk + codes_off;
        for (int b = 0; b < nb; ++b) {
            uint32_t v = scan_batch<NR>(tab, cod + (size_t)b * m * 16, m, lane);
            int slot = b * 16 + slot_of_lane(lane);
            if ((lane & 2) == 0 && slot < cnt) {
                int id = __ldg(ids + slot);
                if (id >= 0) {
                    unsigned long long key = ((unsigned long long)v << 32) | (uint32_t)id;
                    best = key < best ? key : best;
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other < best ? other : best;
    }
    if (lane == 0 && best != ~0ull) atomicMin(out + q, best);
}

// ---- TMA-staged block scan -------------------------------------------------
// Each block is one contiguous region, so a 1-D bulk copy (cp.async.bulk,
// SASS UBLKCP) moves it into a per-warp ring of shared-memory stages; an
// mbarrier per stage carries the transaction count.  Lane 0 keeps kStages
// blocks in flight while the warp scans the oldest one from shared memory
// (lane t reads row t of a batch: 16 contiguous bytes, conflict-free).
constexpr int kScanStages = 2;
constexpr int kScanWarps = 8;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// NR full table rows per lane (rows lane + 32 k); HALF: the m - 32 NR = 16
// remaining rows are split in halves, lane t taking 8 slots (half t & 1) of
// row 32 NR + t / 2 — no lane idles at m = 48, 80, 112.
template <int NR, bool HALF>
__global__ void __launch_bounds__(kScanWarps * 32) scan_select_tma_kernel(
    const uint8_t *__restrict__ adt, int nq, const uint8_t *__restrict__ blocks,
    int64_t block_stride, int64_t codes_off, uint32_t copy_bytes, uint32_t stage_bytes, int cap,
    int m, const int32_t *__restrict__ sel, int nsel, int slices, int stages,
    unsigned long long *__restrict__ out) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = lane_id();
    const int wid = threadIdx.x >> 5;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem) + wid * kScanStages;
    uint8_t *ring = smem + 128 + (size_t)wid * stages * stage_bytes;
    if (lane == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(bars + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int gw = blockIdx.x * kScanWarps + wid;
    const int q = gw / slices;
    const int slice = gw % slices;
    if (q >= nq) return;
    WarpTable<NR> tab;
    tab.load(adt + (size_t)q * m * 16, m, lane);
    const int hrow = 32 * NR + (lane >> 1);
    uint32_t th[4] = {0, 0, 0, 0};
    if (HALF) {
        const uint4 v = *reinterpret_cast<const uint4 *>(adt + (size_t)q * m * 16 + hrow * 16);
        th[0] = v.x; th[1] = v.y; th[2] = v.z; th[3] = v.w;
    }
    const bool hodd = lane & 1;
    const int nb = (cap + 15) >> 4;
    const int per = (nsel + slices - 1) / slices;
    const int lo = slice * per;
    const int hi = min(nsel, lo + per);
    const int nblk = max(0, hi - lo);
    const int32_t *qsel = sel + (size_t)q * nsel + lo;
    if (lane == 0)
        for (int s = 0; s < stages && s < nblk; ++s) {
            mbar_expect_tx(bars + s, copy_bytes);
            bulk_g2s(ring + (size_t)s * stage_bytes, blocks + (int64_t)__ldg(qsel + s) * block_stride,
                     copy_bytes, bars + s);
        }
    unsigned long long best = ~0ull;
    for (int i = 0; i < nblk; ++i) {
        const int st = stages == 1 ? 0 : i & 1;
        mbar_wait(bars + st, (uint32_t)((stages == 1 ? i : i >> 1) & 1));
        const uint8_t *blk = ring + (size_t)st * stage_bytes;
        const int cnt = min(*reinterpret_cast<const int32_t *>(blk), cap);
        const int32_t *ids = reinterpret_cast<const int32_t *>(blk + 16);
        const uint8_t *cod = blk + codes_off;
        for (int b = 0; b < nb; ++b) {
            uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                const int r = lane + 32 * k;
                if (HALF || r < m)
                    acc_row(tab.t[k], *reinterpret_cast<const uint4 *>(cod + (size_t)b * m * 16 + r * 16),
                            acc);
            }
            if (HALF) {
                const uint2 c = *reinterpret_cast<const uint2 *>(cod + (size_t)b * m * 16 + hrow * 16 +
                                                                 (hodd ? 8 : 0));
                uint32_t r0, r1;
                lut16x8(th, c.x, c.y, r0, r1);
                if (hodd) {
                    acc_word(r0, acc[4], acc[5]);
                    acc_word(r1, acc[6], acc[7]);
                } else {
                    acc_word(r0, acc[0], acc[1]);
                    acc_word(r1, acc[2], acc[3]);
                }
            }
            finish_acc(acc);
            const uint32_t v = reduce_batch(acc, lane);
            const int slot = b * 16 + slot_of_lane(lane);
            if ((lane & 2) == 0 && slot < cnt) {
                const int id = ids[slot];
                if (id >= 0) {
                    const unsigned long long key = ((unsigned long long)v << 32) | (uint32_t)id;
                    best = key < best ? key : best;
                }
            }
        }
        __syncwarp();
        if (lane == 0 && i + stages < nblk) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bars + st, copy_bytes);
            bulk_g2s(ring + (size_t)st * stage_bytes,
                     blocks + (int64_t)__ldg(qsel + i + stages) * block_stride, copy_bytes,
                     bars + st);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other < best ? other : best;
    }
    if (lane == 0 && best != ~0ull) atomicMin(out + q, best);
}

}  // namespace fa

using namespace fa;

extern "C" int fa_scan_select_tma_dev(const uint8_t *adt, int nq, const uint8_t *blocks,
                                      int64_t nblocks, int64_t block_stride, int64_t codes_off,
                                      int cap, int m, const int32_t *sel, int nsel,
                                      uint64_t *out_u64, void *stream) {
    FA_CHECK_ARG(m >= 1 && m <= 128, "m=%d outside [1,128]", m);
    FA_CHECK_ARG(codes_off % 16 == 0 && block_stride % 16 == 0, "block layout must be 16B aligned");
    FA_CHECK_ARG(nq >= 0 && nsel >= 0 && nblocks >= 0, "negative sizes");
    if (nq == 0) return FA_OK;
    cudaStream_t st = as_stream(stream);
    unsigned long long *out = reinterpret_cast<unsigned long long *>(out_u64);
    FA_CUDA(cudaMemsetAsync(out, 0xff, sizeof(unsigned long long) * nq, st));
    const int nb = (cap + 15) / 16;
    const uint32_t copy_bytes = (uint32_t)round_up64(codes_off + (int64_t)nb * m * 16, 16);
    FA_CHECK_ARG(copy_bytes <= (uint32_t)block_stride, "block stride smaller than its contents");
    const uint32_t stage_bytes = (uint32_t)round_up64(copy_bytes, 128);
    // two stages per warp while two CTAs still fit an SM, else one (large
    // blocks: more warps beat deeper rings)
    const int stages = 2 * ((size_t)kScanWarps * 2 * stage_bytes + 1024) * 2 <= 227 * 1024 ? 2 : 1;
    const size_t smem = 128 + (size_t)kScanWarps * stages * stage_bytes;
    FA_CHECK_ARG(smem <= 227 * 1024, "block too large for the staged scan");
    int slices = 1;
    while ((int64_t)nq * slices < 148 * 96 && slices * 16 <= nsel) slices *= 2;
    const int64_t warps = (int64_t)nq * slices;
    const int grid = (int)((warps + kScanWarps - 1) / kScanWarps);
#define FA_TMA_LAUNCH(NR_, HALF_)                                                           \
    do {                                                                                    \
        FA_CUDA(cudaFuncSetAttribute(scan_select_tma_kernel<NR_, HALF_>,                    \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        scan_select_tma_kernel<NR_, HALF_><<<grid, kScanWarps * 32, smem, st>>>(            \
            adt, nq, blocks, block_stride, codes_off, copy_bytes, stage_bytes, cap, m, sel,  \
            nsel, slices, stages, out);                                                     \
    } while (0)
    if (m == 48) FA_TMA_LAUNCH(1, true);
    else if (m == 80) FA_TMA_LAUNCH(2, true);
    else if (m == 112) FA_TMA_LAUNCH(3, true);
    else if (m <= 32) FA_TMA_LAUNCH(1, false);
    else if (m <= 64) FA_TMA_LAUNCH(2, false);
    else if (m <= 96) FA_TMA_LAUNCH(3, false);
    else FA_TMA_LAUNCH(4, false);
#undef FA_TMA_LAUNCH
    FA_LAUNCH_CHECK();
    return FA_OK;
}

extern "C" int fa_scan_cases_dev(const uint8_t *adts, const uint8_t *codes, int m, int64_t ncases,
                                 uint8_t *out, void *stream) {
    FA_CHECK_ARG(m >= 1 && m <= 128, "m=%d outside [1,128]", m);
    FA_CHECK_ARG(ncases >= 0, "ncases < 0");
    if (ncases == 0) return FA_OK;
    cudaStream_t st = as_stream(stream);
    int64_t blocks = (ncases + 7) / 8;
    int grid = (int)(blocks < 148 * 64 ? blocks : 148 * 64);
    if (m <= 32) scan_cases_kernel<1><<<grid, 256, 0, st>>>(adts, codes, m, ncases, out);
    else if (m <= 64) scan_cases_kernel<2><<<grid, 256, 0, st>>>(adts, codes, m, ncases, out);
    else if (m <= 96) scan_cases_kernel<3><<<grid, 256, 0, st>>>(adts, codes, m, ncases, out);
    else scan_cases_kernel<4><<<grid, 256, 0, st>>>(adts, codes, m, ncases, out);
    FA_LAUNCH_CHECK();
    return FA_OK;
}

extern "C" int fa_scan_blocks_dev(const uint8_t *adt, const uint8_t *codes, int m, int nb,
                                  uint8_t *out, void *stream) {
    FA_CHECK_ARG(m >= 1 && m <= 128, "m=%d outside [1,128]", m);
    FA_CHECK_ARG(nb >= 0, "nb < 0");
    if (nb == 0) return FA_OK;
    cudaStream_t st = as_stream(stream);
    int grid = (nb + 3) / 4;
    if (m <= 32) scan_blocks_kernel<1><<<grid, 128, 0, st>>>(adt, codes, m, nb, out);
    else if (m <= 64) scan_blocks_kernel<2><<<grid, 128, 0, st>>>(adt, codes, m, nb, out);
    else if (m <= 96) scan_blocks_kernel<3><<<grid, 128, 0, st>>>(adt, codes, m, nb, out);
    else scan_blocks_kernel<4><<<grid, 128, 0, st>>>(adt, codes, m, nb, out);
    FA_LAUNCH_CHECK();
    return FA_OK;
}

extern "C" int fa_scan_select_dev(const uint8_t *adt, int nq, const uint8_t *blocks,
                                  int64_t nblocks, int64_t block_stride, int64_t codes_off, int cap,
                                  int m, const int32_t *sel, int nsel, uint64_t *out_u64,
                                  void *stream) {
    FA_CHECK_ARG(m >= 1 && m <= 128, "m=%d outside [1,128]", m);
    FA_CHECK_ARG(codes_off % 16 == 0 && block_stride % 16 == 0, "block layout must be 16B aligned");
    FA_CHECK_ARG(nq >= 0 && nsel >= 0 && nblocks >= 0, "negative sizes");
    if (nq == 0) return FA_OK;
    cudaStream_t st = as_stream(stream);
    unsigned long long *out = reinterpret_cast<unsigned long long *>(out_u64);
    FA_CUDA(cudaMemsetAsync(out, 0xff, sizeof(unsigned long long) * nq, st));
    // enough warps to keep >= 32 KB of block bytes in flight per SM
    int slices = 1;
    while ((int64_t)nq * slices < 148 * 48 && slices * 8 <= nsel) slices *= 2;
    int64_t warps = (int64_t)nq * slices;
    int grid = (int)((warps + 7) / 8);
    if (m <= 32)
        scan_select_kernel<1><<<grid, 256, 0, st>>>(adt, nq, blocks, block_stride, codes_off, cap,
                                                    m, sel, nsel, slices, out);
    else if (m <= 64)
        scan_select_kernel<2><<<grid, 256, 0, st>>>(adt, nq, blocks, block_stride, codes_off, cap,
                                                    m, sel, nsel, slices, out);
    else if (m <= 96)
        scan_select_kernel<3><<<grid, 256, 0, st>>>(adt, nq, blocks, block_stride, codes_off, cap,
                                                    m, sel, nsel, slices, out);
    else
        scan_select_kernel<4><<<grid, 256, 0, st>>>(adt, nq, blocks, block_stride, codes_off, cap,
                                                    m, sel, nsel, slices, out);
    FA_LAUNCH_CHECK();
    return FA_OK;
}
