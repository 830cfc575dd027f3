// K1: saturating uint8 ADT scan over 16-slot subspace-major code batches.
//
// Semantics (reference _simd.h:111-121 fa_batch_scalar, the definition every
// SIMD width must reproduce): out[lane] = min(sum_i adt[i][code[i][lane]], 255).
// All addends are >= 0, so per-step saturation equals one clamp of the exact
// integer sum: lanes accumulate exact 16-bit sums (m <= 256
// keeps them < 65536) and clamp once.
//
// Warp mapping (B200): lane t owns subspace rows r = t, t+32, ... of a batch.
// It keeps its query-table rows in registers (4 x u32 each) and reads the 16
// codes of row r with ONE coalesced 16-byte load (a warp reads 512 contiguous
// bytes per instruction).  Four lookups are done per PRMT pair (lut16x4), the
// bytes are widened into 16-bit pair accumulators, and a 9-shuffle
// reduce-scatter leaves each batch slot's total in one lane.
#pragma once

#include "common.cuh"

namespace fa {

// Table rows of one query: lane t holds rows t + 32*k (k < NR), zero beyond m.
template <int NR>
struct WarpTable {
    uint32_t t[NR][4];
    __device__ __forceinline__ void load(const uint8_t *adt, int m, int lane) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            int r = lane + 32 * k;
            if (r < m) {
                uint4 v = *reinterpret_cast<const uint4 *>(adt + (size_t)r * 16);
                t[k][0] = v.x; t[k][1] = v.y; t[k][2] = v.z; t[k][3] = v.w;
            } else {
                t[k][0] = t[k][1] = t[k][2] = t[k][3] = 0u;
            }
        }
    }
};

// Accumulate one row's 16 codes (as a uint4) into 8 pair accumulators:
// acc[2g] = slots (4g, 4g+2), acc[2g+1] = slots (4g+1, 4g+3) as 16-bit halves.
__device__ __forceinline__ void acc_row(const uint32_t (&t)[4], uint4 c, uint32_t (&acc)[8]) {
    uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        uint32_t r = lut16x4(t[0], t[1], t[2], t[3], w[g]);
        acc[2 * g] += prmt(r, 0u, 0x4240u);     // bytes 0,2 -> 16-bit halves
        acc[2 * g + 1] += prmt(r, 0u, 0x4341u); // bytes 1,3
    }
}

// Reduce-scatter the 8 per-lane accumulators over the warp.  Returns the
// clamped distance of slot `slot_of_lane()` (valid in lanes with (lane&2)==0).
__device__ __forceinline__ uint32_t reduce_batch(uint32_t (&acc)[8], int lane) {
    uint32_t r4[4];
    const bool b4 = lane & 16;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t send = b4 ? acc[k] : acc[k + 4];
        uint32_t keep = b4 ? acc[k + 4] : acc[k];
        r4[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    uint32_t r2[2];
    const bool b3 = lane & 8;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        uint32_t send = b3 ? r4[k] : r4[k + 2];
        uint32_t keep = b3 ? r4[k + 2] : r4[k];
        r2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    const bool b2 = lane & 4;
    uint32_t send = b2 ? r2[0] : r2[1];
    uint32_t keep = b2 ? r2[1] : r2[0];
    uint32_t r = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    r += __shfl_xor_sync(0xffffffffu, r, 2);
    uint32_t v = (lane & 1) ? (r >> 16) : (r & 0xffffu);
    return v > 255u ? 255u : v;
}

// Batch slot owned by `lane` after reduce_batch (lanes with (lane & 2) == 0).
__device__ __forceinline__ int slot_of_lane(int lane) {
    int j = lane >> 2;  // accumulator index
    int g = j >> 1, odd = j & 1;
    return 4 * g + odd + 2 * (lane & 1);
}

// One 16-slot batch (m x 16 bytes at `codes`, 16-byte aligned).
template <int NR>
__device__ __forceinline__ uint32_t scan_batch(const WarpTable<NR> &tab, const uint8_t *codes,
                                               int m, int lane) {
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        int r = lane + 32 * k;
        if (r < m) {
            uint4 c = __ldg(reinterpret_cast<const uint4 *>(codes + (size_t)r * 16));
            acc_row(tab.t[k], c, acc);
        }
    }
    return reduce_batch(acc, lane);
}

}  // namespace fa
