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

// Eight lookups of one 16-entry byte table: the 4-bit codes in the bytes of
// w0 and w1 (each byte < 16).  r0 / r1 hold the table bytes of w0 / w1 with
// the bytes of each pair swapped: (T[c1], T[c0], T[c3], T[c2]).
// The scan is bound by the integer ALU pipe (PRMT / LOP3 / SHF), so the
// nibble packing runs on the FMA pipe instead: w * 0x1001 = w + (w << 12)
// puts c1 | c0 << 4 in byte 1 and c3 | c2 << 4 in byte 3 (the fields do not
// overlap, so the add carries nothing), one PRMT gathers both words'
// selector bytes, one LOP3 clears their bit 3 (PRMT's sign-replicate flag;
// PRMT reads only the low 16 bits of its selector), and the second word's
// selector comes down with a multiply-high.  The table halves are merged by a
// PRMT too: its selector nibble i is i + 4 x (bit 3 of code i), i.e. the bit-3
// nibbles of the gathered selectors shifted down by one plus 0x3210 (one
// LOP3 and one multiply-high with addend per word pair).  5.5 ALU-pipe
// instructions per four lookups instead of 8, and acc_word widens with one
// more (was two).
__device__ __forceinline__ void lut16x8(const uint32_t (&t)[4], uint32_t w0, uint32_t w1,
                                        uint32_t &r0, uint32_t &r1) {
    const uint32_t y0 = w0 * 0x1001u, y1 = w1 * 0x1001u;
    const uint32_t sr = prmt(y0, y1, 0x7531u);
    const uint32_t s0 = sr & 0x77777777u;
    const uint32_t s1 = __umulhi(s0, 0x10000u);  // s0 >> 16
    const uint32_t b0 = __umulhi(sr & 0x88888888u, 0x80000000u) + 0x32103210u;
    const uint32_t b1 = __umulhi(b0, 0x10000u);
    const uint32_t lo0 = prmt(t[0], t[1], s0), hi0 = prmt(t[2], t[3], s0);
    const uint32_t lo1 = prmt(t[0], t[1], s1), hi1 = prmt(t[2], t[3], s1);
    r0 = prmt(lo0, hi0, b0);
    r1 = prmt(lo1, hi1, b1);
}

// Add the four table bytes r = (x0, x1, x2, x3) of one code word (swapped
// pairs: x1, x3 = slots 4g, 4g+2; x0, x2 = slots 4g+1, 4g+3) to the word's
// accumulator pair: ae += x0 | x2 << 16 (one LOP3), ao += r >> 8 = x1 +
// (x2 << 8) + (x3 << 16) (a multiply-high with addend, FMA pipe).  ao
// carries 256 x the x2 sums until finish_acc() takes them out again, once
// per batch: exact 32-bit integer arithmetic (a lane adds at most 5 rows of
// bytes per batch, so no field reaches 2^32).
__device__ __forceinline__ void acc_word(uint32_t r, uint32_t &ao, uint32_t &ae) {
    ae += r & 0x00ff00ffu;
    ao += __umulhi(r, 1u << 24);
}

// Accumulate one row's 16 codes (as a uint4) into 8 pair accumulators:
// after finish_acc(), acc[2g] = slots (4g, 4g+2), acc[2g+1] = slots (4g+1,
// 4g+3) as 16-bit halves.
__device__ __forceinline__ void acc_row(const uint32_t (&t)[4], uint4 c, uint32_t (&acc)[8]) {
    uint32_t r[4];
    lut16x8(t, c.x, c.y, r[0], r[1]);
    lut16x8(t, c.z, c.w, r[2], r[3]);
#pragma unroll
    for (int g = 0; g < 4; ++g) acc_word(r[g], acc[2 * g], acc[2 * g + 1]);
}

// acc[2g] -= 256 x (the high half of acc[2g+1]): see acc_word.
__device__ __forceinline__ void finish_acc(uint32_t (&acc)[8]) {
#pragma unroll
    for (int g = 0; g < 4; ++g) acc[2 * g] -= __umulhi(acc[2 * g + 1], 1u << 16) << 8;
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
    finish_acc(acc);
    return reduce_batch(acc, lane);
}

}  // namespace fa
