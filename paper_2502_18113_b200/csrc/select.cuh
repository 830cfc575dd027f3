// K5: warp-cooperative neighbour selection (select_heur, _core.pyx:388-408)
// with Flash symmetric-table distances (sym_one -> fa_sdt_sum_sat,
// _core.pyx:179-191, _simd.h:87-95).
//
// Candidates are scanned in the given order; v is kept iff no already-kept u
// has sdt(u, v) < d_v; the scan stops once `cap` are kept.  The decision for v
// is an OR over the kept set, so evaluating the kept set in parallel (lane t
// takes kept[t], kept[t+32], ...) gives exactly the reference's decisions.
//
// Shared-memory layout: the SDT is stored transposed, sdtT[i][b][a] =
// sdt[i][a][b], where b is the CANDIDATE's code.  All lanes test the same
// candidate, so for subspace i every lane reads inside one 16-byte row
// (4 banks): conflict-free.  Kept codes sit in rows of kstride = mpad + 4 bytes
// (an odd number of words) so lane t's word reads land in distinct banks.
#pragma once

#include "common.cuh"

namespace fa {

__host__ __device__ inline int kept_stride(int mpad) { return mpad + 4; }

// Stage sdt (m x 16 x 16, global) transposed into shared memory.
__device__ __forceinline__ void stage_sdt_T(const uint8_t *__restrict__ sdt, int m, uint8_t *sdtT,
                                            int tid, int nthreads) {
    for (int t = tid; t < m * 256; t += nthreads) {
        int i = t >> 8, a = (t >> 4) & 15, b = t & 15;
        sdtT[(i << 8) + (b << 4) + a] = sdt[t];
    }
}

// The same transposition into a global buffer (m x 256 bytes), one CTA.
__global__ void transpose_sdt_kernel(const uint8_t *__restrict__ sdt, int m,
                                     uint8_t *__restrict__ sdtT);

// min(sum_i sdt[i][cu_i][cv_i], 255) with cu from shared (word-aligned row)
// and cv from global/shared (uniform across the warp).
__device__ __forceinline__ uint32_t sdt_sum_rows(const uint8_t *sdtT, int m, const uint8_t *cu,
                                                 const uint8_t *cv) {
    uint32_t acc = 0;
    int i = 0;
    for (; i + 4 <= m; i += 4) {
        uint32_t wu = *reinterpret_cast<const uint32_t *>(cu + i);
        uint32_t wv = *reinterpret_cast<const uint32_t *>(cv + i);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            uint32_t a_ = (wu >> (8 * b)) & 0xffu, b_ = (wv >> (8 * b)) & 0xffu;
            acc += sdtT[((i + b) << 8) + (b_ << 4) + a_];
        }
    }
    for (; i < m; ++i) acc += sdtT[(i << 8) + (cv[i] << 4) + cu[i]];
    return acc > 255u ? 255u : acc;
}

// Generic warp selection.  get(j, &v, &dv_less) must return the candidate id
// and a functor-like comparison: we pass the candidate distance as a double
// (exact for the reference's integer-valued Flash distances and for arbitrary
// hook inputs).  Candidate code rows are read from `codes` (global, row
// stride cs bytes, 4-byte aligned, zero padded to mpad).  Returns the number
// kept; kept ids in kept_ids[0..nk), their codes in kept_codes rows.
// kept_d (optional): the kept candidates' distances (< 256), as uint8.
template <class Get>
__device__ int warp_select_heur(const uint8_t *sdtT, int m, int mpad,
                                const uint8_t *__restrict__ codes, int cs, int ncand, int cap,
                                Get get, int32_t *kept_ids, uint8_t *kept_codes, int lane,
                                unsigned long long *sym_count, uint8_t *kept_d = nullptr) {
    const int ks = kept_stride(mpad);
    int nk = 0;
    unsigned long long sym = 0;
    for (int j = 0; j < ncand && nk < cap; ++j) {
        int v;
        double dv;
        get(j, v, dv);
        const uint8_t *cv = codes + (size_t)v * cs;
        bool bad = false;
        for (int t = lane; t < nk; t += 32) {
            uint32_t s = sdt_sum_rows(sdtT, m, kept_codes + t * ks, cv);
            bad |= ((double)s < dv);
        }
        sym += nk;
        if (!__any_sync(0xffffffffu, bad)) {
            if (lane == 0) {
                kept_ids[nk] = v;
                if (kept_d) kept_d[nk] = (uint8_t)dv;
            }
            for (int i = lane * 4; i < mpad; i += 128)
                *reinterpret_cast<uint32_t *>(kept_codes + nk * ks + i) =
                    *reinterpret_cast<const uint32_t *>(cv + i);
            ++nk;
            __syncwarp();
        }
    }
    if (sym_count && lane == 0) *sym_count += sym;
    return nk;
}

// ---- forward selection of the build (K5, per-candidate table variant) ------
// The same decisions as warp_select_heur for integer candidate distances.
// For candidate v, sdt(u, v) = sum_i sdt[i][u_i][v_i] = sum_i Tv[i][u_i] with
// Tv[i][*] = sdtT row (i, v_i): the warp copies v's m table rows (16 B each,
// one 16-byte load per row) into shared memory, then lane t sums kept[t]'s
// lookups.  Kept code rows are stored pre-offset: byte i holds
// (i % 16) * 16 + u_i, so within a 16-subspace chunk (256 table bytes) one PRMT
// merges the chunk base (256-aligned) with the byte into the lookup address.
__host__ __device__ inline int kept_enc_stride(int mpad) { return mpad + 16; }
__host__ __device__ inline int select_tv_bytes(int m, int mpad, int cap) {
    return round_up(cap * 4, 256) + round_up(cap * kept_enc_stride(mpad), 256) +
           round_up(mpad * 16, 256);
}
// ws bytes of warp_select_tv when Tv lives elsewhere (kept ids + codes)
__host__ __device__ inline int select_tv_ws_bytes(int mpad, int cap) {
    return round_up(cap * 4, 256) + round_up(cap * kept_enc_stride(mpad), 256);
}

// chunk-local row offsets (i % 16) * 16 of the four bytes of code word q
__device__ __forceinline__ uint32_t kept_enc_add(int q) {
    return 0x30201000u + 0x40404040u * (uint32_t)(q & 3);
}

// Copy the 16-byte rows tab[i][x_i] (i < m; zero rows up to mpad) of a
// global m x 16 x 16 table into T (shared, 256-aligned): T[i][c] = tab[i][x_i][c].
__device__ __forceinline__ void build_row_table(const uint8_t *__restrict__ tab, int m, int mpad,
                                                const uint8_t *__restrict__ cx, uint8_t *T,
                                                int lane) {
    for (int i = lane; i < mpad; i += 32) {
        uint4 row = make_uint4(0, 0, 0, 0);
        if (i < m)
            row = __ldg(reinterpret_cast<const uint4 *>(tab + (i << 8) +
                                                         ((uint32_t)__ldg(cx + i) << 4)));
        *reinterpret_cast<uint4 *>(T + i * 16) = row;
    }
}

// sum_i T[i][u_i], saturated, for a raw code row u (global, 16-byte aligned,
// zero padded to mpad); T at shared address tbase (256-aligned).
__device__ __forceinline__ uint32_t row_table_sum(uint32_t tbase, const uint8_t *__restrict__ cu,
                                                  int mpad) {
    uint32_t acc = 0;
    for (int c = 0; c < mpad; c += 16) {
        const uint4 w = __ldg(reinterpret_cast<const uint4 *>(cu + c));
        const uint32_t base = tbase + (uint32_t)c * 16u;
        const uint32_t W[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t e = W[q] + kept_enc_add(q);
            uint32_t b[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t a = prmt(e, base, 0x7650u + (uint32_t)k);
                asm volatile("ld.shared.u8 %0, [%1];" : "=r"(b[k]) : "r"(a));
            }
            acc += b[0] + b[1] + b[2] + b[3];
        }
    }
    return acc > 255u ? 255u : acc;
}

// ws: kept ids then the kept rows' pre-offset codes (any memory: shared in
// the build, per-warp global scratch in the reverse kernel's rare full
// prune); Tv: the candidate's table, shared memory (256-aligned, mpad x 16),
// null = right after the kept codes in ws (ws then must be shared).
template <class Get>
__device__ int warp_select_tv(const uint8_t *__restrict__ sdtT, int m, int mpad,
                              const uint8_t *__restrict__ codes, int cs, int ncand, int cap,
                              Get get, uint8_t *ws, int lane, unsigned long long *sym_count,
                              int32_t *&kept_out, uint8_t *kept_d = nullptr,
                              uint8_t *Tv_shared = nullptr) {
    const int ks = kept_enc_stride(mpad);
    int32_t *kept_ids = reinterpret_cast<int32_t *>(ws);
    uint8_t *kenc = ws + round_up(cap * 4, 256);
    uint8_t *Tv = Tv_shared ? Tv_shared : kenc + round_up(cap * ks, 256);
    kept_out = kept_ids;
    int nk = 0;
    unsigned long long sym = 0;
    for (int j = 0; j < ncand && nk < cap; ++j) {
        int v;
        uint32_t dv;
        get(j, v, dv);
        const uint8_t *cv = codes + (size_t)v * cs;
        bool bad = false;
        if (nk > 0) {
            for (int i = lane; i < mpad; i += 32) {
                uint4 row = make_uint4(0, 0, 0, 0);
                if (i < m)
                    row = __ldg(reinterpret_cast<const uint4 *>(sdtT + (i << 8) +
                                                                 ((uint32_t)__ldg(cv + i) << 4)));
                *reinterpret_cast<uint4 *>(Tv + i * 16) = row;
            }
            __syncwarp();
            const uint32_t tv = (uint32_t)__cvta_generic_to_shared(Tv);
            for (int t = lane; t < nk; t += 32) {
                const uint8_t *ku = kenc + t * ks;
                uint32_t acc = 0;
                for (int c = 0; c < mpad; c += 16) {
                    const uint4 w = *reinterpret_cast<const uint4 *>(ku + c);
                    const uint32_t base = tv + (uint32_t)c * 16u;  // 256-aligned
                    const uint32_t W[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t b[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            uint32_t a = prmt(W[q], base, 0x7650u + (uint32_t)k);
                            uint32_t x;
                            asm volatile("ld.shared.u8 %0, [%1];" : "=r"(x) : "r"(a));
                            b[k] = x;
                        }
                        acc += b[0] + b[1] + b[2] + b[3];
                    }
                }
                bad |= (acc > 255u ? 255u : acc) < dv;
            }
            sym += nk;
        }
        if (!__any_sync(0xffffffffu, bad)) {
            if (lane == 0) {
                kept_ids[nk] = v;
                if (kept_d) kept_d[nk] = (uint8_t)dv;
            }
            for (int q = lane; q < mpad / 4; q += 32)
                *reinterpret_cast<uint32_t *>(kenc + nk * ks + 4 * q) =
                    __ldg(reinterpret_cast<const uint32_t *>(cv) + q) + kept_enc_add(q);
            ++nk;
        }
        __syncwarp();
    }
    if (sym_count && lane == 0) *sym_count += sym;
    return nk;
}

}  // namespace fa
