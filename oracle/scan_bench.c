/*
 * scan_bench.c — CPU baseline harness for the block scan.
 *
 * TEST/BASELINE INFRASTRUCTURE ONLY.  Compiled by `make -C oracle ref` against
 * the reference's own kernel header (flashann/_kernels/_simd.h, included from
 * /root/reference at build time, never copied) with the reference's flags, so
 * the timed inner loop is the reference's fa_batch_lanes at its widest ISA.
 * Same block array and query tables as the GPU scan (the padded device layout:
 * int32 count | pad | int32 ids[cap] | codes nb x m x 16 at codes_off).
 */
#include <omp.h>
#include <stdint.h>

#include "_simd.h"

int scan_bench_widest_kernel(void) {
    return FA_HAVE_V512 ? 3 : (FA_HAVE_V256 ? 2 : (FA_HAVE_V128 ? 1 : 0));
}

/* out[q] = min over live slots of (d << 32 | id); returns lanes evaluated. */
int64_t scan_bench(const uint8_t *adt, int nq, const uint8_t *blocks, int64_t stride,
                   int64_t codes_off, int cap, int m, const int32_t *sel, int nsel,
                   uint64_t *out, int threads, int kernel) {
    const int nb = (cap + 15) >> 4;
    int64_t lanes = 0;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 4) reduction(+ : lanes)
    for (int q = 0; q < nq; ++q) {
        uint8_t buf[16 * 16];
        uint64_t best = ~0ull;
        const uint8_t *tab = adt + (size_t)q * m * 16;
        for (int s = 0; s < nsel; ++s) {
            const uint8_t *b = blocks + (int64_t)sel[(size_t)q * nsel + s] * stride;
            int cnt = *(const int32_t *)b;
            if (cnt > cap) cnt = cap;
            const int32_t *ids = (const int32_t *)(b + 16);
            fa_batch_lanes(tab, b + codes_off, m, nb, kernel, buf);
            lanes += nb * 16;
            for (int j = 0; j < cnt; ++j) {
                if (ids[j] < 0) continue;
                uint64_t k = ((uint64_t)buf[j] << 32) | (uint32_t)ids[j];
                if (k < best) best = k;
            }
        }
        out[q] = best;
    }
    return lanes;
}
