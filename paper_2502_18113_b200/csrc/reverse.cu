// K6: grouped reverse-edge insertion (reverse_add, _core.pyx:441-477).
//
// The batch's forward selections emit requests (row(y, layer) << 32 | x);
// after a radix sort each row's incoming x arrive ascending, which is the
// order the sequential reference applies them in.  One warp owns a row and
// replays the reference's per-edge rule exactly:
//   count < cap : append x (write_code_slot + id, count+1)
//   count == cap: d(y,u) = sdt-sum for all cap+1 candidates, sort by (d, id)
//                 (fa_sort_pairs), select_heur(cap), rewrite the row.
// Fast path: a row whose content is exactly the previous prune's output (kept
// order = ascending (d, id), pairwise non-dominated) stays kept except for
// candidates x itself dominates, so the prune of L + {x} needs only the
// sums against x — decision-identical to the full scan.
#include "kernels.cuh"

namespace fa {

// u uniform across the warp: sdtN[i][cu][cv] rows are 16 contiguous bytes.
__device__ __forceinline__ uint32_t sdt_sum_u_uniform(const uint8_t *sdtN, int m, const uint8_t *cu,
                                                      const uint8_t *cv) {
    uint32_t acc = 0;
    int i = 0;
    for (; i + 4 <= m; i += 4) {
        uint32_t wu = *reinterpret_cast<const uint32_t *>(cu + i);
        uint32_t wv = *reinterpret_cast<const uint32_t *>(cv + i);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            uint32_t a_ = (wu >> (8 * b)) & 0xffu, b_ = (wv >> (8 * b)) & 0xffu;
            acc += sdtN[((i + b) << 8) + (a_ << 4) + b_];
        }
    }
    for (; i < m; ++i) acc += sdtN[(i << 8) + (cu[i] << 4) + cv[i]];
    return acc > 255u ? 255u : acc;
}

// Bitonic sort of np (power of two <= 128) keys in shared memory, ascending.
__device__ __forceinline__ void warp_bitonic_smem(unsigned long long *a, int np, int lane) {
    for (int k = 2; k <= np; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < np; i += 32) {
                int l = i ^ j;
                if (l > i) {
                    unsigned long long x = a[i], y = a[l];
                    bool up = (i & k) == 0;
                    if ((x > y) == up) {
                        a[i] = y;
                        a[l] = x;
                    }
                }
            }
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(kReverseWarps * 32) reverse_kernel(
    Graph g, const uint8_t *__restrict__ sdt, const unsigned long long *__restrict__ keys,
    int64_t N, const int32_t *__restrict__ upper_owner, ReverseLayout L,
    unsigned long long *__restrict__ ctr) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int tb = round_up(g.m * 256, 128);
    uint8_t *sdtN = smem;
    uint8_t *sdtT = smem + tb;
    for (int t = threadIdx.x; t < g.m * 256; t += blockDim.x) sdtN[t] = sdt[t];
    stage_sdt_T(sdt, g.m, sdtT, threadIdx.x, blockDim.x);
    __syncthreads();
    const int lane = lane_id();
    const int wid = threadIdx.x >> 5;
    uint8_t *base = smem + 2 * tb + wid * L.total;
    int32_t *row_s = reinterpret_cast<int32_t *>(base + L.row);
    unsigned long long *cand = reinterpret_cast<unsigned long long *>(base + L.cand);
    int32_t *kept = reinterpret_cast<int32_t *>(base + L.kept);
    uint8_t *kcodes = base + L.kcodes;
    const int64_t chunk = (int64_t)blockIdx.x * kReverseWarps + wid;
    const int64_t i = chunk * 32 + lane;
    unsigned long long key = i < N ? keys[i] : KEY_MAX;
    unsigned long long prev = (i > 0 && i < N) ? keys[i - 1] : KEY_MAX;
    bool head = key != KEY_MAX && (i == 0 || (prev >> 32) != (key >> 32));
    unsigned heads = __ballot_sync(0xffffffffu, head);
    unsigned long long n_prune = 0, n_app = 0, n_sym = 0;
    while (heads) {
        const int64_t h = chunk * 32 + __ffs(heads) - 1;
        heads &= heads - 1;
        const unsigned long long hk = keys[h];
        const int64_t rowg = (int64_t)(hk >> 32);
        int64_t e = -1;
        for (int64_t b = h + 1;; b += 32) {
            int64_t j = b + lane;
            bool same = j < N && (keys[j] >> 32) == (hk >> 32);
            unsigned nb = __ballot_sync(0xffffffffu, !same);
            if (nb) {
                e = b + __ffs(nb) - 1;
                break;
            }
        }
        const bool l0 = rowg < g.n;
        const int y = l0 ? (int)rowg : upper_owner[rowg - g.n];
        const int cap = l0 ? g.cap0 : g.capU;
        int32_t *ids = l0 ? g.adj0 + rowg * g.cap0p : g.adjU + (rowg - g.n) * g.capUp;
        int32_t *cntp = l0 ? g.cnt0 + rowg : g.cntU + (rowg - g.n);
        uint8_t *consp = l0 ? g.cons0 + rowg : g.consU + (rowg - g.n);
        for (int j = lane; j < cap; j += 32) row_s[j] = ids[j];
        int cnt = *cntp;
        int cons = *consp;
        const uint8_t *cy = g.codes + (size_t)y * g.mpad;
        __syncwarp();
        for (int64_t t = h; t < e; ++t) {
            const int x = (int)(keys[t] & 0xffffffffu);
            if (cnt < cap) {
                if (lane == 0) row_s[cnt] = x;
                ++cnt;
                cons = 0;
                ++n_app;
                __syncwarp();
                continue;
            }
            ++n_prune;
            // candidates: row + x, keys (d(y,u) << 32 | u), sorted (fa_sort_pairs)
            int np = 32;
            while (np < cap + 1) np <<= 1;
            for (int j = lane; j < np; j += 32) {
                unsigned long long k = KEY_MAX;
                if (j <= cap) {
                    int u = j < cap ? row_s[j] : x;
                    uint32_t d = sdt_sum_u_uniform(sdtN, g.m, cy, g.codes + (size_t)u * g.mpad);
                    k = ((unsigned long long)d << 32) | (uint32_t)u;
                }
                cand[j] = k;
            }
            n_sym += cap + 1;
            __syncwarp();
            warp_bitonic_smem(cand, np, lane);
            int nk;
            const uint8_t *cx = g.codes + (size_t)x * g.mpad;
            if (cons) {
                // position of x in the sorted candidates
                int p = -1;
                for (int j = lane; j <= cap; j += 32)
                    if ((int)(cand[j] & 0xffffffffu) == x) p = j;
#pragma unroll
                for (int o = 16; o; o >>= 1) p = max(p, __shfl_xor_sync(0xffffffffu, p, o));
                const uint32_t dx = (uint32_t)(cand[p] >> 32);
                bool dom = false;  // some earlier (kept) candidate dominates x
                for (int j = lane; j < p; j += 32) {
                    const uint8_t *cu = g.codes + (size_t)(uint32_t)(cand[j] & 0xffffffffu) * g.mpad;
                    dom |= sdt_sum_rows(sdtT, g.m, cu, cx) < dx;
                }
                const bool xkept = !__any_sync(0xffffffffu, dom);
                n_sym += p;
                // survivors in order; L_j (j > p) drops iff x kept and x dominates it
                nk = 0;
                for (int base2 = 0; base2 <= cap; base2 += 32) {
                    int j = base2 + lane;
                    bool keep = false;
                    int u = -1;
                    if (j <= cap) {
                        u = (int)(cand[j] & 0xffffffffu);
                        if (j < p) keep = true;
                        else if (j == p) keep = xkept;
                        else {
                            keep = true;
                            if (xkept) {
                                uint32_t dj = (uint32_t)(cand[j] >> 32);
                                keep = sdt_sum_u_uniform(sdtN, g.m, cx,
                                                         g.codes + (size_t)u * g.mpad) >= dj;
                            }
                        }
                    }
                    unsigned bk = __ballot_sync(0xffffffffu, keep);
                    int pos = nk + __popc(bk & ((1u << lane) - 1u));
                    if (keep && pos < cap) kept[pos] = u;
                    nk += __popc(bk);
                }
                if (xkept) n_sym += cap - p;
                nk = min(nk, cap);
            } else {
                unsigned long long sym = 0;
                nk = warp_select_heur(
                    sdtT, g.m, g.mpad, g.codes, g.mpad, cap + 1, cap,
                    [&](int j, int &v, double &dv) {
                        unsigned long long k = cand[j];
                        v = (int)(k & 0xffffffffu);
                        dv = (double)(uint32_t)(k >> 32);
                    },
                    kept, kcodes, lane, &sym);
                n_sym += sym;
            }
            __syncwarp();
            for (int j = lane; j < cap; j += 32) row_s[j] = j < nk ? kept[j] : -1;
            cnt = nk;
            cons = 1;
            __syncwarp();
        }
        for (int j = lane; j < cap; j += 32) ids[j] = j < cnt ? row_s[j] : -1;
        if (lane == 0) {
            *cntp = cnt;
            *consp = (uint8_t)cons;
        }
        __syncwarp();
    }
    if (lane == 0 && (n_prune | n_app)) {
        atomicAdd(ctr + 1, n_sym);
        atomicAdd(ctr + 4, n_prune);
        atomicAdd(ctr + 5, n_app);
    }
}

}  // namespace fa
