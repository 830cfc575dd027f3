// K6: grouped reverse-edge insertion (reverse_add, _core.pyx:441-477).
//
// The batch's forward selections emit requests (row(y, layer) << 32 | x);
// each row applies its incoming x in ascending order, which is the order the
// sequential reference applies them in.  The requests are bucketed
// by row without a sort: the search kernel counts each target row and lists
// the rows a batch touches; bucket_place_kernel gives every touched row a
// contiguous segment (its head), bucket_scatter_kernel drops each request
// into its row's segment (in arbitrary order), and the reverse warp that
// owns the segment applies its requests in ascending x (a warp minimum per
// step for segments of <= 32, a rank sort into scratch for longer ones).
// reverse_kernel's warps pull segments dynamically and replay the
// reference's per-edge rule exactly:
//   count < cap : append x (write_code_slot + id, count+1)
//   count == cap: d(y,u) = sdt-sum for all cap+1 candidates, sort by (d, id)
//                 (fa_sort_pairs), select_heur(cap), rewrite the row.
// Fast path: a row whose content is exactly the previous prune's output (kept
// order = ascending (d, id), pairwise non-dominated) keeps every member that x
// does not dominate, so the prune of L + {x} needs only the sums against x and
// no sort — decision-identical to the full scan.
#include "kernels.cuh"

namespace fa {

// sum_i tab[(i << 8) + (p_i << 4) + q_i] over i < m, saturated at 255; p, q
// are code rows of the flat table (16-byte aligned, zero padded to mpad).
// With p uniform across the warp every lane reads inside one 16-byte row.
__device__ __forceinline__ uint32_t sdt_sum16(const uint8_t *tab, int m,
                                              const uint8_t *__restrict__ p,
                                              const uint8_t *__restrict__ q) {
    uint32_t acc = 0;
    for (int i0 = 0; i0 < m; i0 += 16) {
        const uint4 wp = __ldg(reinterpret_cast<const uint4 *>(p + i0));
        const uint4 wq = __ldg(reinterpret_cast<const uint4 *>(q + i0));
        const uint32_t P[4] = {wp.x, wp.y, wp.z, wp.w};
        const uint32_t Q[4] = {wq.x, wq.y, wq.z, wq.w};
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int i = i0 + 4 * w + b;
                if (i < m)
                    acc += tab[(i << 8) + (((P[w] >> (8 * b)) & 0xffu) << 4) +
                               ((Q[w] >> (8 * b)) & 0xffu)];
            }
    }
    return acc > 255u ? 255u : acc;
}

// Segments of the touched rows: row touched[t] gets [heads[t], heads[t] +
// rowcnt[row]), allocated in warp-sized groups from *cursor; rowcnt of the
// row is reset to 0 (bucket_scatter_kernel counts it up again as its fill
// pointer; the reverse warp zeroes it once the segment is applied).
__global__ void bucket_place_kernel(const int32_t *__restrict__ touched,
                                    const int *__restrict__ ntouched, int32_t *__restrict__ rowcnt,
                                    int32_t *__restrict__ rowoff, int64_t *__restrict__ heads,
                                    int *__restrict__ cursor) {
    const int nt = *ntouched;
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int t0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; t0 < nt; t0 += warps * 32) {
        const int t = t0 + lane;
        int row = 0, c = 0;
        if (t < nt) {
            row = touched[t];
            c = rowcnt[row];
            rowcnt[row] = 0;
        }
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        int base = 0;
        if (lane == 31) base = atomicAdd(cursor, incl);
        base = __shfl_sync(0xffffffffu, base, 31);
        if (t < nt) {
            rowoff[row] = base + incl - c;
            // the segment record: its length above its head (the row is
            // touched[t]), so a reverse warp needs neither the keys nor a scan
            // for the segment's end before it can fetch the row
            heads[t] = ((int64_t)c << 32) | (int64_t)(base + incl - c);
        }
    }
}

// Every request into its row's segment; out[total] = KEY_MAX terminates the
// last segment (segments of different rows abut, so a row change ends one).
__global__ void bucket_scatter_kernel(const unsigned long long *__restrict__ req, int64_t N,
                                      int32_t *__restrict__ fill,
                                      const int32_t *__restrict__ rowoff,
                                      const int *__restrict__ cursor,
                                      unsigned long long *__restrict__ out) {
    if (blockIdx.x == 0 && threadIdx.x == 0) out[*cursor] = KEY_MAX;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = req[i];
        if (k == KEY_MAX) continue;
        const int64_t row = (int64_t)(k >> 32);
        out[rowoff[row] + atomicAdd(fill + row, 1)] = k;
    }
}

// The segment [h, e) of one row in ascending x: segments of <= 32 requests
// stay in registers (lane j: the j-th key, unordered) and each step takes
// the warp minimum; longer ones are rank-sorted into g.seg_scratch[h, e).
struct SegOrder {
    uint32_t kx;                           // this lane's unconsumed x (~0 = none)
    const unsigned long long *sorted;      // long segments: the ordered keys
    __device__ __forceinline__ void init(const Graph &g, const unsigned long long *keys,
                                         unsigned long long kk, int64_t h, int64_t e, int lane) {
        const int64_t L = e - h;
        sorted = nullptr;
        kx = lane < L ? (uint32_t)kk : 0xffffffffu;
        if (L > 32) {
            for (int64_t j = lane; j < L; j += 32) {
                const unsigned long long kj = keys[h + j];
                int64_t r = 0;
                for (int64_t i = 0; i < L; ++i) r += keys[h + i] < kj;
                g.seg_scratch[h + r] = kj;
            }
            __syncwarp();
            sorted = g.seg_scratch;
        }
    }
    // x of the t-th request (t = h, h + 1, ... in order)
    __device__ __forceinline__ int next(int64_t t) {
        if (sorted) return (int)(sorted[t] & 0xffffffffu);
        const uint32_t m = __reduce_min_sync(0xffffffffu, kx);
        if (kx == m) kx = 0xffffffffu;
        return (int)m;
    }
};

// RC: row chunks of 32 slots compiled in (cap <= 32 RC)
// 64 registers: 32 warps per SM (the kernel is latency-bound; its shared
// workspace is ~3.7 KB per warp once the rare full prune's select workspace
// lives in global scratch)
#ifndef FA_REV_MAXNREG
#define FA_REV_MAXNREG 64
#endif
template <int RC>
__global__ void __maxnreg__(FA_REV_MAXNREG) reverse_kernel(
    Graph g, const uint8_t *__restrict__ sdt, const uint8_t *__restrict__ sdtT,
    const unsigned long long *__restrict__ keys, int64_t N, const int64_t *__restrict__ heads,
    const int *__restrict__ nheads, int *__restrict__ next, const int32_t *__restrict__ upper_owner,
    ReverseLayout L, unsigned long long *__restrict__ ctr, uint8_t *__restrict__ sel_scratch,
    int sel_bytes) {
    // sdt, sdtT: the SDT and its transpose in global memory (L1-resident)
    extern __shared__ __align__(256) uint8_t smem[];
    const int lane = lane_id();
    const int wid = threadIdx.x >> 5;
    uint8_t *base = smem + wid * L.total;
    uint8_t *tdom = base + L.tdom;
    uint8_t *tkeep = base + L.tkeep;
    const uint32_t tdom_a = (uint32_t)__cvta_generic_to_shared(tdom);
    const uint32_t tkeep_a = (uint32_t)__cvta_generic_to_shared(tkeep);
    int32_t *row_s = reinterpret_cast<int32_t *>(base + L.row);
    uint8_t *rowd_s = base + L.rowd;
    uint8_t *keptd = base + L.keptd;
    unsigned long long *cand = reinterpret_cast<unsigned long long *>(base + L.cand);
    int32_t *kept = reinterpret_cast<int32_t *>(base + L.sel);  // fast prune's output
    // this warp's global select workspace (full prunes: kept ids + codes)
    uint8_t *selws = sel_scratch + (size_t)(blockIdx.x * (blockDim.x >> 5) + wid) * sel_bytes;
    const int nseg = *nheads;
    unsigned long long n_prune = 0, n_app = 0, n_sym = 0, n_full = 0;
    while (true) {
        int s = 0;
        if (lane == 0) s = atomicAdd(next, 1);
        s = __shfl_sync(0xffffffffu, s, 0);
        if (s >= nseg) break;
        // segment s: row touched[s], requests keys[h, e)
        const int64_t rec = heads[s];
        const int64_t rowg = __ldg(g.touched + s);
        const int64_t h = rec & 0xffffffffll, e = h + (rec >> 32);
        // the segment's first 32 keys stay in registers (lane j: keys[h + j])
        const unsigned long long kk = h + lane < e ? keys[h + lane] : KEY_MAX;
        const bool l0 = rowg < g.n;
        const int y = l0 ? (int)rowg : upper_owner[rowg - g.n];
        const int cap = l0 ? g.cap0 : g.capU;
        int32_t *ids = l0 ? g.adj0 + rowg * g.cap0p : g.adjU + (rowg - g.n) * g.capUp;
        int32_t *cntp = l0 ? g.cnt0 + rowg : g.cntU + (rowg - g.n);
        uint8_t *consp = l0 ? g.cons0 + rowg : g.consU + (rowg - g.n);
        uint8_t *distp = l0 ? g.dist0 + rowg * g.cap0p : g.distU + (rowg - g.n) * g.capUp;
        int cnt = *cntp;
        int cons = *consp;
        for (int j = lane; j < cap; j += 32) {
            row_s[j] = ids[j];
            if (cons) rowd_s[j] = distp[j];
        }
        const uint8_t *cy = g.codes + (size_t)y * g.mpad;
        // y's code bytes of this lane's subspaces (lane + 32 k), packed
        uint32_t cyl = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = lane + 32 * k;
            if (i < g.m) cyl |= (uint32_t)__ldg(cy + i) << (8 * k);
        }
        bool dirty = false;
        SegOrder so;
        so.init(g, keys, kk, h, e, lane);
        __syncwarp();
        for (int64_t t = h; t < e; ++t) {
            const int x = so.next(t);
            if (cnt < cap) {
                if (lane == 0) row_s[cnt] = x;
                ++cnt;
                cons = 0;
                dirty = true;
                ++n_app;
                __syncwarp();
                continue;
            }
            ++n_prune;
            const uint8_t *cx = g.codes + (size_t)x * g.mpad;
            // d(y, x) = sum_i sdt[i][y_i][x_i], looked up directly (the SDT is
            // L1-resident): most prunes end at the p = cap test below, which
            // needs nothing else
            uint32_t dx;
            {
                uint32_t acc = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int i = lane + 32 * k;
                    if (i < g.m)
                        acc += __ldg(sdt + (i << 8) + (((cyl >> (8 * k)) & 0xffu) << 4) +
                                     __ldg(cx + i));
                }
                acc = __reduce_add_sync(0xffffffffu, acc);
                dx = acc > 255u ? 255u : acc;
            }
            const unsigned long long kx = ((unsigned long long)dx << 32) | (uint32_t)x;
            int nk = 0;
            const int32_t *kept_src = kept;
            if (cons) {
                // L = row_s is sorted by (d, id) and pairwise non-dominated, its
                // distances d(y, L_j) cached in rowd_s.  p = position of x among
                // the candidates; x survives iff no L_j (j < p) dominates it;
                // L_j (j >= p) drops iff x survives and dominates it.
                int p = 0;
                unsigned long long kj[RC];
#pragma unroll
                for (int c = 0; c < RC; ++c) {
                    const int j = c * 32 + lane;
                    kj[c] = KEY_MAX;
                    if (j < cap) kj[c] = ((unsigned long long)rowd_s[j] << 32) | (uint32_t)row_s[j];
                    p += __popc(__ballot_sync(0xffffffffu, kj[c] < kx));
                }
                n_sym += cap + 1 + p;
                // x after every member (p = cap; e.g. a saturated d(y, x) = 255
                // with x newer than all members): the members alone fill the
                // row before x is reached, so the prune leaves it unchanged
                // (and still consistent) — whether or not x is dominated
                if (p >= cap) continue;
                // Tdom[i][c] = sdt[i][c][x_i]: d(L_j, x) = sum_i Tdom[i][L_j,i]
                if (p > 0) {
                    build_row_table(sdtT, g.m, g.mpad, cx, tdom, lane);
                    __syncwarp();
                }
                // domination of x, one 32-member chunk at a time: the first
                // dominating member settles it
                bool xkept = true;
#pragma unroll
                for (int c = 0; c < RC; ++c) {
                    if (c * 32 >= p) break;
                    bool domx = false;
                    if (kj[c] < kx)
                        domx = row_table_sum(tdom_a, g.codes + (size_t)(uint32_t)kj[c] * g.mpad,
                                             g.mpad) < dx;
                    if (__any_sync(0xffffffffu, domx)) {
                        xkept = false;
                        break;
                    }
                }
                if (!xkept) continue;  // the row is unchanged (and still consistent)
                n_sym += cap - p;
                if (p < cap) {
                    // Tkeep[i][c] = sdt[i][x_i][c]: d(x, L_j) = sum_i Tkeep[i][L_j,i]
                    build_row_table(sdt, g.m, g.mpad, cx, tkeep, lane);
                    __syncwarp();
                }
                // survivors in candidate order: L_0..L_{p-1}, x, L_p..
#pragma unroll
                for (int c = 0; c < RC; ++c) {
                    const int j = c * 32 + lane;
                    bool keep = false;
                    int uj = -1;
                    if (j < cap) {
                        uj = (int)(kj[c] & 0xffffffffu);
                        keep = true;
                        if (j >= p)
                            keep = row_table_sum(tkeep_a, g.codes + (size_t)uj * g.mpad,
                                                 g.mpad) >= (uint32_t)(kj[c] >> 32);
                    }
                    const unsigned bk = __ballot_sync(0xffffffffu, keep);
                    if (keep) {
                        int pos = nk + __popc(bk & ((1u << lane) - 1u));
                        if (j >= p) ++pos;  // x sits at position p
                        if (pos < cap) {
                            kept[pos] = uj;
                            keptd[pos] = (uint8_t)(kj[c] >> 32);
                        }
                    }
                    nk += __popc(bk);
                }
                if (lane == 0 && p < cap) {
                    kept[p] = x;
                    keptd[p] = (uint8_t)dx;
                }
                nk = min(nk + 1, cap);
            } else {
                ++n_full;
                // candidates row + x with (d, id) keys, sorted by rank
                for (int j = lane; j <= cap; j += 32) {
                    if (j < cap) {
                        const int uj = row_s[j];
                        const uint32_t dj = sdt_sum16(sdt, g.m, cy, g.codes + (size_t)uj * g.mpad);
                        cand[j] = ((unsigned long long)dj << 32) | (uint32_t)uj;
                    } else {
                        cand[j] = kx;
                    }
                }
                __syncwarp();
                unsigned long long mine[RC + 1];
                int rk[RC + 1];
#pragma unroll
                for (int c = 0; c <= RC; ++c) {
                    const int j = c * 32 + lane;
                    rk[c] = -1;
                    if (j <= cap) {
                        mine[c] = cand[j];
                        rk[c] = count_less(cand, cap + 1, mine[c]);
                    }
                }
                __syncwarp();
#pragma unroll
                for (int c = 0; c <= RC; ++c)
                    if (rk[c] >= 0) cand[rk[c]] = mine[c];
                __syncwarp();
                unsigned long long sym = 0;
                int32_t *kept_sel;
                nk = warp_select_tv(
                    sdtT, g.m, g.mpad, g.codes, g.mpad, cap + 1, cap,
                    [&](int j, int &v, uint32_t &dv) {
                        unsigned long long k = cand[j];
                        v = (int)(k & 0xffffffffu);
                        dv = (uint32_t)(k >> 32);
                    },
                    selws, lane, &sym, kept_sel, keptd, tkeep);
                kept_src = kept_sel;
                n_sym += cap + 1 + sym;
            }
            __syncwarp();
            for (int j = lane; j < cap; j += 32) {
                row_s[j] = j < nk ? kept_src[j] : -1;
                rowd_s[j] = j < nk ? keptd[j] : 0;
            }
            cnt = nk;
            cons = 1;
            dirty = true;
            __syncwarp();
        }
        if (dirty) {
            for (int j = lane; j < cap; j += 32) {
                ids[j] = j < cnt ? row_s[j] : -1;
                if (cons) distp[j] = rowd_s[j];
            }
            if (lane == 0) {
                *cntp = cnt;
                *consp = (uint8_t)cons;
            }
        }
        if (lane == 0) g.rowcnt[rowg] = 0;  // the row's bucket count, for the next batch
        __syncwarp();
    }
    if (lane == 0 && (n_prune | n_app)) {
        atomicAdd(ctr + 1, n_sym);
        atomicAdd(ctr + 4, n_prune);
        atomicAdd(ctr + 5, n_app);
        atomicAdd(ctr + 6, n_full);
    }
}

// Exact kind (kind 0): the same row segments and the same two prune paths as
// reverse_kernel, with fp32 L2 distances (symmetric: d(a, b) = d(b, a) bit
// for bit) computed four pairs at a time by 8-lane groups.  Fast path (the row
// is a prune output, its owner distances cached as fp32 bits): d(y, x), then
// d(L_j, x) for the members closer than x until one dominates, then the keep
// test of the rest.  Full path (rows written by appends / forward writes):
// d(y, u) for the row and x, (d, id) sort, select_heur (reverse_add,
// _core.pyx:441-477).
__global__ void __maxnreg__(96) reverse_exact_kernel(
    Graph g, const unsigned long long *__restrict__ keys, int64_t N,
    const int64_t *__restrict__ heads, const int *__restrict__ nheads, int *__restrict__ next,
    const int32_t *__restrict__ upper_owner, ReverseLayout L, unsigned long long *__restrict__ ctr) {
    extern __shared__ __align__(256) uint8_t smem[];
    const int lane = lane_id();
    const int wid = threadIdx.x >> 5;
    uint8_t *base = smem + wid * L.total;
    int32_t *row_s = reinterpret_cast<int32_t *>(base + L.row);
    unsigned long long *cand = reinterpret_cast<unsigned long long *>(base + L.cand);
    int32_t *kept = reinterpret_cast<int32_t *>(base + L.sel);
    float *qv = reinterpret_cast<float *>(base + L.qv);
    float *cv = reinterpret_cast<float *>(base + L.cv);
    int32_t *cid = reinterpret_cast<int32_t *>(base + L.cid);
    uint32_t *cd = reinterpret_cast<uint32_t *>(base + L.cd);
    uint32_t *kd = reinterpret_cast<uint32_t *>(base + L.kd);
    uint32_t *rowd = reinterpret_cast<uint32_t *>(base + L.rowd32);
    uint32_t *keptd = reinterpret_cast<uint32_t *>(base + L.keptd32);
    uint8_t *kflag = base + L.kflag;
    const int nseg = *nheads;
    unsigned long long n_prune = 0, n_app = 0, n_sym = 0, n_full = 0;
    while (true) {
        int s = 0;
        if (lane == 0) s = atomicAdd(next, 1);
        s = __shfl_sync(0xffffffffu, s, 0);
        if (s >= nseg) break;
        const int64_t rec = heads[s];
        const int64_t rowg = __ldg(g.touched + s);
        const int64_t h = rec & 0xffffffffll, e = h + (rec >> 32);
        const unsigned long long kk = h + lane < e ? keys[h + lane] : KEY_MAX;
        const bool l0 = rowg < g.n;
        const int y = l0 ? (int)rowg : upper_owner[rowg - g.n];
        const int cap = l0 ? g.cap0 : g.capU;
        int32_t *ids = l0 ? g.adj0 + rowg * g.cap0p : g.adjU + (rowg - g.n) * g.capUp;
        int32_t *cntp = l0 ? g.cnt0 + rowg : g.cntU + (rowg - g.n);
        uint8_t *consp = l0 ? g.cons0 + rowg : g.consU + (rowg - g.n);
        uint32_t *distp = reinterpret_cast<uint32_t *>(l0 ? g.dist0 : g.distU) +
                          (l0 ? rowg * g.cap0p : (rowg - g.n) * g.capUp);
        int cnt = *cntp;
        int cons = *consp;
        for (int j = lane; j < cap; j += 32) {
            row_s[j] = ids[j];
            if (cons) rowd[j] = distp[j];
        }
        const float *vy = g.vecs + (size_t)y * g.dim;
        bool have_y = false, dirty = false;
        SegOrder so;
        so.init(g, keys, kk, h, e, lane);
        __syncwarp();
        for (int64_t t = h; t < e; ++t) {
            const int x = so.next(t);
            if (cnt < cap) {
                if (lane == 0) row_s[cnt] = x;
                ++cnt;
                cons = 0;
                dirty = true;
                ++n_app;
                __syncwarp();
                continue;
            }
            ++n_prune;
            int nk = 0;
            if (cons) {
                // x's vector staged; d(y, x) from lane group 0
                for (int i = lane; i < g.dim; i += 32) cv[i] = __ldg(g.vecs + (size_t)x * g.dim + i);
                __syncwarp();
                const uint32_t dx = __shfl_sync(
                    0xffffffffu,
                    __float_as_uint(warp_l2_group8(lane < 8 ? cv : nullptr,
                                                   lane < 8 ? vy : nullptr, g.dim, lane)),
                    0);
                const unsigned long long kx = ((unsigned long long)dx << 32) | (uint32_t)x;
                // warp-uniform chunk loop, full-mask ballots (lanes past cap vote false)
                int p = 0;
                for (int c0 = 0; c0 < cap; c0 += 32) {
                    const int j = c0 + lane;
                    bool lt = false;
                    if (j < cap)
                        lt = (((unsigned long long)rowd[j] << 32) | (uint32_t)row_s[j]) < kx;
                    p += __popc(__ballot_sync(0xffffffffu, lt));
                }
                n_sym += cap + 1 + p;
                if (p >= cap) continue;  // x after every member: the row is unchanged
                // domination of x by a closer member, four at a time
                bool xkept = true;
                for (int b0 = 0; b0 < p; b0 += 4) {
                    const int j = b0 + (lane >> 3);
                    const float *a = j < p ? g.vecs + (size_t)row_s[j] * g.dim : nullptr;
                    const float d = warp_l2_group8(j < p ? cv : nullptr, a, g.dim, lane);
                    const bool dom = (lane & 7) == 0 && j < p && __float_as_uint(d) < dx;
                    if (__any_sync(0xffffffffu, dom)) {
                        xkept = false;
                        break;
                    }
                }
                if (!xkept) continue;  // the row is unchanged (and still consistent)
                n_sym += cap - p;
                // the farther members stay unless x dominates them
                for (int b0 = p; b0 < cap; b0 += 4) {
                    const int j = b0 + (lane >> 3);
                    const float *a = j < cap ? g.vecs + (size_t)row_s[j] * g.dim : nullptr;
                    const float d = warp_l2_group8(j < cap ? cv : nullptr, a, g.dim, lane);
                    if ((lane & 7) == 0 && j < cap) kflag[j] = __float_as_uint(d) >= rowd[j];
                }
                __syncwarp();
                // survivors in candidate order: L_0..L_{p-1}, x, L_p..
                for (int c0 = 0; c0 < cap; c0 += 32) {
                    const int j = c0 + lane;
                    const bool keep = j < cap && (j < p || kflag[j]);
                    const unsigned bk = __ballot_sync(0xffffffffu, keep);
                    if (keep) {
                        int pos = nk + __popc(bk & ((1u << lane) - 1u)) + (j >= p ? 1 : 0);
                        if (pos < cap) {
                            kept[pos] = row_s[j];
                            keptd[pos] = rowd[j];
                        }
                    }
                    nk += __popc(bk);
                }
                if (lane == 0 && p < cap) {
                    kept[p] = x;
                    keptd[p] = dx;
                }
                nk = min(nk + 1, cap);
            } else {
                ++n_full;
                if (!have_y) {
                    for (int i = lane; i < g.dim; i += 32) qv[i] = __ldg(vy + i);
                    have_y = true;
                }
                for (int j = lane; j <= cap; j += 32) cid[j] = j < cap ? row_s[j] : x;
                __syncwarp();
                ExactDist::dists(g, reinterpret_cast<const uint8_t *>(qv), cid, cap + 1, cd, lane);
                for (int j = lane; j <= cap; j += 32)
                    cand[j] = ((unsigned long long)cd[j] << 32) | (uint32_t)cid[j];
                __syncwarp();
                unsigned long long mine[kRowChunks + 1];
                int rk[kRowChunks + 1];
#pragma unroll
                for (int c = 0; c <= kRowChunks; ++c) {
                    const int j = c * 32 + lane;
                    rk[c] = -1;
                    if (j <= cap) {
                        mine[c] = cand[j];
                        rk[c] = count_less(cand, cap + 1, mine[c]);
                    }
                }
                __syncwarp();
#pragma unroll
                for (int c = 0; c <= kRowChunks; ++c)
                    if (rk[c] >= 0) cand[rk[c]] = mine[c];
                __syncwarp();
                unsigned long long sym = 0;
                nk = warp_select_exact(
                    g, cap + 1, cap,
                    [&](int j, int &v, uint32_t &dv) {
                        const unsigned long long k = cand[j];
                        v = (int)(k & 0xffffffffu);
                        dv = (uint32_t)(k >> 32);
                    },
                    kept, cv, kd, lane, &sym, keptd);
                n_sym += cap + 1 + sym;
            }
            __syncwarp();
            for (int j = lane; j < cap; j += 32) {
                row_s[j] = j < nk ? kept[j] : -1;
                rowd[j] = j < nk ? keptd[j] : 0u;
            }
            cnt = nk;
            cons = 1;
            dirty = true;
            __syncwarp();
        }
        if (dirty) {
            for (int j = lane; j < cap; j += 32) {
                ids[j] = j < cnt ? row_s[j] : -1;
                if (cons) distp[j] = rowd[j];
            }
            if (lane == 0) {
                *cntp = cnt;
                *consp = (uint8_t)cons;
            }
        }
        if (lane == 0) g.rowcnt[rowg] = 0;  // the row's bucket count, for the next batch
        __syncwarp();
    }
    if (lane == 0 && (n_prune | n_app)) {
        atomicAdd(ctr + 1, n_sym);
        atomicAdd(ctr + 4, n_prune);
        atomicAdd(ctr + 5, n_app);
        atomicAdd(ctr + 6, n_full);
    }
}

template __global__ void reverse_kernel<2>(Graph, const uint8_t *, const uint8_t *,
                                           const unsigned long long *, int64_t, const int64_t *,
                                           const int *, int *, const int32_t *, ReverseLayout,
                                           unsigned long long *, uint8_t *, int);
template __global__ void reverse_kernel<kRowChunks>(Graph, const uint8_t *, const uint8_t *,
                                                    const unsigned long long *, int64_t,
                                                    const int64_t *, const int *, int *,
                                                    const int32_t *, ReverseLayout,
                                                    unsigned long long *, uint8_t *, int);

}  // namespace fa
