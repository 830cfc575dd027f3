// K4/K7: warp-per-point best-first layer search with (d, id) total order,
// greedy upper-layer descent, and the shared per-warp workspace.
//
// Reference semantics restated with a strict total order:
//   search_layer (_core.pyx:278-342)  -> layer_search below
//   hill_climb   (_core.pyx:345-385)  -> hill_climb below
// key(u) = (d(u) << 32) | (u << 1) | expanded, d = min(sum ADT, 255).
//
// Device graph layout (B200-first, SoA instead of the reference's inlined
// blocks, layout.py:1-45): per layer, ids rows of `capp` int32 (cap rounded to
// 32 -> 128-byte aligned rows, -1 beyond the live count) + a count array, and
// one flat code table n x mpad bytes (mpad = m rounded to 16, zero padded).
// A visited neighbour costs only its 4-byte id; fresh neighbours gather their
// m code bytes from the L2-resident code table.
#pragma once

#include <type_traits>

#include "select.cuh"

#ifndef FA_PHASE_PROFILE
#define FA_PHASE_PROFILE 0
#endif

namespace fa {

struct Graph {
    int64_t n;
    int m, mpad;
    int cap0, capU;    // live capacity per layer kind (2R, R)
    int cap0p, capUp;  // row stride in int32
    int32_t *adj0, *cnt0;
    int32_t *adjU, *cntU;
    uint8_t *cons0, *consU;  // row holds exactly a prune result, in order
    uint8_t *dist0, *distU;  // per slot: SDT distance owner -> member (valid iff cons)
    const uint8_t *codes;    // n x mpad
    const int32_t *levels;
    const int64_t *uoff;
    int64_t nU;
    int tie;     // tie order of the searches (TieOrder modes)
    int expand;  // frontier entries expanded per step (1 = semantic core)
    uint32_t *gvis;        // global visited tables, gvis_nslots of 2^gvis_log2 (or null)
    uint32_t *gvis_epoch;  // their epoch counters
    uint32_t *gvis_owner;  // 1 while a search holds the slot (claimed atomically)
    int gvis_log2, gvis_nslots;
    int gvis_words;        // u32 words per entry: 1 (narrow ids), 2 (wide: 64-bit entries)
    const float *vecs;     // n x dim vectors (exact kind: every distance; rerank)
    int dim;
    // reverse-request bucketing of a build batch (reverse.cu): requests per
    // row (n + nU, zero between batches), the rows touched by the batch and
    // their count, and scratch for ordering long row segments
    int32_t *rowcnt;
    int32_t *touched;
    int *ntouched;
    unsigned long long *seg_scratch;
};

constexpr int kMaxExpand = 8;

// candidate slots one search step can produce: E rows of up to cap ids
__host__ __device__ inline int cand_capacity(int expand, int capmax) {
    const int e = expand > 1 ? (expand < kMaxExpand ? expand : kMaxExpand) : 1;
    return e * round_up(capmax, 32);
}
__host__ __device__ inline int cand_capacity(const Graph &g) {
    return cand_capacity(g.expand, g.cap0 > g.capU ? g.cap0 : g.capU);
}

__device__ __forceinline__ const int32_t *row_ids(const Graph &g, int layer, int v) {
    if (layer == 0) return g.adj0 + (int64_t)v * g.cap0p;
    return g.adjU + (__ldg(g.uoff + v) + layer - 1) * g.capUp;
}
// Row addressing of one layer, set up once per layer search: base + index *
// stride, the index the vertex itself on layer 0 and its upper-row offset
// above (one predicated load); keeps the per-step address to a few
// instructions instead of re-deriving both cases from the kernel parameters
struct RowAddr {
    const int32_t *base;
    const int64_t *uoff;  // null on layer 0
    int stride;
    __device__ __forceinline__ RowAddr(const Graph &g, int layer) {
        if (layer == 0) {
            base = g.adj0;
            uoff = nullptr;
            stride = g.cap0p;
        } else {
            base = g.adjU + (int64_t)(layer - 1) * g.capUp;
            uoff = g.uoff;
            stride = g.capUp;
        }
    }
    __device__ __forceinline__ const int32_t *operator()(int v) const {
        // row indices and strides are below 2^31: one 32 x 32 -> 64 multiply
        const uint32_t i = uoff ? (uint32_t)__ldg(uoff + v) : (uint32_t)v;
        return base + (uint64_t)i * (uint32_t)stride;
    }
};
__device__ __forceinline__ int layer_cap(const Graph &g, int layer) {
    return layer == 0 ? g.cap0 : g.capU;
}

// ---- per-warp workspace ----------------------------------------------------
// Largest search width kept in registers (lane l owns slots l + 32 j, j < 16);
// wider searches keep their result set in shared memory.
constexpr int kRegSetMax = 512;

// Visited table geometry for a requested size of 2^hlog2 16-bit slots: buckets
// of 8 slots, at least 2^9 buckets (15-bit remainders of 24-bit ids); below
// 2^12 slots only the first 2^hlog2 / 512 slots of each bucket are used.
__host__ __device__ inline int vis_buckets_log2(int hlog2) { return hlog2 > 12 ? hlog2 - 3 : 9; }
__host__ __device__ inline int vis_bucket_slots(int hlog2) {
    return hlog2 >= 12 ? 8 : 1 << (hlog2 > 9 ? hlog2 - 9 : 0);
}

// Per-warp shared memory, in two blocks: a 256-aligned block (the ADT rows
// and the visited table, both addressed by PRMT-merged byte offsets) and a
// small block (candidate keys, tie queue, fresh ids/distances).  A CTA of w
// warps holds w big blocks, then w small blocks: total = w * (big + small).
struct WarpLayout {
    int adt, hash, big;                  // offsets in the big block
    int T, S, TQ, fresh, fdist, small;   // offsets in the small block (T: see t_big)
    int t_big;                           // T lives at the end of the visited table
    int total;
    int hash_log2;
    __host__ __device__ static int adt_bytes(int mpad) { return round_up(mpad * 16, 256); }
    // t_alias: the sorted results live at the end of the visited table (the
    // build: the table is dead once a layer search has sorted its results, and
    // forward selection's kept rows use only its start)
    // ctx_bytes: the query context (default: the ADT, mpad x 16; the exact
    // kind: the query vector, dim x 4); key_bytes: 4 (Flash) or 8 (exact)
    // t_alias 2: the sorted results overlay the small block's search state
    // (candidate keys, tie queue, fresh ids/distances: all dead once a layer
    // search has sorted its results) -- the build, when the results do not
    // fit beside the selection workspace in the visited table
    __host__ __device__ void init(int mpad, int W, int capmax, int hlog2, int expand,
                                  int t_alias = 0, int ctx_bytes = -1, int key_bytes = 4) {
        hash_log2 = hlog2;
        const int nc = cand_capacity(expand, capmax);
        const int Wp = round_up(W, 32);
        const int hbytes = 16 << vis_buckets_log2(hlog2);
        t_big = t_alias == 1 && W <= kRegSetMax;
        const bool t_small = t_alias == 2 && W <= kRegSetMax;
        adt = 0;
        hash = ctx_bytes < 0 ? adt_bytes(mpad) : round_up(ctx_bytes, 256);
        big = hash + hbytes;  // a multiple of 256
        int o = 0;
        if (t_big) {
            T = hash + hbytes - Wp * 8;
        } else if (t_small) {
            T = 0;
        } else {
            // sorted 64-bit results (+ 32-bit keys and flags when the set lives here)
            T = o;
            o += Wp * (W > kRegSetMax ? 8 + key_bytes + 1 : 8);
            o = round_up(o, 16);
        }
        // candidate keys; their rank-sorted copy overlays fresh + fdist (read
        // for the last time when the keys are formed)
        S = o; o += nc * key_bytes;
        TQ = o; o += Wp * 4;     // tie queue
        fresh = o; o += nc * 4;
        fdist = o; o += nc * 4;
        if (t_small && o < Wp * 8) o = Wp * 8;
        small = round_up(o, 16);
        total = big + small;
    }
};

// ADT rows in shared memory: 16-row chunks of 256 bytes (256-aligned), row r
// of chunk c stored at slot (r + c) mod 16, so the lane groups that read the
// same row of different chunks hit different banks.  A lookup address is then
// chunk base | byte, byte = slot * 16 + code: one PRMT merges a pre-offset code
// byte into the base.
__device__ __forceinline__ int adt_row_off(int r) {
    const int c = r >> 4;
    return (c << 8) + ((((r & 15) + c) & 15) << 4);
}

__device__ __forceinline__ void load_adt_smem(uint8_t *adt_s, const uint8_t *adt, int mpad,
                                              int lane) {
    for (int r = lane; r < mpad; r += 32)
        *reinterpret_cast<uint4 *>(adt_s + adt_row_off(r)) =
            __ldg(reinterpret_cast<const uint4 *>(adt + (size_t)r * 16));
}

// Saturated ADT distance of one code row (single vertex: entry point).
__device__ __forceinline__ uint32_t adt_one(const uint8_t *adt_s, const uint8_t *code, int mpad,
                                            int lane) {
    uint32_t s = 0;
    for (int r = lane; r < mpad; r += 32) s += adt_s[adt_row_off(r) + __ldg(code + r)];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s > 255u ? 255u : s;
}

// Distances of the nf ids in ids_s[] (shared) into out_s[] (shared).  G lanes
// per id (G = chunks rounded up to a power of two), each summing one
// 16-subspace chunk gathered with a 16-byte load.
// Lanes per id of dists_for: the id's 16-byte code chunks rounded up to a
// power of two (log2); a pass covers 32 >> lg ids.
__device__ __forceinline__ int dist_lanes_log2(int mpad) {
    const int chunks = mpad >> 4;
    return chunks <= 1 ? 0 : 32 - __clz(chunks - 1);
}

__device__ __forceinline__ void dists_for(const uint8_t *adt_s, const uint8_t *__restrict__ codes,
                                          int mpad, const int32_t *ids_s, int nf,
                                          uint32_t *out_s, int lane) {
    const int chunks = mpad >> 4;
    const int lg = dist_lanes_log2(mpad);
    const int G = 1 << lg;
    const int gi = lane >> lg, c = lane & (G - 1);
    const bool active = c < chunks;
    const uint32_t cbase = (uint32_t)__cvta_generic_to_shared(adt_s) + ((uint32_t)c << 8);
    // pre-offsets of the 4 code bytes of word q: slot((4q + b + c) mod 16) * 16
    uint32_t K[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
        K[q] = ((0x03020100u + 0x04040404u * (uint32_t)q + 0x01010101u * (uint32_t)c) &
                0x0f0f0f0fu)
               << 4;
    const uint8_t *cb = codes + c * 16;
    uint4 w = make_uint4(0, 0, 0, 0);
    if (gi < nf && active)
        w = __ldg(reinterpret_cast<const uint4 *>(cb + (size_t)ids_s[gi] * mpad));
    for (int base = 0; base < nf; base += (32 >> lg)) {
        const int f = base + gi;
        uint32_t sum = 0;
        if (f < nf && active) {
            const uint32_t W[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t e = W[q] + K[q];
                uint32_t b[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t a = prmt(e, cbase, 0x7650u + (uint32_t)k);
                    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(b[k]) : "r"(a));
                }
                sum += b[0] + b[1] + b[2] + b[3];
            }
        }
        // the next pass's code rows, in flight under this pass's reduction
        const int fn = f + (32 >> lg);
        if (fn < nf && active)
            w = __ldg(reinterpret_cast<const uint4 *>(cb + (size_t)ids_s[fn] * mpad));
        if (G > 1) sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        if (G > 2) sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        if (G > 4) sum += __shfl_xor_sync(0xffffffffu, sum, 4);
        if (c == 0 && f < nf) out_s[f] = sum > 255u ? 255u : sum;
    }
    __syncwarp();
}

// ---- visited set (exact) ---------------------------------------------------
// Shared tier: 2^kb buckets of eight 16-bit slots.  A 24-bit id maps through a
// bijection h = id * odd (mod 2^24) to bucket h >> (24 - kb) and remainder
// (h & low bits) + 1 (0 = empty), so a slot needs 16 bits and one 16-byte load
// tests a whole bucket.  Slots fill in order and are never removed; an id whose
// bucket is full lives in the global tier: an open-addressing table in global
// memory (L2-resident) holding (epoch << 24 | id), one per claimed slot.
// Entries of older epochs count as empty, so a slot's table is cleared only
// once every 255 searches.  Either way every id lives in exactly one tier.
//
// Global-tier slots are claimed per search with an atomic on an owner word
// (the probe starts at %smid / %warpid, which is free in the common case) and
// released when the search ends, so a preempted or migrated warp can never
// share a table with another live search.  The host sizes the pool to the
// launch's resident warps and each table (2^gvis_log2 entries) to the search
// width (gvis_log2_for).
constexpr int kMaxWarpsPerSM = 64;
constexpr uint32_t kVisMul = 0x9E3779B1u;

// log2 entries of a global-tier table for searches of width W over n vertices:
// room for every id such a search can plausibly visit (the shared tier holds
// the first few thousand), at a 3/4 load limit.
__host__ __device__ inline int gvis_log2_for(int W, int capmax, int64_t n) {
    int64_t want = 16 * (int64_t)W + 2 * (int64_t)capmax;
    if (want > n) want = n;
    want = want * 4 / 3 + 1;
    int l = 14;
    while (l < 20 && ((int64_t)1 << l) < want) ++l;
    return l;
}

__device__ __forceinline__ uint4 lds128_volatile(const uint4 *p) {
    uint4 v;
    asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"((uint32_t)__cvta_generic_to_shared(p))
                 : "memory");
    return v;
}

// The global tier's probe (ids whose shared bucket is full: the cold path,
// kept out of line so the hot loop stays compact).  0 = already visited,
// 2 = inserted.  Reads bypass L1 (the table may have been written on another SM
// by the slot's previous owner).
// Narrow entries are 32-bit (epoch << 24 | id), wide ones 64-bit
// (epoch << 32 | id).
constexpr int kGlobalMaxProbe = 256;
template <bool W>
static __device__ __noinline__ int global_visit(uint32_t *G32, int glog2, uint32_t epoch, int id) {
    using E = typename std::conditional<W, unsigned long long, uint32_t>::type;
    constexpr int kEpochShift = W ? 32 : 24;
    E *G = reinterpret_cast<E *>(G32);
    const uint32_t key = (uint32_t)id + 1u;
    const E gk = ((E)epoch << kEpochShift) | (E)((uint32_t)id & (W ? 0xffffffffu : 0xFFFFFFu));
    const uint32_t gmask = (1u << glog2) - 1u;
    uint32_t p = (key * 2654435761u) >> (32 - glog2);
    // a probe run this long only happens once the table is nearly full: report
    // overflow (FA_EOVERFLOW upstream) instead of probing on
    for (int probe = 0; probe < kGlobalMaxProbe;) {
        const E v = __ldcg(G + p);
        if (v == gk) return 0;
        if ((uint32_t)(v >> kEpochShift) != epoch) {
            const E old = atomicCAS(G + p, v, gk);
            if (old == v) return 2;
            if (old == gk) return 0;
            continue;
        }
        p = (p + 1u) & gmask;
        ++probe;
    }
    return 3;
}

// A warp's claimed global-tier table: claimed once per warp per launch (the
// build kernel's persistent warps keep it across their insertions), its epoch
// counted in a register and written back at release.
struct GSlot {
    uint32_t *G = nullptr;     // the table (null: no global tier)
    uint32_t *own = nullptr;   // its owner word
    uint32_t *ep = nullptr;    // its epoch word
    uint32_t epoch = 0;
};

__device__ __forceinline__ uint32_t gslot_hint() {
    uint32_t sm, w;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(w));
    return sm * kMaxWarpsPerSM + w;
}

// Claim a free slot (the probe starts at %smid / %warpid, free in the common
// case; the pool holds one slot per resident warp, so one is always free).
__device__ inline GSlot gslot_claim(const Graph &g, int lane) {
    GSlot gs;
    if (!g.gvis) return gs;
    uint32_t slot = 0, e = 0;
    if (lane == 0) {
        const uint32_t ns = (uint32_t)g.gvis_nslots;
        slot = gslot_hint() % ns;
        while (atomicCAS(g.gvis_owner + slot, 0u, 1u) != 0u) slot = (slot + 1u) % ns;
        e = atomicAdd(g.gvis_epoch + slot, 0u);  // the last owner's epoch (L2, coherent)
    }
    slot = __shfl_sync(0xffffffffu, slot, 0);
    gs.epoch = __shfl_sync(0xffffffffu, e, 0);
    gs.G = g.gvis + ((size_t)slot << g.gvis_log2) * g.gvis_words;
    gs.own = g.gvis_owner + slot;
    gs.ep = g.gvis_epoch + slot;
    return gs;
}
__device__ inline void gslot_release(const GSlot &gs, int lane) {
    __syncwarp();
    if (gs.G && lane == 0) {
        atomicExch(gs.ep, gs.epoch);
        __threadfence();
        atomicExch(gs.own, 0u);
    }
}

// KB: log2 of the shared tier's bucket count compiled in (0 = from hlog2 at
// run time); the build kernels fix it at 9 (the 8 KB table).
// W: wide ids (n >= 2^24): 32-bit shared slots (4 per bucket) holding a
// 32 - kb bit remainder + 1, 64-bit global entries.
template <int KB = 0, bool W = false>
struct VisitedSet {
    uint4 *B;          // shared tier buckets
    int kb;            // log2 buckets
    int nslots;        // usable slots per bucket
    uint32_t *G;       // global tier (the warp's claimed table)
    int glog2;
    uint32_t epoch;

    // a new search: clear the shared tier, advance the global tier's epoch
    // (entries of older epochs count as empty; the table is wiped once every
    // 255 searches)
    __device__ void begin(void *H, int hlog2, const Graph &g, GSlot &gs, int lane) {
        B = reinterpret_cast<uint4 *>(H);
        kb = KB ? KB : vis_buckets_log2(hlog2);
        nslots = W ? min(4, vis_bucket_slots(hlog2)) : vis_bucket_slots(hlog2);
        const uint4 z = make_uint4(0, 0, 0, 0);
        for (int i = lane; i < (1 << kb); i += 32) B[i] = z;
        glog2 = g.gvis_log2;
        G = gs.G;
        if (G) {
            uint32_t e = gs.epoch + 1u;
            if (e > 255u) {  // wrap: clear this slot's table once
                for (int i = lane; i < (1 << glog2) / (W ? 2 : 4); i += 32)
                    __stcg(reinterpret_cast<uint4 *>(G) + i, z);
                e = 1u;
            }
            gs.epoch = e;
            epoch = e;
        }
        __syncwarp();
    }

    // bucket of id and its remainder r (1 .. 2^(bits - kb)), bits = 24 or 32
    __device__ __forceinline__ uint4 *bucket(int id, uint32_t &r) const {
        constexpr int bits = W ? 32 : 24;
        const int k = KB ? KB : kb;
        const uint32_t h = ((uint32_t)id * kVisMul) & (W ? 0xffffffffu : 0xffffffu);
        r = (h & ((1u << (bits - k)) - 1u)) + 1u;
        return B + (h >> (bits - k));
    }
    // some 16-bit slot of v equals the remainder (rr = r in both halves):
    // unsigned 16x2 minimum of v ^ rr (VIMNMX) has a zero half
    __device__ static __forceinline__ bool holds(const uint4 &v, uint32_t rr) {
        const uint32_t m = __vminu2(__vminu2(v.x ^ rr, v.y ^ rr), __vminu2(v.z ^ rr, v.w ^ rr));
        return ((m & 0xffffu) == 0u) | (m < 0x10000u);
    }
    // filled slots (they fill in order, so also the first free one)
    __device__ static __forceinline__ int filled(const uint4 &v) {
        const uint32_t o = 0x00010001u;
        const uint32_t f = __vminu2(v.x, o) + __vminu2(v.y, o) + __vminu2(v.z, o) + __vminu2(v.w, o);
        return (int)((f & 0xffffu) + (f >> 16));
    }

    // 0 = already visited, 1 = new (shared tier), 2 = new (global tier),
    // 3 = the global tier is unavailable (overflow)
    __device__ int visit(int id) {
        uint32_t r;
        uint4 *bk = bucket(id, r);
        if constexpr (W) {
            uint4 v = *bk;
            while (true) {
                if ((v.x == r) | (v.y == r) | (v.z == r) | (v.w == r)) return 0;
                const int e = (v.x != 0u) + (v.y != 0u) + (v.z != 0u) + (v.w != 0u);
                if (e >= nslots) break;
                const uint32_t ow = (e & 2) ? ((e & 1) ? v.w : v.z) : ((e & 1) ? v.y : v.x);
                if (atomicCAS(reinterpret_cast<uint32_t *>(bk) + e, ow, r) == ow) return 1;
                v = lds128_volatile(bk);
            }
            return G == nullptr ? 3 : global_visit<true>(G, glog2, epoch, id);
        }
        const uint32_t rr = r * 0x10001u;
        uint4 v = *bk;  // the common case (a visited id) needs this one read
        while (true) {
            if (holds(v, rr)) return 0;
            const int e = filled(v);
            if (e >= nslots) break;
            const int wi = e >> 1;
            const uint32_t ow = (wi & 2) ? ((wi & 1) ? v.w : v.z) : ((wi & 1) ? v.y : v.x);
            const uint32_t nw = ow | (r << (16 * (e & 1)));
            if (atomicCAS(reinterpret_cast<uint32_t *>(bk) + wi, ow, nw) == ow) return 1;
            // another lane took the slot: re-read the bucket
            v = lds128_volatile(bk);
        }
        return G == nullptr ? 3 : global_visit<false>(G, glog2, epoch, id);
    }
};

// ---- sorted top-W buffer ---------------------------------------------------
constexpr unsigned long long KEY_MAX = ~0ull;

// sorted results: (d << 32 | tie id), the tie id a full 32 bits (wide keys)
__device__ __forceinline__ unsigned long long make_key(uint32_t d, uint32_t tie) {
    return ((unsigned long long)d << 32) | (unsigned long long)tie;
}
__device__ __forceinline__ uint32_t key_id(unsigned long long k) { return (uint32_t)k; }
__device__ __forceinline__ uint32_t key_d(unsigned long long k) { return (uint32_t)(k >> 32); }

// Order among equal distances inside one search.  mode 0: vertex id (the
// reference's semantic core, _pycore.py tuple order).  mode 1: a fixed
// bijective scramble of the id.  mode 2: the scramble salted per search (the
// inserted vertex / query), a deterministic stand-in for the compiled core's
// history-dependent heap order — without it, every insertion prefers the same
// (lowest-id) vertices among the many uint8 ties and the graph degrades
// (DESIGN.md §ties).  Keys carry the tie id; `back` recovers the vertex id.
constexpr uint32_t kTieMul = 0x2545F491u;
__host__ __device__ constexpr uint32_t tie_inverse(uint32_t a) {
    uint32_t x = a;
    for (int i = 0; i < 5; ++i) x *= 2u - a * x;
    return x;
}
struct TieOrder {
    int mode;
    uint32_t salt;
    uint32_t mask;  // tie-id bits: 24 (narrow keys, n < 2^24) or 32 (wide)
    __device__ static TieOrder make(int mode, uint32_t who, bool wide = false) {
        TieOrder t;
        t.mode = mode;
        t.mask = wide ? 0xffffffffu : 0xffffffu;
        t.salt = mode == 2 ? ((who + 1u) * 0x9E3779B1u) & t.mask : 0u;
        return t;
    }
    // an odd multiplier is a bijection modulo 2^24 and 2^32 alike
    __device__ __forceinline__ uint32_t fwd(uint32_t u) const {
        return mode ? ((u ^ salt) * kTieMul) & mask : u;
    }
    __device__ __forceinline__ int back(uint32_t t) const {
        return (int)(mode ? ((t * tie_inverse(kTieMul)) & mask) ^ salt : t);
    }
};

// number of entries of the unsorted (small) a[0..n) strictly less than x;
// every lane reads the same word: shared-memory broadcast
__device__ __forceinline__ int count_less(const unsigned long long *a, int n, unsigned long long x) {
    int c = 0;
    for (int j = 0; j < n; ++j) c += a[j] < x;
    return c;
}

// Per-search counters (32-bit: one search never reaches 2^32 of anything);
// kernels accumulate them into 64-bit totals.
struct SearchCounters {
    uint32_t dist, kcalls, visited, sym;
#if FA_PHASE_PROFILE
    // SM cycles per phase of layer_search (diagnostics, point_stats; build with
    // -DFA_PHASE_PROFILE=1): 0 pop + prediction, 1 row + visited filter,
    // 2 distances, 3 acceptance
    unsigned long long ph[4];
#endif
};

#if FA_PHASE_PROFILE
__device__ __forceinline__ long long phase_clock() { return clock64(); }
__device__ __forceinline__ void phase_mark(SearchCounters &c, int k, long long &t) {
    const long long now = clock64();
    c.ph[k] += (unsigned long long)(now - t);
    t = now;
}
#else
__device__ __forceinline__ long long phase_clock() { return 0; }
__device__ __forceinline__ void phase_mark(SearchCounters &, int, long long &) {}
#endif

// Warp-cooperative best-first search on one layer.
// On return T[0..ts) holds the result ascending by (d, id).
// Returns false on visited-hash overflow.
constexpr int kRowChunks = 4;  // id rows up to 128 slots (cap = 2R <= 127)

template <int RC = kRowChunks>
__device__ __forceinline__ void load_row(const int32_t *ids, int cap, int lane, int (&u)[RC]) {
#pragma unroll
    for (int k = 0; k < RC; ++k) {
        int j = k * 32 + lane;
        u[k] = j < cap ? __ldg(ids + j) : -1;
    }
}

// Best-first search on one layer with the reference's semantic-core rules
// (flashann/_pycore.py:246-283; ties by vertex id through tuple order):
//   * the frontier pops in (d, id) order; the search stops once the result set
//     is full and the popped distance exceeds the worst kept distance;
//   * an expansion's fresh neighbours are offered in ascending (d, id); one is
//     accepted while the set is not full or its distance is strictly below the
//     worst, evicting the worst (largest d, smallest id on ties).
// Representation (B200): the result set is an UNSORTED array of 32-bit keys
// (d << 24 | tie id) with an "expanded" byte each.  Pop = warp min-reduction
// over the unexpanded keys, eviction = min over the largest-distance group,
// acceptance = an O(1) append or slot replacement; the set is sorted once at
// the end.  Its unexpanded members are exactly the frontier entries that can
// still be popped, plus the tie queue TQ of unexpanded entries evicted at the
// current worst distance (a popped frontier entry with d > worst stops the
// search, so nothing else in the frontier can matter).  Evictions at one worst
// distance remove members of the last distance group, so TQ holds < W tie ids,
// ascending, and empties when the worst distance drops.
// On return T[0..ts) holds the result as 64-bit keys (make_key of the tie id)
// ascending by (d, tie id).  false = visited-set overflow.

// ---- distance policies -------------------------------------------------------
// fp32 L2 (fa_l2sq_f32 tree, common.cuh l2_tree) of four (query, vector) pairs
// at once: lane group g = lane / 8 handles pair g, lane k = lane % 8 owns
// accumulator k of the 8-wide main loop.  q may live in shared memory.  The
// result is valid in lane k == 0 of the group; null pointers = idle group.
__device__ __forceinline__ float warp_l2_group8(const float *q, const float *__restrict__ v,
                                                int d, int lane) {
    const int k = lane & 7;
    const int nfull = d >= 8 ? d / 8 : 0;
    float acc = 0.f;
    if (q && v)
        for (int c = 0; c < nfull; ++c) {
            const float e = __fsub_rn(q[8 * c + k], __ldg(v + 8 * c + k));
            acc = __fadd_rn(acc, __fmul_rn(e, e));
        }
    const unsigned full = 0xffffffffu;
    const float hi = __shfl_down_sync(full, acc, 4);
    const float vk = (k < 4) ? __fadd_rn(acc, hi) : 0.f;  // v[k] = acc[k] + acc[k+4]
    int i = 8 * nfull;
    const bool four = (d - i) >= 4;
    float wk = vk;
    if (four && k < 4 && q && v) {
        const float e = __fsub_rn(q[i + k], __ldg(v + i + k));
        wk = __fmaf_rn(e, e, vk);
    }
    const float w2 = __shfl_down_sync(full, wk, 2);
    const float t = __fadd_rn(wk, w2);  // lane0: w0+w2, lane1: w1+w3
    const float t1 = __shfl_down_sync(full, t, 1);
    float sum = __fadd_rn(t, t1);       // lane k == 0: (w0+w2)+(w1+w3)
    if (!four && nfull == 0) sum = 0.f;
    if (four) i += 4;
    if (k == 0 && q && v)
        for (; i < d; ++i) {
            const float e = __fsub_rn(q[i], __ldg(v + i));
            sum = __fmaf_rn(e, e, sum);
        }
    return sum;
}

// Key layout of a policy: (d << kShift) | tie id, tie ids of kShift bits.
// Narrow (W = false): 24-bit ids (n < 2^24), Flash keys fit 32 bits.  Wide
// (W = true, n >= 2^24): 32-bit ids, 64-bit keys (d << 32 | tie), 32-bit
// visited-set slots and 64-bit global-tier entries.
template <typename KeyT, bool W>
struct KeyLayout {
    using Key = KeyT;
    static constexpr bool kWide = W;
    static constexpr int kShift = W ? 32 : 24;
    static constexpr uint32_t kTieMask = W ? 0xffffffffu : 0xffffffu;
    __device__ static __forceinline__ Key key(uint32_t d, uint32_t tie) {
        return ((Key)d << kShift) | (Key)tie;
    }
    __device__ static __forceinline__ uint32_t dist(Key k) { return (uint32_t)(k >> kShift); }
    __device__ static __forceinline__ uint32_t tie(Key k) { return (uint32_t)k & kTieMask; }
};

// Flash (kind 4): keys (d << 24 | tie id) with the uint8 table distance d
// (wide: d << 32 | tie); the query context is the query's ADT in shared memory.
template <bool W>
struct FlashDistT : KeyLayout<typename std::conditional<W, uint64_t, uint32_t>::type, W> {
    static constexpr bool kExact = false;
    __device__ static __forceinline__ void dists(const Graph &g, const uint8_t *qc,
                                                 const int32_t *ids, int nf, uint32_t *out,
                                                 int lane) {
        dists_for(qc, g.codes, g.mpad, ids, nf, out, lane);
    }
    __device__ static __forceinline__ uint32_t one(const Graph &g, const uint8_t *qc, int v,
                                                   int lane) {
        return adt_one(qc, g.codes + (size_t)v * g.mpad, g.mpad, lane);
    }
};
using FlashDist = FlashDistT<false>;
using FlashDistW = FlashDistT<true>;

// Exact (kind 0, asym_one / sym_one of K_EXACT, _core.pyx:167-191): every
// distance is the fp32 L2 of the vectors; keys (fp32 bits << 24 | tie id) —
// the bit pattern of a non-negative float orders like its value (wide: << 32).
// The query context is the query vector in shared memory.
template <bool W>
struct ExactDistT : KeyLayout<uint64_t, W> {
    static constexpr bool kExact = true;
    __device__ static __forceinline__ void dists(const Graph &g, const uint8_t *qc,
                                                 const int32_t *ids, int nf, uint32_t *out,
                                                 int lane) {
        const float *q = reinterpret_cast<const float *>(qc);
        for (int base = 0; base < nf; base += 4) {
            const int j = base + (lane >> 3);
            const float *v = j < nf ? g.vecs + (size_t)ids[j] * g.dim : nullptr;
            const float s = warp_l2_group8(j < nf ? q : nullptr, v, g.dim, lane);
            if ((lane & 7) == 0 && j < nf) out[j] = __float_as_uint(s);
        }
        __syncwarp();
    }
    __device__ static __forceinline__ uint32_t one(const Graph &g, const uint8_t *qc, int v,
                                                   int lane) {
        const float *q = reinterpret_cast<const float *>(qc);
        const bool act = lane < 8;
        const float s = warp_l2_group8(act ? q : nullptr, act ? g.vecs + (size_t)v * g.dim : nullptr,
                                       g.dim, lane);
        return __shfl_sync(0xffffffffu, __float_as_uint(s), 0);
    }
};
using ExactDist = ExactDistT<false>;
using ExactDistW = ExactDistT<true>;

// ---- register-resident result set (W <= kRegSetMax) -------------------------
// Lane l owns slots l + 32 j (j < J); slot s is live iff s < ts.  Bit j of `fl`
// marks slot j expanded.  Every loop over j is unrolled (no dynamic register
// indexing), so pop / worst distance / eviction are register compares plus one
// warp reduction instead of passes over shared memory.
template <int J, typename P>
struct RegSet {
    using K = typename P::Key;
    K key[J];
    uint32_t fl;
    // this lane's live slots when the set holds ts entries (a prefix of j)
    __device__ __forceinline__ static uint32_t live_mask(int ts, int lane) {
        const int c = ts > lane ? (ts - lane + 31) >> 5 : 0;
        return c >= 32 ? 0xffffffffu : (1u << c) - 1u;
    }
    // smallest key (b1, slot j1; j1 = -1 if none) and second smallest key b2
    // over the slots of mask um
    __device__ __forceinline__ void min2(uint32_t um, K &b1, int &j1, K &b2) const {
        b1 = b2 = ~K(0);
        j1 = -1;
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const K k = key[j];
            if ((um >> j) & 1u) {
                if (j1 < 0 || k < b1) {
                    b2 = b1;
                    b1 = k;
                    j1 = j;
                } else {
                    b2 = min(b2, k);
                }
            }
        }
    }
    // eviction victim over the slots of mask lm: the largest distance, smallest
    // tie among those = the largest key ^ tie mask (vf; vj = -1 if none)
    __device__ __forceinline__ void victim(uint32_t lm, K &vf, int &vj) const {
        vf = 0;
        vj = -1;
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const K kf = key[j] ^ K(P::kTieMask);
            if (((lm >> j) & 1u) && (vj < 0 || kf > vf)) {
                vf = kf;
                vj = j;
            }
        }
    }
    // largest distance over the live slots
    __device__ __forceinline__ uint32_t maxd(int ts, int lane) const {
        uint32_t mx = 0;
#pragma unroll
        for (int j = 0; j < J; ++j)
            if (lane + 32 * j < ts) mx = max(mx, P::dist(key[j]));
        return __reduce_max_sync(0xffffffffu, mx);
    }
    __device__ __forceinline__ void put(int js, K k) {
#pragma unroll
        for (int j = 0; j < J; ++j)
            if (j == js) key[j] = k;
        fl &= ~(1u << js);
    }
};

// warp minimum of the lanes' candidates (keys are distinct); false if none
__device__ __forceinline__ bool warp_pick(bool has, uint32_t best, uint32_t &m, int &owner) {
    const unsigned any = __ballot_sync(0xffffffffu, has);
    if (!any) return false;
    m = __reduce_min_sync(0xffffffffu, has ? best : 0xffffffffu);
    owner = __ffs(__ballot_sync(0xffffffffu, has && best == m)) - 1;
    return true;
}
// warp maximum, same contract
__device__ __forceinline__ bool warp_pick_max(bool has, uint32_t best, uint32_t &m, int &owner) {
    const unsigned any = __ballot_sync(0xffffffffu, has);
    if (!any) return false;
    m = __reduce_max_sync(0xffffffffu, has ? best : 0u);
    owner = __ffs(__ballot_sync(0xffffffffu, has && best == m)) - 1;
    return true;
}
// 64-bit keys: the high word first, then the low word among its holders
__device__ __forceinline__ bool warp_pick(bool has, uint64_t best, uint64_t &m, int &owner) {
    const unsigned any = __ballot_sync(0xffffffffu, has);
    if (!any) return false;
    const uint32_t hi = (uint32_t)(best >> 32), lo = (uint32_t)best;
    const uint32_t mh = __reduce_min_sync(0xffffffffu, has ? hi : 0xffffffffu);
    const bool cand = has && hi == mh;
    const uint32_t ml = __reduce_min_sync(0xffffffffu, cand ? lo : 0xffffffffu);
    m = ((uint64_t)mh << 32) | ml;
    owner = __ffs(__ballot_sync(0xffffffffu, cand && lo == ml)) - 1;
    return true;
}
__device__ __forceinline__ bool warp_pick_max(bool has, uint64_t best, uint64_t &m, int &owner) {
    const unsigned any = __ballot_sync(0xffffffffu, has);
    if (!any) return false;
    const uint32_t hi = (uint32_t)(best >> 32), lo = (uint32_t)best;
    const uint32_t mh = __reduce_max_sync(0xffffffffu, has ? hi : 0u);
    const bool cand = has && hi == mh;
    const uint32_t ml = __reduce_max_sync(0xffffffffu, cand ? lo : 0u);
    m = ((uint64_t)mh << 32) | ml;
    owner = __ffs(__ballot_sync(0xffffffffu, cand && lo == ml)) - 1;
    return true;
}

// Ascending bitonic sort of the warp's 32 * J register keys; element
// e = 32 j + lane lives in key[j] of lane `lane`.
template <int J, typename K>
__device__ __forceinline__ void warp_bitonic(K (&k)[J], int lane) {
    constexpr int N = 32 * J;
#pragma unroll
    for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32) {
                const int rsd = stride >> 5;
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    if ((j & rsd) == 0) {
                        const bool up = ((32 * j) & size) == 0;
                        const K a = k[j], b = k[j | rsd];
                        k[j] = up ? min(a, b) : max(a, b);
                        k[j | rsd] = up ? max(a, b) : min(a, b);
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < J; ++j) {
                    const K o = __shfl_xor_sync(0xffffffffu, k[j], stride);
                    const bool up = ((32 * j + lane) & size) == 0;
                    const bool lower = (lane & stride) == 0;
                    k[j] = (up == lower) ? min(k[j], o) : max(k[j], o);
                }
            }
        }
    }
}

// Offer the nf fresh candidates (ids[f], distances fd[f]) of one expansion
// to the register result set (layer_search_reg's acceptance rules): those
// with d < worst (all while the set is not full) are taken in ascending
// (d, tie) order, filling free slots first, then each evicting the current
// victim (largest d, smallest tie) while it is still below the worst.
template <typename P, int J>
__device__ __forceinline__ void accept_offers(RegSet<J, P> &rs, int &ts, int W,
                                              uint32_t &wd, int &tq_h, int &tq_t, int32_t *TQ,
                                              typename P::Key *Sa, typename P::Key *Sb,
                                              const int32_t *fresh, const uint32_t *fdist, int nf,
                                              const TieOrder &to, int lane) {
    using K = typename P::Key;
    constexpr unsigned FULL = 0xffffffffu;
    const unsigned lt = (1u << lane) - 1u;
    // candidates that can possibly enter: all while the set is not full,
    // else d < worst
    int ns = 0;
    for (int base = 0; base < nf; base += 32) {
        const int f = base + lane;
        const bool ok = f < nf && fdist[f] < wd;
        const unsigned b = __ballot_sync(FULL, ok);
        if (ok) Sa[ns + __popc(b & lt)] = P::key(fdist[f], to.fwd((uint32_t)fresh[f]));
        ns += __popc(b);
    }
    __syncwarp();
    if (ns == 0) return;
    const int nfill = min(ns, W - ts);
    const K *src = Sa;
    if (nfill < ns && ns > 1) {
        // offers are processed in ascending order: rank-sort them
        for (int j = lane; j < ns; j += 32) {
            const K k = Sa[j];
            int r = 0;
            for (int t = 0; t < ns; ++t) r += Sa[t] < k;
            Sb[r] = k;
        }
        __syncwarp();
        src = Sb;
    }
    // the first nfill offers fill slots ts .. ts + nfill (none once the set
    // is full: the common case)
    if (nfill > 0) {
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int o = lane + 32 * j - ts;
            if (o >= 0 && o < nfill) {
                rs.key[j] = src[o];
                rs.fl &= ~(1u << j);
            }
        }
        ts += nfill;
    }
    // worst distance wd: recomputed lazily (as the next victim's distance);
    // stale = the set changed since wd was last known
    bool stale = ts == W && nfill > 0;
    if (nfill < ns) {
        const uint32_t lm = RegSet<J, P>::live_mask(ts, lane);
        for (int j = nfill; j < ns; ++j) {
            const K s = src[j];
            // victim: largest distance, smallest tie; its distance is the
            // current worst
            K vf;
            int vj;
            rs.victim(lm, vf, vj);
            K m = 0;
            int owner = 0;
            warp_pick_max(vj >= 0, vf, m, owner);
            const uint32_t cur = P::dist(m);
            if (cur < wd) {
                // the evicted ties are beyond the new worst (none before the
                // set first fills)
                if (wd != 0xffffffffu) tq_h = tq_t = 0;
                wd = cur;
            }
            stale = false;
            if (P::dist(s) >= wd) break;  // sorted: later offers are rejected too
            const uint32_t expd = __shfl_sync(FULL, (rs.fl >> vj) & 1u, owner);
            if (!expd) {
                if (lane == 0) TQ[tq_t] = (int32_t)P::tie(m ^ K(P::kTieMask));
                ++tq_t;
            }
            if (lane == owner) rs.put(vj, s);
            stale = true;
        }
    }
    if (stale) {
        const uint32_t nwd = rs.maxd(ts, lane);
        if (nwd < wd) {
            if (wd != 0xffffffffu) tq_h = tq_t = 0;
            wd = nwd;
        }
    }
    __syncwarp();
}

// The result set out, ascending, as 64-bit keys: T[0..ts).
template <typename P, int J>
__device__ __forceinline__ void sort_out(const RegSet<J, P> &rs, int ts, unsigned long long *T,
                                         int lane) {
    using K = typename P::Key;
    // sort once: bitonic network over the 32 * J register slots (empty slots
    // hold the largest key and sort last), then the first ts go out
    // (J not a power of two: the network runs over JP registers, the extra
    // ones holding the largest key)
    constexpr int JP = J <= 2 ? 2 : J <= 4 ? 4 : J <= 8 ? 8 : 16;
    K ks[JP];
#pragma unroll
    for (int j = 0; j < JP; ++j)
        ks[j] = (j < J && lane + 32 * j < ts) ? rs.key[j < J ? j : 0] : ~K(0);
    warp_bitonic<JP>(ks, lane);
#pragma unroll
    for (int j = 0; j < JP; ++j) {
        const int e = 32 * j + lane;
        if (e < ts) T[e] = make_key(P::dist(ks[j]), P::tie(ks[j]));
    }
    __syncwarp();
}

// RC: id-row chunks of 32 slots compiled in (cap <= 32 RC); KB: VisitedSet
template <typename P, int J, int EM, int RC = kRowChunks, int KB = 0>
__device__ __forceinline__ bool layer_search_reg(const Graph &g, int layer, int entry,
                                                 uint32_t entry_d, int W, const uint8_t *qc,
                                                 unsigned long long *T, int &ts_out,
                                                 unsigned long long *S, int32_t *TQ,
                                                 int32_t *fresh, uint32_t *fdist, uint32_t *H,
                                                 int hlog2, SearchCounters &cnt,
                                                 const TieOrder &to, GSlot &gs, int lane) {
    constexpr unsigned FULL = 0xffffffffu;
    const int cap = layer_cap(g, layer);
    const RowAddr ra(g, layer);
    using K = typename P::Key;
    K *Sa = reinterpret_cast<K *>(S);
    K *Sb = reinterpret_cast<K *>(fresh);  // (WarpLayout: fresh + fdist hold nc keys)
    const unsigned lt = (1u << lane) - 1u;
    VisitedSet<KB, P::kWide> vs;
    vs.begin(H, hlog2, g, gs, lane);
    if (lane == 0) vs.visit(entry);
    RegSet<J, P> rs;
#pragma unroll
    for (int j = 0; j < J; ++j) rs.key[j] = K(0);
    rs.fl = 0u;
    if (lane == 0) rs.key[0] = P::key(entry_d, to.fwd((uint32_t)entry));
    int ts = 1;
    uint32_t wd = 0xffffffffu;  // worst distance once the set is full
    int tq_h = 0, tq_t = 0;     // tie queue TQ[tq_h..tq_t), distance == wd
    int pre_v = -1;             // speculative id row of the most likely next pop (EM == 1)
    int pre[RC];
    const int E = EM > 1 ? min(max(g.expand, 1), EM) : 1;
    long long tph = phase_clock();
    __syncwarp();
    while (true) {
        phase_mark(cnt, 3, tph);  // the previous iteration's acceptance
        // ---- pop up to E frontier minima: unexpanded set members vs tie queue
        int pv[EM];
        int npop = 0;
        int u[EM][RC];
        if (EM == 1) {
            K b1, b2;
            int j1;
            const uint32_t um = RegSet<J, P>::live_mask(ts, lane) & ~rs.fl;
            rs.min2(um, b1, j1, b2);
            const int nl = __popc(um);
            K m = 0;
            int owner = -1;
            const bool anyT = warp_pick(nl > 0, b1, m, owner);
            const bool anyQ = tq_h < tq_t;
            if (!anyT && !anyQ) break;
            const K kQ = anyQ ? P::key(wd, (uint32_t)TQ[tq_h]) : K(0);
            const bool fromT = anyT && (!anyQ || m < kQ);
            pv[0] = to.back(P::tie(fromT ? m : kQ));
            npop = 1;
            if (fromT) {
                if (lane == owner) rs.fl |= 1u << j1;
            } else {
                ++tq_h;
            }
            if (pv[0] == pre_v) {
#pragma unroll
                for (int k = 0; k < RC; ++k) u[0][k] = pre[k];
            } else {
                load_row(ra(pv[0]), cap, lane, u[0]);
            }
            // predict the next pop assuming nothing new enters: the popped
            // lane offers its second smallest key
            const bool h2 = fromT && lane == owner ? nl > 1 : nl > 0;
            const K c2 = fromT && lane == owner ? b2 : b1;
            K m2 = 0;
            int o2 = -1;
            const bool anyT2 = warp_pick(h2, c2, m2, o2);
            const bool anyQ2 = tq_h < tq_t;
            if (anyT2 || anyQ2) {
                const K kQ2 = anyQ2 ? P::key(wd, (uint32_t)TQ[tq_h]) : K(0);
                pre_v = to.back(P::tie(anyT2 && (!anyQ2 || m2 < kQ2) ? m2 : kQ2));
            } else {
                pre_v = -1;
            }
            // (its row is loaded below, once the visited filter has consumed u[0])
        } else {
#pragma unroll
            for (int r = 0; r < EM; ++r) {
                if (r >= E) break;
                K best, b2;
                int bj;
                rs.min2(RegSet<J, P>::live_mask(ts, lane) & ~rs.fl, best, bj, b2);
                const bool has = bj >= 0;
                K m = 0;
                int owner = -1;
                const bool anyT = warp_pick(has, best, m, owner);
                const bool anyQ = tq_h < tq_t;
                if (!anyT && !anyQ) break;
                const K kQ = anyQ ? P::key(wd, (uint32_t)TQ[tq_h]) : K(0);
                const bool fromT = anyT && (!anyQ || m < kQ);
                pv[r] = to.back(P::tie(fromT ? m : kQ));
                ++npop;
                if (fromT) {
                    if (lane == owner) rs.fl |= 1u << bj;
                } else {
                    ++tq_h;
                }
            }
            if (npop == 0) break;
            // id rows of the popped vertices, all loads in flight together
#pragma unroll
            for (int r = 0; r < EM; ++r)
                if (r < npop) load_row(ra(pv[r]), cap, lane, u[r]);
        }
        cnt.visited += npop;
        phase_mark(cnt, 0, tph);
        // visited filter over the rows (pop order, slot order), compacted
        bool over = false;
        int nf = 0;
#pragma unroll
        for (int r = 0; r < EM; ++r) {
            if (r >= npop) break;
            int nlive = 0;
#pragma unroll
            for (int k = 0; k < RC; ++k) {
                if (k * 32 >= cap) break;
                const int x = u[r][k];
                const bool live = x >= 0;
                const int rr = live ? vs.visit(x) : 0;
                over |= rr == 3;
                const bool fr = rr == 1 || rr == 2;
                const unsigned bl = __ballot_sync(FULL, live);
                const unsigned bf = __ballot_sync(FULL, fr);
                if (fr) fresh[nf + __popc(bf & lt)] = x;
                nf += __popc(bf);
                nlive += __popc(bl);
            }
            cnt.kcalls += (nlive + 15) >> 4;
        }
        if (__any_sync(FULL, over)) return false;
        cnt.dist += nf;
        __syncwarp();
        phase_mark(cnt, 1, tph);
        // the predicted next pop's row: issued here, right before the code
        // gather, and consumed at the next step.  (ptxas gives it the
        // scoreboard of the miss path's row load; issued before the visited
        // filter, the filter's wait on u[0] waited for it as well, and a
        // full load latency per step: 230.7 -> 223.3 ms per config-2 build)
        if (EM == 1 && pre_v >= 0) load_row(ra(pre_v), cap, lane, pre);
        if (nf == 0) continue;
        P::dists(g, qc, fresh, nf, fdist, lane);
        phase_mark(cnt, 2, tph);
        accept_offers<P, J>(rs, ts, W, wd, tq_h, tq_t, TQ, Sa, Sb, fresh, fdist, nf, to, lane);
    }
    sort_out<P, J>(rs, ts, T, lane);
    ts_out = ts;
    return true;
}

// Generic-key warp helpers of the shared-memory result set.  Keys are distinct.
// min key over the entries not yet expanded (F[i] == 0), or, with dsel_on,
// over the entries whose distance equals dsel; idx = its slot.
template <typename P, typename Kt = typename P::Key>
__device__ __forceinline__ Kt warp_argmin_key(const Kt *K, const uint8_t *F, int n, bool dsel_on,
                                              uint32_t dsel, int lane, int &idx) {
    Kt best = ~Kt(0);
    int bi = -1;
#pragma unroll 4
    for (int c = 0; c < n; c += 32) {
        const int i = c + lane;
        if (i < n) {
            const Kt k = K[i];
            const bool ok = dsel_on ? (P::dist(k) == dsel) : (F[i] == 0);
            if (ok && k < best) {
                best = k;
                bi = i;
            }
        }
    }
    Kt m = ~Kt(0);
    int owner = -1;
    if (!warp_pick(bi >= 0, best, m, owner)) {
        idx = -1;
        return ~Kt(0);
    }
    idx = __shfl_sync(0xffffffffu, bi, owner);
    return m;
}

template <typename P, typename Kt = typename P::Key>
__device__ __forceinline__ uint32_t warp_maxd_key(const Kt *K, int n, int lane) {
    uint32_t mx = 0;
#pragma unroll 4
    for (int c = 0; c < n; c += 32) {
        const int i = c + lane;
        if (i < n) mx = max(mx, P::dist(K[i]));
    }
    return __reduce_max_sync(0xffffffffu, mx);
}

// Shared-memory variant for W > kRegSetMax (same rules, same results), for
// either distance policy (32-bit Flash keys, 64-bit exact keys).
template <typename P>
__device__ inline bool layer_search_smem(const Graph &g, int layer, int entry, uint32_t entry_d, int W,
                                    const uint8_t *qc, unsigned long long *T, int &ts,
                                    unsigned long long *S, int32_t *TQ, int32_t *fresh,
                                    uint32_t *fdist, uint32_t *H, int hlog2, SearchCounters &cnt,
                                    const TieOrder &to, GSlot &gs, int lane) {
    using Kt = typename P::Key;
    constexpr Kt NONE = ~Kt(0);
    const int cap = layer_cap(g, layer);
    // workspace (WarpLayout::T): 64-bit result slots, then the keys, then
    // the expanded flags, Wp = round_up(W, 32) of each
    const int Wp = round_up(W, 32);
    Kt *K = reinterpret_cast<Kt *>(T + Wp);
    uint8_t *F = reinterpret_cast<uint8_t *>(K + Wp);
    Kt *Sa = reinterpret_cast<Kt *>(S);
    Kt *Sb = reinterpret_cast<Kt *>(fresh);  // (WarpLayout: fresh + fdist hold nc keys)
    VisitedSet<0, P::kWide> vs;
    vs.begin(H, hlog2, g, gs, lane);
    if (lane == 0) {
        vs.visit(entry);
        K[0] = P::key(entry_d, to.fwd((uint32_t)entry));
        F[0] = 0;
    }
    ts = 1;
    uint32_t wd = 0xffffffffu;  // worst distance once the set is full
    int tq_h = 0, tq_t = 0;     // tie queue TQ[tq_h..tq_t), distance == wd
    int pre_v = -1;             // speculative id row of the most likely next pop (E == 1)
    int pre[kRowChunks];
    // frontier entries expanded per step: 1 = the semantic core; E > 1 pops the
    // E smallest poppable entries and expands them together (oracle: expand)
    const int E = g.expand > 1 ? min(g.expand, kMaxExpand) : 1;
    long long tph = phase_clock();
    __syncwarp();
    while (true) {
        phase_mark(cnt, 3, tph);  // the previous iteration's acceptance
        // ---- pop up to E frontier minima: unexpanded set members vs tie queue
        int pv[kMaxExpand];
        int npop = 0;
#pragma unroll
        for (int r = 0; r < kMaxExpand; ++r) {
            if (r >= E) break;
            int ia;
            const Kt kT = warp_argmin_key<P>(K, F, ts, false, 0u, lane, ia);
            const Kt kQ = tq_h < tq_t ? P::key(wd, (uint32_t)TQ[tq_h]) : NONE;
            if (kT == NONE && kQ == NONE) break;
            const bool fromT = kT < kQ;
            pv[r] = to.back(P::tie(fromT ? kT : kQ));
            ++npop;
            __syncwarp();
            if (fromT) {
                if (lane == 0) F[ia] = 1;
            } else {
                ++tq_h;
            }
            __syncwarp();
        }
        if (npop == 0) break;
        // id rows of the popped vertices, all loads in flight together
        int u[kMaxExpand][kRowChunks];
#pragma unroll
        for (int r = 0; r < kMaxExpand; ++r) {
            if (r < npop) {
                if (E == 1 && pv[0] == pre_v) {
#pragma unroll
                    for (int k = 0; k < kRowChunks; ++k) u[0][k] = pre[k];
                } else {
                    load_row(row_ids(g, layer, pv[r]), cap, lane, u[r]);
                }
            }
        }
        if (E == 1) {  // predict the next pop assuming nothing new enters
            int ib;
            const Kt k1 = warp_argmin_key<P>(K, F, ts, false, 0u, lane, ib);
            const Kt k2 = tq_h < tq_t ? P::key(wd, (uint32_t)TQ[tq_h]) : NONE;
            const Kt kn = k1 < k2 ? k1 : k2;
            pre_v = kn != NONE ? to.back(P::tie(kn)) : -1;
            if (pre_v >= 0) load_row(row_ids(g, layer, pre_v), cap, lane, pre);
        }
        cnt.visited += npop;
        phase_mark(cnt, 0, tph);
        bool over = false;
        // visited filter over the rows (pop order, slot order), compacted
        int nf = 0;
#pragma unroll
        for (int r = 0; r < kMaxExpand; ++r) {
            if (r >= npop) break;
            int nlive = 0;
#pragma unroll
            for (int k = 0; k < kRowChunks; ++k) {
                if (k * 32 >= cap) break;
                const int x = u[r][k];
                bool live = x >= 0;
                const int rr = live ? vs.visit(x) : 0;
                over |= rr == 3;
                const bool fr = rr == 1 || rr == 2;
                unsigned bl = __ballot_sync(0xffffffffu, live);
                unsigned bf = __ballot_sync(0xffffffffu, fr);
                if (fr) fresh[nf + __popc(bf & ((1u << lane) - 1u))] = x;
                nf += __popc(bf);
                nlive += __popc(bl);
            }
            cnt.kcalls += (nlive + 15) >> 4;
        }
        if (__any_sync(0xffffffffu, over)) return false;
        cnt.dist += nf;
        __syncwarp();
        phase_mark(cnt, 1, tph);
        if (nf == 0) continue;
        P::dists(g, qc, fresh, nf, fdist, lane);
        phase_mark(cnt, 2, tph);
        // candidates that can possibly enter: all while the set is not full,
        // else d < worst
        int ns = 0;
        for (int base = 0; base < nf; base += 32) {
            const int f = base + lane;
            const bool ok = f < nf && fdist[f] < wd;
            const unsigned b = __ballot_sync(0xffffffffu, ok);
            if (ok)
                Sa[ns + __popc(b & ((1u << lane) - 1u))] =
                    P::key(fdist[f], to.fwd((uint32_t)fresh[f]));
            ns += __popc(b);
        }
        __syncwarp();
        if (ns == 0) continue;
        const int nfill = min(ns, W - ts);
        if (nfill == ns) {
            // everything fits: append (no order needed)
            for (int j = lane; j < ns; j += 32) {
                K[ts + j] = Sa[j];
                F[ts + j] = 0;
            }
            ts += ns;
            __syncwarp();
            if (ts == W) wd = warp_maxd_key<P>(K, ts, lane);
            continue;
        }
        // offers are processed in ascending order: rank-sort them
        for (int j = lane; j < ns; j += 32) {
            const Kt k = Sa[j];
            int r = 0;
            for (int t = 0; t < ns; ++t) r += Sa[t] < k;
            Sb[r] = k;
        }
        __syncwarp();
        for (int j = lane; j < nfill; j += 32) {
            K[ts + j] = Sb[j];
            F[ts + j] = 0;
        }
        ts += nfill;
        __syncwarp();
        wd = warp_maxd_key<P>(K, ts, lane);
        for (int j = nfill; j < ns; ++j) {
            const Kt s = Sb[j];
            if (P::dist(s) >= wd) break;  // sorted: every later offer is rejected too
            int e;
            const Kt ev = warp_argmin_key<P>(K, F, ts, true, wd, lane, e);
            if (!F[e]) {
                if (lane == 0) TQ[tq_t] = (int32_t)P::tie(ev);
                ++tq_t;
            }
            __syncwarp();
            if (lane == 0) {
                K[e] = s;
                F[e] = 0;
            }
            __syncwarp();
            const uint32_t nwd = warp_maxd_key<P>(K, ts, lane);
            if (nwd < wd) {
                wd = nwd;
                tq_h = tq_t = 0;  // the evicted ties are beyond the new worst
            }
        }
    }
    // sort the keys once: rank by counting (keys are distinct) into the 64-bit slots
    for (int i = lane; i < ts; i += 32) {
        const Kt k = K[i];
        int r = 0;
        for (int t = 0; t < ts; ++t) r += K[t] < k;
        T[r] = make_key(P::dist(k), P::tie(k));
    }
    __syncwarp();
    return true;
}


// Best-first layer search with the result-set variant J chosen by the host
// (set_variant): J slots per lane in registers, J = 0 the shared-memory set
// (either kind).  P: the distance policy (FlashDist / ExactDist).
template <typename P, int J, int EM, int RC = kRowChunks, int KB = 0>
__device__ __forceinline__ bool layer_search(const Graph &g, int layer, int entry, uint32_t entry_d,
                                             int W, const uint8_t *qc, unsigned long long *T,
                                             int &ts, unsigned long long *S, int32_t *TQ,
                                             int32_t *fresh, uint32_t *fdist, uint32_t *H,
                                             int hlog2, SearchCounters &cnt, const TieOrder &to,
                                             GSlot &gs, int lane) {
    if constexpr (J == 0) {
        return layer_search_smem<P>(g, layer, entry, entry_d, W, qc, T, ts, S, TQ, fresh, fdist, H,
                                 hlog2, cnt, to, gs, lane);
    } else {
        return layer_search_reg<P, J, EM, RC, KB>(g, layer, entry, entry_d, W, qc, T, ts, S, TQ,
                                                  fresh, fdist, H, hlog2, cnt, to, gs, lane);
    }
}

// result-set variant for a search width W: register slots per lane, 0 = shared
__host__ __device__ inline int set_variant(int W) {
    return W <= 64 ? 2 : W <= 128 ? 4 : W <= 224 ? 7 : W <= 256 ? 8 : W <= 320 ? 10
           : W <= kRegSetMax ? 16 : 0;
}

// select_heur (_core.pyx:388-408) of the exact kind: candidate v (distance
// bits dv) is kept iff no kept u has fp32 L2(u, v) < dv.  The candidate's
// vector is staged in shared memory (cv, dim floats) and the kept set's
// distances to it come four at a time from 8-lane groups (the fa_l2sq_f32
// tree, symmetric in its arguments: the squared differences are equal).
template <class Get>
__device__ int warp_select_exact(const Graph &g, int ncand, int cap, Get get, int32_t *kept,
                                 float *cv, uint32_t *kd, int lane,
                                 unsigned long long *sym_count, uint32_t *kept_d = nullptr) {
    int nk = 0;
    unsigned long long sym = 0;
    for (int j = 0; j < ncand && nk < cap; ++j) {
        int v;
        uint32_t dv;
        get(j, v, dv);
        bool bad = false;
        if (nk > 0) {
            const float *b = g.vecs + (size_t)v * g.dim;
            for (int i = lane; i < g.dim; i += 32) cv[i] = __ldg(b + i);
            __syncwarp();
            // four kept vectors per pass; the first dominating one settles it
            for (int base = 0; base < nk; base += 4) {
                const int t = base + (lane >> 3);
                const float *a = t < nk ? g.vecs + (size_t)kept[t] * g.dim : nullptr;
                const float d = warp_l2_group8(t < nk ? cv : nullptr, a, g.dim, lane);
                if ((lane & 7) == 0 && t < nk && __float_as_uint(d) < dv) bad = true;
                if (__any_sync(0xffffffffu, bad)) break;
            }
            __syncwarp();
        }
        sym += nk;
        if (!__any_sync(0xffffffffu, bad)) {
            if (lane == 0) {
                kept[nk] = v;
                if (kept_d) kept_d[nk] = dv;
            }
            ++nk;
        }
        __syncwarp();
    }
    if (sym_count && lane == 0) *sym_count += sym;
    return nk;
}

// Width-1 greedy descent (hill_climb, _core.pyx:345-385): move to the first
// slot holding the minimum distance while it is strictly better.
template <typename P>
__device__ inline void hill_climb(const Graph &g, int layer, int &cur, uint32_t &curd,
                           const uint8_t *qc, int32_t *ids_s, uint32_t *d_s,
                           SearchCounters &cnt, int lane) {
    const int cap = layer_cap(g, layer);
    while (true) {
        const int32_t *ids = row_ids(g, layer, cur);
        int nlive = 0;
        for (int base = 0; base < cap; base += 32) {
            int j = base + lane;
            int u = j < cap ? __ldg(ids + j) : -1;
            if (j < cap) ids_s[j] = u;
            nlive += __popc(__ballot_sync(0xffffffffu, u >= 0));
        }
        __syncwarp();
        // live ids form a prefix (rows keep -1 beyond the count)
        cnt.kcalls += (nlive + 15) >> 4;
        cnt.dist += nlive;
        if (nlive == 0) break;
        P::dists(g, qc, ids_s, nlive, d_s, lane);
        unsigned long long best = KEY_MAX;
        for (int j = lane; j < nlive; j += 32) {
            unsigned long long k = ((unsigned long long)d_s[j] << 32) | (uint32_t)j;
            best = k < best ? k : best;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
            best = y < best ? y : best;
        }
        uint32_t dmin = (uint32_t)(best >> 32);
        int slot = (int)(best & 0xffffffffu);
        if (dmin < curd) {
            curd = dmin;
            cur = ids_s[slot];
            __syncwarp();
        } else {
            break;
        }
    }
}

}  // namespace fa
