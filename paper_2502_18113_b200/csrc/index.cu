// Device graph runtime: allocation, the batched-insertion build loop,
// query search, and reference-layout import/export.
//
// Build = reference build_graph (_core.pyx:711-764) with the OpenMP prange
// replaced by deterministic insertion batches: every vertex of a batch
// searches the graph as of the batch start (one warp each), then all reverse
// edges of the batch are grouped by target row and applied in ascending x.
// The batch schedule is a pure function of the layer draws, so the whole
// build is enqueued without a host round trip.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <vector>

#include "kernels.cuh"

struct fa_index {
    fa::Graph g;
    fa_index_desc d;
    int cap0, capU;
    std::vector<int32_t> levels_h;
    std::vector<int64_t> uoff_h;
    // derived once from levels_h (immutable): the record positions (a level
    // above every earlier one: a new top layer) and the largest level
    bool sched_ready = false;
    std::vector<int64_t> raisers;
    // host drop-in: projected rows >= late_from arrive while the build runs;
    // late_hook (wait for them, encode them) runs before the first batch
    // that needs them is enqueued
    int64_t late_from = -1;
    std::function<int(cudaStream_t)> late_hook;
    uint8_t *codes = nullptr;
    int32_t *adj0 = nullptr, *cnt0 = nullptr, *adjU = nullptr, *cntU = nullptr;
    uint8_t *cons0 = nullptr, *consU = nullptr;
    uint8_t *dist0 = nullptr, *distU = nullptr;  // prune-distance caches
    int32_t *upper_owner = nullptr;
    uint32_t *gvis = nullptr, *gvis_epoch = nullptr, *gvis_owner = nullptr;  // global visited tier
    int search_tie = 0;
    bool wide = false;       // 32-bit-id kernels (n >= 2^24 - 1, or forced)
    int64_t n_inserted = 0;  // vertices [0, n_inserted) are in the graph
    int64_t entry = -1;
    int max_layer = -1;
    int maxlv = 0;  // the largest level (with raisers)
};

namespace fa {

static int dev_alloc(void **p, size_t bytes) { return pool_alloc(p, bytes); }

// The build's per-batch processing order and request offsets go up from
// process-wide pinned buffers (grown on demand, never freed: pinning and
// unpinning cost more than the buffers).  Builds are serialised on them.
static std::mutex g_order_mu;
static int32_t *g_order_h = nullptr;
static int64_t *g_reqoff_h = nullptr;
static int64_t g_order_cap = 0;
static int pinned_order(int64_t n, int32_t **order, int64_t **reqoff) {
    if (n > g_order_cap) {
        if (g_order_h) cudaFreeHost(g_order_h);
        if (g_reqoff_h) cudaFreeHost(g_reqoff_h);
        g_order_h = nullptr;
        g_reqoff_h = nullptr;
        g_order_cap = 0;
        cudaError_t e = cudaHostAlloc((void **)&g_order_h, sizeof(int32_t) * (size_t)n,
                                      cudaHostAllocDefault);
        if (e == cudaSuccess)
            e = cudaHostAlloc((void **)&g_reqoff_h, sizeof(int64_t) * (size_t)n,
                              cudaHostAllocDefault);
        if (e != cudaSuccess) {
            set_error("cudaHostAlloc(build order): %s", cudaGetErrorString(e));
            return FA_ENOMEM;
        }
        g_order_cap = n;
    }
    *order = g_order_h;
    *reqoff = g_reqoff_h;
    return FA_OK;
}

__global__ void fill_i32(int32_t *p, int64_t n, int32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

static int reset_graph(fa_index *ix, cudaStream_t st) {
    Graph &g = ix->g;
    fill_i32<<<1184, 256, 0, st>>>(g.adj0, g.n * g.cap0p, -1);
    if (g.nU) fill_i32<<<1184, 256, 0, st>>>(g.adjU, g.nU * g.capUp, -1);
    FA_LAUNCH_CHECK();
    FA_CUDA(cudaMemsetAsync(g.cnt0, 0, sizeof(int32_t) * g.n, st));
    FA_CUDA(cudaMemsetAsync(g.cons0, 0, g.n, st));
    if (g.nU) {
        FA_CUDA(cudaMemsetAsync(g.cntU, 0, sizeof(int32_t) * g.nU, st));
        FA_CUDA(cudaMemsetAsync(g.consU, 0, g.nU, st));
    }
    return FA_OK;
}

// Global visited tier (VisitedSet): a pool of tables claimed per search.  The
// pool holds one slot per warp the launch can keep resident (occupancy x SMs)
// and each table 2^gvis_log2_for(W) entries; it grows on demand (reallocated
// only when a launch needs more slots or a wider table).  Wide indexes (32-bit
// ids) use 64-bit entries.
// Warps per CTA of a search launch: kSearchWarps, fewer when the per-warp
// workspace (wide searches) does not fit; 0 if one warp does not fit.
static int search_warps_for(int per_warp_bytes, int wmax = kSearchWarps) {
    int w = wmax;
    while (w > 0 && (size_t)w * per_warp_bytes > 227 * 1024) --w;
    return w;
}

static int ensure_gvis(fa_index *ix, const void *kernel, int threads, size_t smem, int W,
                       cudaStream_t st) {
    int dev = 0, nsm = 0, per_sm = 0;
    FA_CUDA(cudaGetDevice(&dev));
    FA_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    FA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
    const int slots = std::max(1, nsm * std::max(per_sm, 1) * (threads / 32));
    const int capmax = std::max(ix->g.cap0, ix->g.capU);
    const int l2 = gvis_log2_for(W, capmax, ix->g.n);
    if (ix->gvis && slots <= ix->g.gvis_nslots && l2 <= ix->g.gvis_log2) return FA_OK;
    // grow to cover both this launch and earlier ones
    const int ns = std::max(slots, ix->gvis ? ix->g.gvis_nslots : 0);
    const int lg = std::max(l2, ix->gvis ? ix->g.gvis_log2 : 0);
    if (ix->gvis) FA_CUDA(cudaDeviceSynchronize());  // no search may still hold the old pool
    pool_free(ix->gvis);
    pool_free(ix->gvis_epoch);
    pool_free(ix->gvis_owner);
    ix->gvis = ix->gvis_epoch = ix->gvis_owner = nullptr;
    ix->g.gvis = ix->g.gvis_epoch = ix->g.gvis_owner = nullptr;
    // entries: 32-bit (epoch << 24 | id) or, wide, 64-bit (epoch << 32 | id)
    const size_t tab = ((size_t)ns << lg) * (ix->wide ? 8 : 4);
    FA_TRY(dev_alloc((void **)&ix->gvis, tab));
    FA_TRY(dev_alloc((void **)&ix->gvis_epoch, (size_t)ns * sizeof(uint32_t)));
    FA_TRY(dev_alloc((void **)&ix->gvis_owner, (size_t)ns * sizeof(uint32_t)));
    // on the launch's stream: ordered before the searches that use it
    FA_CUDA(cudaMemsetAsync(ix->gvis, 0, tab, st));
    FA_CUDA(cudaMemsetAsync(ix->gvis_epoch, 0, (size_t)ns * sizeof(uint32_t), st));
    FA_CUDA(cudaMemsetAsync(ix->gvis_owner, 0, (size_t)ns * sizeof(uint32_t), st));
    ix->g.gvis = ix->gvis;
    ix->g.gvis_epoch = ix->gvis_epoch;
    ix->g.gvis_owner = ix->gvis_owner;
    ix->g.gvis_nslots = ns;
    ix->g.gvis_log2 = lg;
    ix->g.gvis_words = ix->wide ? 2 : 1;
    return FA_OK;
}

// log2 of the shared visited table's 16-bit slots (search.cuh VisitedSet);
// the table also hosts the kept ids + codes of forward selection and the
// rerank distances (alias_bytes).
static int pick_hash_log2(int W, int capmax, int R, int mpad, int req, size_t alias_bytes = 0) {
    int l;
    if (req > 0) {
        l = std::max(req, 9);
    } else {
        const int want = 16 * W + 2 * capmax;  // the global tier absorbs longer searches
        l = 12;
        while ((1 << l) < want && l < 13) ++l;
    }
    const size_t need =
        std::max(alias_bytes, (size_t)round_up(R * 4, 16) + (size_t)R * kept_stride(mpad));
    while (((size_t)16 << vis_buckets_log2(l)) < need) ++l;
    return l;
}

// Export rows to the reference block layout (layout.py:1-45): count, ids
// (-1 beyond count), subspace-major 16-slot code batches (0 beyond count).
// One warp per row: the live neighbours' code rows are staged in shared
// memory (row stride mpad + 4: the 16 lanes of one output chunk read 16
// different banks), then every 16-byte chunk (batch bt, subspace i) = the
// i-th code byte of slots bt*16 .. bt*16+15 is packed into four words.
constexpr int kExportWarps = 8;
__global__ void __launch_bounds__(kExportWarps * 32) export_kernel(
    Graph g, int64_t rows, bool upper, uint8_t *__restrict__ blocks, int64_t stride, int cap,
    int capp) {
    extern __shared__ __align__(16) uint8_t xs[];
    const int lane = lane_id();
    const int wid = threadIdx.x >> 5;
    const int cs = g.mpad + 4;  // staged row stride
    const int nb = (cap + 15) >> 4;
    uint8_t *st = xs + (size_t)wid * nb * 16 * cs;
    const int64_t warps = (int64_t)gridDim.x * kExportWarps;
    const int q16 = g.mpad >> 4;  // 16-byte words per code row
    for (int64_t r = (int64_t)blockIdx.x * kExportWarps + wid; r < rows; r += warps) {
        const int32_t *ids = (upper ? g.adjU : g.adj0) + r * capp;
        const int cnt = (upper ? g.cntU : g.cnt0)[r];
        uint8_t *b = blocks + r * stride;
        if (lane == 0) *reinterpret_cast<int32_t *>(b) = cnt;
        int32_t *bid = reinterpret_cast<int32_t *>(b + 4);
        for (int j = lane; j < cap; j += 32) bid[j] = j < cnt ? ids[j] : -1;
        // stage: slot j's code row (zeros past the count or for a -1 id)
        for (int t = lane; t < nb * 16 * q16; t += 32) {
            const int j = t / q16, w = t - j * q16;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (j < cnt) {
                const int u = ids[j];
                if (u >= 0)
                    v = __ldg(reinterpret_cast<const uint4 *>(g.codes + (size_t)u * g.mpad) + w);
            }
            uint32_t *d = reinterpret_cast<uint32_t *>(st + j * cs + w * 16);
            d[0] = v.x;
            d[1] = v.y;
            d[2] = v.z;
            d[3] = v.w;
        }
        __syncwarp();
        // the reference's rows are 4 (mod 16) bytes long: 4-byte stores
        uint32_t *region = reinterpret_cast<uint32_t *>(b + 4 + 4 * cap);
        for (int t = lane; t < nb * g.m; t += 32) {
            const int bt = t / g.m, i = t - bt * g.m;
            const uint8_t *c = st + (bt * 16) * cs + i;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t b0 = c[(4 * k + 0) * cs], b1 = c[(4 * k + 1) * cs];
                const uint32_t b2 = c[(4 * k + 2) * cs], b3 = c[(4 * k + 3) * cs];
                region[4 * t + k] = b0 | (b1 << 8) | (b2 << 16) | (b3 << 24);
            }
        }
        __syncwarp();
    }
}

static int launch_export(const Graph &g, int64_t rows, bool upper, uint8_t *blocks, int64_t stride,
                         int cap, int capp, cudaStream_t st) {
    const size_t smem = (size_t)kExportWarps * round_up(cap, 16) * (g.mpad + 4);
    if (smem > 48 * 1024)
        FA_CUDA(cudaFuncSetAttribute(export_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    const int grid = (int)std::min<int64_t>((rows + kExportWarps - 1) / kExportWarps,
                                            (int64_t)num_sms() * 8);
    export_kernel<<<std::max(grid, 1), kExportWarps * 32, smem, st>>>(g, rows, upper, blocks,
                                                                      stride, cap, capp);
    FA_LAUNCH_CHECK();
    return FA_OK;
}

__global__ void import_kernel(Graph g, int64_t rows, bool upper, const uint8_t *__restrict__ blocks,
                              int64_t stride, int cap, int capp) {
    const int lane = lane_id();
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < rows;
         r += warps) {
        const uint8_t *b = blocks + r * stride;
        int cnt = *reinterpret_cast<const int32_t *>(b);
        cnt = cnt < 0 ? 0 : (cnt > cap ? cap : cnt);
        const int32_t *bid = reinterpret_cast<const int32_t *>(b + 4);
        int32_t *ids = (upper ? g.adjU : g.adj0) + r * capp;
        // live ids are compacted to a prefix (-1 slots inside the count are
        // skipped by every reader of the reference layout, _core.pyx:308-311)
        int w = 0;
        for (int base = 0; base < cnt; base += 32) {
            int j = base + lane;
            int u = j < cnt ? bid[j] : -1;
            unsigned bl = __ballot_sync(0xffffffffu, u >= 0);
            if (u >= 0) ids[w + __popc(bl & ((1u << lane) - 1u))] = u;
            w += __popc(bl);
        }
        for (int j = w + lane; j < capp; j += 32) ids[j] = -1;
        if (lane == 0) {
            (upper ? g.cntU : g.cnt0)[r] = w;
            (upper ? g.consU : g.cons0)[r] = 0;
        }
    }
}

struct Batch {
    int start, size, ep, ml;
    int64_t nreq;
    bool raiser;  // a vertex that opens a new top layer, inserted alone
};

}  // namespace fa

using namespace fa;

extern "C" int fa_index_create(const fa_index_desc *desc, fa_index **out) {
    FA_CHECK_ARG(desc && out, "null argument");
    // n < 2^24 - 1: 24-bit tie ids in 32-bit search keys; above, the wide
    // kernels (32-bit ids, 64-bit keys).  Ids are int32.
    FA_CHECK_ARG(desc->n >= 0 && desc->n < (1ll << 31) - 1, "n=%lld out of range [0, 2^31 - 1)",
                 (long long)desc->n);
    // m = 0: the exact strategy (kind 0, code_subspaces = 0): fp32 L2 over vecs
    FA_CHECK_ARG(desc->m >= 0 && desc->m <= 128, "m=%d outside [0,128]", desc->m);
    FA_CHECK_ARG(desc->m > 0 || (desc->vecs && desc->dim >= 1),
                 "the exact kind (m = 0) needs the vectors");
    FA_CHECK_ARG(desc->R >= 1, "R must be >= 1");
    FA_CHECK_ARG(2 * desc->R <= 127, "base capacity 2R=%d exceeds 127", 2 * desc->R);
    fa_index *ix = new fa_index();
    ix->d = *desc;
    ix->wide = desc->n >= (1ll << 24) - 1;
    if (const char *e = getenv("FLASHANN_B200_WIDE")) ix->wide = ix->wide || atoi(e) > 0;
    Graph &g = ix->g;
    g.n = desc->n;
    g.m = desc->m;
    g.mpad = round_up(desc->m, 16);
    g.cap0 = 2 * desc->R;
    g.capU = desc->R;
    g.cap0p = round_up(g.cap0, 32);
    g.capUp = round_up(g.capU, 32);
    g.nU = desc->n_upper_rows;
    g.levels = desc->levels;
    g.uoff = desc->uoff;
    g.vecs = desc->vecs;
    g.dim = desc->dim;
    int rc = FA_OK;
    auto fail = [&](int r) {
        fa_index_destroy(ix);
        return r;
    };
    if ((rc = dev_alloc((void **)&ix->codes, (size_t)g.n * g.mpad))) return fail(rc);
    if ((rc = dev_alloc((void **)&ix->adj0, sizeof(int32_t) * g.n * g.cap0p))) return fail(rc);
    if ((rc = dev_alloc((void **)&ix->cnt0, sizeof(int32_t) * g.n))) return fail(rc);
    if ((rc = dev_alloc((void **)&ix->cons0, g.n))) return fail(rc);
    if ((rc = dev_alloc((void **)&ix->adjU, sizeof(int32_t) * g.nU * g.capUp))) return fail(rc);
    if ((rc = dev_alloc((void **)&ix->cntU, sizeof(int32_t) * g.nU))) return fail(rc);
    if ((rc = dev_alloc((void **)&ix->consU, g.nU))) return fail(rc);
    // prune-distance caches: u8 per slot (Flash), fp32 bits per slot (exact)
    const size_t dbytes = desc->m == 0 ? 4 : 1;
    if ((rc = dev_alloc((void **)&ix->dist0, (size_t)g.n * g.cap0p * dbytes))) return fail(rc);
    if ((rc = dev_alloc((void **)&ix->distU, (size_t)g.nU * g.capUp * dbytes))) return fail(rc);
    if ((rc = dev_alloc((void **)&ix->upper_owner, sizeof(int32_t) * g.nU))) return fail(rc);
    g.codes = ix->codes;
    g.adj0 = ix->adj0; g.cnt0 = ix->cnt0; g.cons0 = ix->cons0;
    g.adjU = ix->adjU; g.cntU = ix->cntU; g.consU = ix->consU;
    g.dist0 = ix->dist0; g.distU = ix->distU;
    g.tie = 0;
    g.expand = 1;
    g.gvis = nullptr;
    g.gvis_epoch = nullptr;
    g.gvis_owner = nullptr;
    g.gvis_log2 = 14;
    g.gvis_nslots = 0;
    g.gvis_words = 1;
    g.rowcnt = nullptr;
    g.touched = nullptr;
    g.ntouched = nullptr;
    g.seg_scratch = nullptr;
    // host copies of the layer draws drive the batch schedule
    ix->levels_h.resize(g.n);
    ix->uoff_h.resize(g.n);
    if (g.n) {
        cudaError_t e1 = cudaMemcpy(ix->levels_h.data(), desc->levels, sizeof(int32_t) * g.n,
                                    cudaMemcpyDeviceToHost);
        cudaError_t e2 = cudaMemcpy(ix->uoff_h.data(), desc->uoff, sizeof(int64_t) * g.n,
                                    cudaMemcpyDeviceToHost);
        if (e1 != cudaSuccess || e2 != cudaSuccess) {
            set_error("copying levels/upper offsets: %s", cudaGetErrorString(e1 ? e1 : e2));
            return fail(FA_ECUDA);
        }
    }
    std::vector<int32_t> owner(g.nU > 0 ? g.nU : 1, -1);
    for (int64_t v = 0; v < g.n; ++v) {
        int lv = ix->levels_h[v];
        if (lv > 0) {
            int64_t o = ix->uoff_h[v];
            if (o < 0 || o + lv > g.nU) {
                set_error("upper_offsets[%lld]=%lld inconsistent with levels", (long long)v,
                          (long long)o);
                return fail(FA_EINVAL);
            }
            for (int l = 0; l < lv; ++l) owner[o + l] = (int32_t)v;
        }
    }
    if (g.nU) {
        cudaError_t e = cudaMemcpy(ix->upper_owner, owner.data(), sizeof(int32_t) * g.nU,
                                   cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            set_error("upper owner copy: %s", cudaGetErrorString(e));
            return fail(FA_ECUDA);
        }
    }
    if ((rc = reset_graph(ix, 0))) return fail(rc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        set_error("index init: %s", cudaGetErrorString(e));
        return fail(FA_ECUDA);
    }
    *out = ix;
    return FA_OK;
}

extern "C" int fa_index_destroy(fa_index *ix) {
    if (!ix) return FA_OK;
    for (void *p : {(void *)ix->codes, (void *)ix->adj0, (void *)ix->cnt0, (void *)ix->cons0,
                    (void *)ix->adjU, (void *)ix->cntU, (void *)ix->consU, (void *)ix->dist0,
                    (void *)ix->distU, (void *)ix->upper_owner, (void *)ix->gvis,
                    (void *)ix->gvis_epoch, (void *)ix->gvis_owner})
        pool_free(p);
    delete ix;
    return FA_OK;
}

extern "C" int fa_index_set_search_tie(fa_index *ix, int mode) {
    FA_CHECK_ARG(ix && mode >= 0 && mode <= 2, "tie mode must be 0, 1 or 2");
    ix->search_tie = mode;
    return FA_OK;
}

namespace fa {
// codes of rows [r0, r1) from the projected vectors (K2)
int index_encode_rows(fa_index *ix, int64_t r0, int64_t r1, cudaStream_t st) {
    if (ix->g.m == 0 || r1 <= r0) return FA_OK;  // exact kind: no codes
    FA_CHECK_ARG(ix->d.proj, "index has no projected vectors to encode");
    const size_t cs = ix->g.mpad;
    FA_CUDA(cudaMemsetAsync(ix->codes + (size_t)r0 * cs, 0, (size_t)(r1 - r0) * cs, st));
    return launch_encode_adt(ix->d.proj + (size_t)r0 * ix->d.dproj, r1 - r0, ix->d.dproj,
                             ix->d.cent, ix->d.dims, ix->d.offs, ix->g.m, ix->d.dmax,
                             ix->d.dist_min, ix->d.delta, ix->codes + (size_t)r0 * cs,
                             ix->g.mpad, nullptr, 0, st);
}
void index_set_late_rows(fa_index *ix, int64_t from, std::function<int(cudaStream_t)> hook) {
    ix->late_from = from;
    ix->late_hook = std::move(hook);
}
}  // namespace fa

extern "C" int fa_index_encode(fa_index *ix, void *stream) {
    FA_CHECK_ARG(ix, "null index");
    return index_encode_rows(ix, 0, ix->g.n, as_stream(stream));
}

extern "C" int fa_index_set_codes(fa_index *ix, const uint8_t *codes, int code_stride,
                                  void *stream) {
    FA_CHECK_ARG(ix, "null index");
    if (ix->g.m == 0) return FA_OK;  // exact kind: no codes
    FA_CHECK_ARG(codes, "null codes");
    FA_CHECK_ARG(code_stride >= ix->g.m, "code_stride < m");
    cudaStream_t st = as_stream(stream);
    FA_CUDA(cudaMemsetAsync(ix->codes, 0, (size_t)ix->g.n * ix->g.mpad, st));
    if (ix->g.n)
        FA_CUDA(cudaMemcpy2DAsync(ix->codes, ix->g.mpad, codes, code_stride, ix->g.m, ix->g.n,
                                  cudaMemcpyDeviceToDevice, st));
    return FA_OK;
}

extern "C" const uint8_t *fa_index_codes(fa_index *ix, int *code_stride) {
    if (!ix) return nullptr;
    if (code_stride) *code_stride = ix->g.mpad;
    return ix->codes;
}

extern "C" int fa_index_adjacency(fa_index *ix, int layer_kind, const int32_t **ids,
                                  const int32_t **cnt, int *cap, int64_t *rows) {
    FA_CHECK_ARG(ix, "null index");
    if (layer_kind == 0) {
        *ids = ix->adj0; *cnt = ix->cnt0; *cap = ix->g.cap0p; *rows = ix->g.n;
    } else {
        *ids = ix->adjU; *cnt = ix->cntU; *cap = ix->g.capUp; *rows = ix->g.nU;
    }
    return FA_OK;
}

extern "C" int fa_index_build(fa_index *ix, const fa_build_opts *opts, fa_build_result *res,
                              void *stream) {
    FA_CHECK_ARG(ix && opts && res, "null argument");
    Graph &g = ix->g;
    const int C = opts->C;
    const int R = ix->d.R;
    FA_CHECK_ARG(C >= 1 && C <= 2048, "C=%d outside [1,2048]", C);
    const bool exact = g.m == 0;  // kind 0: fp32 L2 everywhere
    FA_CHECK_ARG(exact || ix->d.sdt, "index has no SDT");
    cudaStream_t st = as_stream(stream);
    memset(res, 0, sizeof(*res));
    res->entry_point = -1;
    res->max_layer = -1;
    const auto t_host0 = std::chrono::steady_clock::now();
    // FLASHANN_B200_TIMING: the host set-up's phases (diagnostics)
    const bool tmarks = getenv("FLASHANN_B200_TIMING") != nullptr;
    auto t_last = t_host0;
    auto tmark = [&](const char *what) {
        if (!tmarks) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[fa timing]   build set-up: %-22s %7.2f ms\n", what,
                std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    const int64_t r0 = opts->start, r1 = opts->end > 0 ? opts->end : g.n;
    FA_CHECK_ARG(r0 >= 0 && r0 <= r1 && r1 <= g.n, "insertion range [%lld, %lld) outside [0, %lld]",
                 (long long)r0, (long long)r1, (long long)g.n);
    FA_CHECK_ARG(r0 == 0 || r0 == ix->n_inserted,
                 "resuming at %lld but the graph holds %lld inserted vertices", (long long)r0,
                 (long long)ix->n_inserted);
    FA_CHECK_ARG(opts->tie >= 0 && opts->tie <= 2, "tie mode must be 0, 1 or 2");
    if (r0 == 0) {
        FA_TRY(reset_graph(ix, st));
        ix->n_inserted = 0;
        ix->entry = -1;
        ix->max_layer = -1;
    }
    Graph gb = g;  // the build's view: its own tie order
    gb.tie = opts->tie;
    gb.expand = opts->expand > 1 ? std::min(opts->expand, kMaxExpand) : 1;
    if (g.n == 0 || r1 == 0) {
        ix->entry = -1;
        ix->max_layer = -1;
        return FA_OK;
    }
    FA_CHECK_ARG(exact || ix->d.proj, "build needs the projected vectors (per-insertion tables)");
    const int Bmax = opts->batch_max > 0 ? opts->batch_max : 65536;
    const double frac = opts->batch_frac > 0 ? opts->batch_frac : 0.2;
    const int prefix = opts->seq_prefix >= 0 ? opts->seq_prefix : 256;
    const int Bmin = opts->batch_min >= 0 ? opts->batch_min
                                          : (int)std::min<int64_t>(4096, std::max<int64_t>(1, g.n / 256));

    tmark("graph reset");
    // ---- schedule (pure function of the layer draws) ----
    // From the record positions and one pass over the inserted range's
    // levels (each batch's request bound); the per-vertex request offsets are
    // written per batch in the launch loop.
    if (!ix->sched_ready) {
        ix->raisers.clear();
        int run = -1;
        const int32_t *lvh = ix->levels_h.data();
        for (int64_t v = 0; v < g.n; ++v) {
            if (lvh[v] > run) {
                if (v > 0) ix->raisers.push_back(v);
                run = lvh[v];
            }
        }
        ix->maxlv = std::max(run, 0);
        ix->sched_ready = true;
    }
    tmark("record positions");
    std::vector<Batch> batches;
    // vertex 0 seeds an empty graph; a resumed build starts from the state
    // the earlier calls left (entry point, top layer)
    int ep = r0 == 0 ? 0 : (int)ix->entry, ml = r0 == 0 ? ix->levels_h[0] : ix->max_layer;
    int64_t maxreq = 0;
    int maxB = 1;
    int64_t x = std::max<int64_t>(1, r0);
    size_t ri = 0;  // next record position at or after x
    while (x < r1) {
        while (ri < ix->raisers.size() && ix->raisers[ri] < x) ++ri;
        Batch b;
        b.start = (int)x;
        b.ep = ep;
        b.ml = ml;
        const bool raiser = ri < ix->raisers.size() && ix->raisers[ri] == x;
        int size;
        if (raiser) {
            size = 1;  // a new top layer goes alone
            b.nreq = (int64_t)(ml + 1) * R;
        } else {
            const int B = x < prefix ? 1
                          : std::max(1, std::min(Bmax, std::max((int)(frac * (double)x),
                                                                (int)std::min<int64_t>(x, Bmin))));
            int64_t end = std::min<int64_t>(r1, x + B);
            if (ri < ix->raisers.size()) end = std::min<int64_t>(end, ix->raisers[ri]);
            size = (int)(end - x);
            int64_t lsum = 0;  // the batch's levels: its upper-layer request slots
            const int32_t *lvh = ix->levels_h.data();
            for (int64_t v = x; v < end; ++v) lsum += lvh[v];
            b.nreq = (int64_t)R * (size + lsum);
        }
        b.size = size;
        b.raiser = raiser;
        batches.push_back(b);
        maxreq = std::max(maxreq, b.nreq);
        maxB = std::max(maxB, size);
        x += size;
        if (raiser) {
            ep = b.start;
            ml = ix->levels_h[b.start];
        }
    }

    tmark("batch schedule");
    // ---- scratch ----
    const int capmax = std::max(g.cap0, g.capU);
    if (exact || ix->wide) gb.expand = 1;
    // Visited table: 2^12 16-bit slots (8 KB) unless requested — a larger one
    // costs occupancy (the ids it cannot hold go to the global tier).  The
    // forward selection's workspace always lives in the dead table; the
    // sorted results join it when both fit, else they take their own space.
    const size_t sel_bytes = exact ? (size_t)2 * round_up(R, 4) * 4 + (size_t)g.dim * 4
                                   : (size_t)select_tv_bytes(g.m, g.mpad, R);
    // (the build kernels compile the table's 2^9 buckets in: requests above
    // 2^12 slots are clamped; growing hl below only makes room for the
    // selection workspace)
    int hl = opts->hash_log2 > 0 ? std::min(std::max(opts->hash_log2, 9), 12) : 12;
    while (((size_t)16 << vis_buckets_log2(hl)) < sel_bytes) ++hl;
    // (else they overlay the small block's search state, dead by then)
    const int t_alias =
        sel_bytes + (size_t)round_up(C, 32) * 8 <= ((size_t)16 << vis_buckets_log2(hl)) ? 1 : 2;
    WarpLayout L;
    L.init(g.mpad, C, capmax, hl, gb.expand, t_alias, exact ? g.dim * 4 : -1, (exact || ix->wide) ? 8 : 4);
    const size_t sdt_bytes = round_up(std::max(g.m, 1) * 256, 128);
    int bw = search_warps_for(L.total, kBuildWarpsMax);  // warps per CTA
    FA_CHECK_ARG(bw > 0, "search workspace %d B per warp exceeds shared memory", L.total);
    const BuildSearchFn search_fn =
        exact ? build_search_exact_variant(C, g.cap0, ix->wide)
              : build_search_variant(C, ix->wide ? 1 : gb.expand, g.cap0, ix->wide);
    FA_CUDA(cudaFuncSetAttribute((const void *)search_fn,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, bw * L.total));
    // the CTA width that keeps the most warps resident (each CTA also costs
    // 1 KB of reserved shared memory; 96 registers cap an SM at 5 warps per
    // scheduler = 20): config 2's 10.9 KB per warp runs 20 warps as 4 CTAs of
    // 5 (or 5 of 4), config 4's 11.3 KB 20 as 4 of 5 where CTAs of 4 reach
    // only 16; ties go to the wider CTA
    {
        int best = 0;
        const int wmax = bw;
        for (int w = wmax; w >= 1; --w) {
            int per = 0;
            FA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, search_fn, w * 32,
                                                                  (size_t)w * L.total));
            if (per * w > best) {
                best = per * w;
                bw = w;
            }
        }
        if (const char *e = getenv("FLASHANN_B200_SEARCH_WARPS"))
            bw = std::min(std::max(atoi(e), 1), wmax);
    }
    const size_t smem_search = (size_t)bw * L.total;
    ReverseLayout RL;
    RL.init(capmax, g.m, g.mpad, exact ? g.dim : 0);
    const bool rc2 = g.cap0 <= 64;  // base rows of <= 64 slots: two 32-slot chunks
    const void *rev_fn = exact ? (const void *)reverse_exact_kernel
                         : rc2 ? (const void *)reverse_kernel<2>
                               : (const void *)reverse_kernel<kRowChunks>;
    const size_t smem_rev = (size_t)kReverseWarps * RL.total;
    FA_CUDA(cudaFuncSetAttribute(rev_fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem_rev));

    // global select workspace of the reverse kernel's full prunes, per warp
    const int rev_sel_bytes = exact ? 16 : select_tv_ws_bytes(g.mpad, capmax + 1);
    int rev_per_sm = 0;
    FA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rev_per_sm, rev_fn,
                                                          kReverseWarps * 32, smem_rev));
    const int64_t rev_ctas = (int64_t)std::max(rev_per_sm, 1) * num_sms();
    int search_per_sm = 0;
    FA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&search_per_sm, search_fn,
                                                          bw * 32, smem_search));
    const int64_t search_ctas = (int64_t)std::max(search_per_sm, 1) * num_sms();
    // carve out only the shared memory the resident CTAs use: the rest stays
    // L1, which holds the transposed SDT and the hot code rows
    {
        const double need = (double)std::max(search_per_sm, 1) * (smem_search + 1024);
        int pct = (int)std::ceil(100.0 * need / (228.0 * 1024.0));
        if (const char *e = getenv("FLASHANN_B200_CARVEOUT")) pct = atoi(e);
        FA_CUDA(cudaFuncSetAttribute((const void *)search_fn,
                                     cudaFuncAttributePreferredSharedMemoryCarveout,
                                     std::min(100, std::max(0, pct))));
    }
    tmark("schedule + launch set-up");
    FA_TRY(ensure_gvis(ix, (const void *)search_fn, bw * 32, smem_search, C, st));
    tmark("global visited tier");
    gb.gvis = g.gvis;
    gb.gvis_epoch = g.gvis_epoch;
    gb.gvis_owner = g.gvis_owner;
    gb.gvis_log2 = g.gvis_log2;
    gb.gvis_nslots = g.gvis_nslots;
    gb.gvis_words = g.gvis_words;

    // batch descents + processing order (Flash kind): for the batches with
    // more vertices than resident search warps, where the order sets the tail
    const bool descend = !exact;
    const int maxlv = ix->maxlv;
    const int nkeys = (maxlv + 1) * 256;
    const int desc_ctx = WarpLayout::adt_bytes(g.mpad);
    const size_t smem_desc = (size_t)kSearchWarps * round_up(desc_ctx + 8 * capmax, 256);
    int64_t desc_ctas = 0;
    if (descend) {
        const void *df = ix->wide ? (const void *)batch_descend_kernel<FlashDistW>
                                  : (const void *)batch_descend_kernel<FlashDist>;
        if (smem_desc > 48 * 1024)
            FA_CUDA(cudaFuncSetAttribute(df, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem_desc));
        int per = 0;
        FA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, df, kSearchWarps * 32, smem_desc));
        desc_ctas = (int64_t)std::max(per, 1) * num_sms();
    }
    int32_t *start_v = nullptr, *hist = nullptr;
    uint32_t *start_d = nullptr;
    uint8_t *adt_batch = nullptr, *sdtT = nullptr, *rev_sel = nullptr;
    unsigned long long *req = nullptr, *req_sorted = nullptr, *ctr = nullptr;
    int64_t *req_off_d = nullptr, *heads = nullptr;
    int32_t *order_d = nullptr, *rowcnt = nullptr, *rowoff = nullptr, *touched = nullptr;
    int *err = nullptr, *nheads = nullptr, *next_seg = nullptr;
    int rc = FA_OK;
    // scratch is stream-ordered (cudaMallocAsync from the device's pool, kept
    // cached across builds): no allocation or free synchronises the device
    auto cleanup = [&]() {
        for (void *p : {(void *)start_v, (void *)start_d, (void *)hist})
            if (p) cudaFreeAsync(p, st);
        for (void *p : {(void *)adt_batch, (void *)req, (void *)req_sorted, (void *)ctr,
                        (void *)req_off_d, (void *)order_d, (void *)err, (void *)heads,
                        (void *)nheads, (void *)next_seg, (void *)sdtT, (void *)rev_sel,
                        (void *)rowcnt, (void *)rowoff, (void *)touched})
            if (p) cudaFreeAsync(p, st);
    };
    auto dev_alloc = [&](void **p, size_t bytes) -> int {
        cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 16, st);
        if (e != cudaSuccess) {
            set_error("cudaMallocAsync(%zu bytes): %s", bytes, cudaGetErrorString(e));
            return e == cudaErrorMemoryAllocation ? FA_ENOMEM : FA_ECUDA;
        }
        return FA_OK;
    };
    keep_pool();  // scratch stays mapped in the pool between builds
    const int64_t nrows = g.n + g.nU;  // layer-0 rows, then the upper rows
    if ((rc = dev_alloc((void **)&adt_batch, (size_t)maxB * g.mpad * 16)) ||
        (rc = dev_alloc((void **)&req, sizeof(unsigned long long) * std::max<int64_t>(maxreq, 1))) ||
        (rc = dev_alloc((void **)&req_sorted, sizeof(unsigned long long) * (std::max<int64_t>(maxreq, 1) + 1))) ||
        (rc = dev_alloc((void **)&rowcnt, sizeof(int32_t) * nrows)) ||
        (rc = dev_alloc((void **)&rowoff, sizeof(int32_t) * nrows)) ||
        (rc = dev_alloc((void **)&touched, sizeof(int32_t) * std::max<int64_t>(maxreq, 1))) ||
        (rc = dev_alloc((void **)&ctr, sizeof(unsigned long long) * 8)) ||
        (rc = dev_alloc((void **)&req_off_d, sizeof(int64_t) * g.n)) ||
        (rc = dev_alloc((void **)&order_d, sizeof(int32_t) * g.n)) ||
        (rc = dev_alloc((void **)&heads, sizeof(int64_t) * std::max<int64_t>(maxreq, 1))) ||
        (rc = dev_alloc((void **)&nheads, 4 * sizeof(int))) ||
        (descend && (rc = dev_alloc((void **)&start_v, sizeof(int32_t) * (size_t)maxB))) ||
        (descend && (rc = dev_alloc((void **)&start_d, sizeof(uint32_t) * (size_t)maxB))) ||
        (descend && (rc = dev_alloc((void **)&hist, sizeof(int32_t) * (size_t)nkeys))) ||
        (rc = dev_alloc((void **)&next_seg, sizeof(int))) ||
        (rc = dev_alloc((void **)&sdtT, sdt_bytes)) ||
        (rc = dev_alloc((void **)&rev_sel, (size_t)rev_ctas * kReverseWarps * rev_sel_bytes)) ||
        (rc = dev_alloc((void **)&err, sizeof(int)))) {
        cleanup();
        return rc;
    }
#define FA_BUILD_CUDA(call)                                                              \
    do {                                                                                 \
        cudaError_t _e = (call);                                                         \
        if (_e != cudaSuccess) {                                                         \
            set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
            cleanup();                                                                   \
            return FA_ECUDA;                                                             \
        }                                                                                \
    } while (0)
    tmark("scratch");
    FA_BUILD_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * 8, st));
    // per-row request counts: zero here, re-zeroed by the reverse warps
    FA_BUILD_CUDA(cudaMemsetAsync(rowcnt, 0, sizeof(int32_t) * nrows, st));
    gb.rowcnt = rowcnt;
    gb.touched = touched;
    gb.ntouched = nheads;  // nheads[0]: touched rows = row segments of the batch
    gb.seg_scratch = req;  // the unbucketed requests are dead once scattered
    if (!exact) {
        transpose_sdt_kernel<<<1, 256, 0, st>>>(ix->d.sdt, g.m, sdtT);
        FA_BUILD_CUDA(cudaGetLastError());
    }
    FA_BUILD_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
    // processing order inside each batch: higher levels first (their searches
    // are the longest: hill climb plus one beam search per layer), ties in
    // vertex order.  Every vertex of a batch sees the graph as of the batch
    // start and writes only its own rows and request slots, so the order
    // changes no result, only the length of the batch's tail.  Filled per
    // batch in the launch loop (pinned buffer, async copy): the host work
    // overlaps the device's earlier batches.
    int32_t *order_h = nullptr;
    int64_t *reqoff_h = nullptr;
    std::unique_lock<std::mutex> order_lock(g_order_mu);  // held to the final sync
    if ((rc = pinned_order(g.n, &order_h, &reqoff_h))) {
        cleanup();
        return rc;
    }
    std::vector<int> lvpos((size_t)maxlv + 2);
    // optional per-kernel-class timing: 5 events per batch on the build stream
    const bool prof = opts->profile != 0;
    std::vector<cudaEvent_t> ev;
    if (prof) {
        ev.resize(batches.size() * 5);
        for (auto &e : ev) FA_BUILD_CUDA(cudaEventCreate(&e));
    }
    if (getenv("FLASHANN_B200_TIMING"))
        fprintf(stderr, "[fa timing] build host setup (schedule, scratch) %8.2f ms\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                          t_host0).count());
    int64_t launches = r0 == 0 ? 3 : 1;  // the two row resets of reset_graph, the SDT transpose
    for (size_t bi = 0; bi < batches.size(); ++bi) {
        const Batch &b = batches[bi];
        if (ix->late_hook && ix->late_from >= 0 && (int64_t)b.start + b.size > ix->late_from) {
            auto hook = std::move(ix->late_hook);
            ix->late_hook = nullptr;
            ix->late_from = -1;
            if ((rc = hook(st))) {
                cleanup();
                return rc;
            }
        }
        if (prof) FA_BUILD_CUDA(cudaEventRecord(ev[bi * 5 + 0], st));
        if (!exact) {
            rc = launch_encode_adt(ix->d.proj + (size_t)b.start * ix->d.dproj, b.size,
                                   ix->d.dproj, ix->d.cent, ix->d.dims, ix->d.offs, g.m,
                                   ix->d.dmax, ix->d.dist_min, ix->d.delta, nullptr, g.mpad,
                                   adt_batch, g.mpad, st);
            if (rc) {
                cleanup();
                return rc;
            }
        }
        if (prof) FA_BUILD_CUDA(cudaEventRecord(ev[bi * 5 + 1], st));
        // more vertices than resident search warps: descents first, then the
        // processing order from them (build_search.cu batch_descend_kernel)
        const bool desc_b = descend && (int64_t)b.size > search_ctas * bw;
        {
            const int32_t *lv = ix->levels_h.data() + b.start;
            if (!desc_b) {  // stable counting sort of the batch by level, descending
                int32_t *o = order_h + b.start;
                std::fill(lvpos.begin(), lvpos.end(), 0);
                for (int k = 0; k < b.size; ++k) ++lvpos[maxlv - lv[k] + 1];
                for (int l = 1; l <= maxlv + 1; ++l) lvpos[l] += lvpos[l - 1];
                for (int k = 0; k < b.size; ++k) o[lvpos[maxlv - lv[k]]++] = k;
                FA_BUILD_CUDA(cudaMemcpyAsync(order_d + b.start, o, sizeof(int32_t) * b.size,
                                              cudaMemcpyHostToDevice, st));
            }
            // request slots: (min(ml, level) + 1) R per vertex, in vertex order
            int64_t *ro = reqoff_h + b.start;
            int64_t off = 0;
            for (int k = 0; k < b.size; ++k) {
                ro[k] = off;
                off += (int64_t)(std::min(b.ml, lv[k]) + 1) * R;
            }
            FA_BUILD_CUDA(cudaMemcpyAsync(req_off_d + b.start, ro, sizeof(int64_t) * b.size,
                                          cudaMemcpyHostToDevice, st));
        }
        // nheads[0]: touched rows (= row segments), nheads[1]: the search's
        // work counter, nheads[2]: the bucketing cursor
        FA_BUILD_CUDA(cudaMemsetAsync(nheads, 0, 4 * sizeof(int), st));
        if (desc_b) {
            FA_BUILD_CUDA(cudaMemsetAsync(hist, 0, sizeof(int32_t) * (size_t)nkeys, st));
            const int dgrid = (int)std::min<int64_t>(desc_ctas, (b.size + kSearchWarps - 1) / kSearchWarps);
            if (ix->wide)
                batch_descend_kernel<FlashDistW><<<dgrid, kSearchWarps * 32, smem_desc, st>>>(
                    gb, adt_batch, b.start, b.size, b.ep, b.ml, nkeys / 256 - 1, desc_ctx, capmax,
                    start_v, start_d, hist, ctr, nheads + 3);
            else
                batch_descend_kernel<FlashDist><<<dgrid, kSearchWarps * 32, smem_desc, st>>>(
                    gb, adt_batch, b.start, b.size, b.ep, b.ml, nkeys / 256 - 1, desc_ctx, capmax,
                    start_v, start_d, hist, ctr, nheads + 3);
            descend_scan_kernel<<<1, 1024, 0, st>>>(hist, nkeys);
            descend_order_kernel<<<(int)std::min<int64_t>(num_sms() * 4, (b.size + 255) / 256), 256, 0,
                                   st>>>(ix->d.levels, b.start, b.size, nkeys / 256 - 1, start_d, hist,
                                         order_d + b.start);
            FA_BUILD_CUDA(cudaGetLastError());
            launches += 3;
        }
        int grid = (int)std::min<int64_t>(search_ctas, (b.size + bw - 1) / bw);
        search_fn<<<grid, bw * 32, smem_search, st>>>(
            gb, sdtT, adt_batch, b.start, b.size, b.ep, b.ml, C, R, L, req_off_d + b.start,
            order_d + b.start,
            req, ctr, err, opts->point_stats, nheads + 1, desc_b ? start_v : nullptr,
            desc_b ? start_d : nullptr);
        FA_BUILD_CUDA(cudaGetLastError());
        if (prof) FA_BUILD_CUDA(cudaEventRecord(ev[bi * 5 + 2], st));
        // bucket the requests by row: segments for the touched rows, then
        // every request into its row's segment (no sort; reverse.cu)
        {
            const int bgrid = (int)std::min<int64_t>(num_sms() * 4, (b.nreq + 255) / 256 + 1);
            bucket_place_kernel<<<bgrid, 256, 0, st>>>(touched, nheads, rowcnt, rowoff, heads,
                                                        nheads + 2);
            bucket_scatter_kernel<<<bgrid, 256, 0, st>>>(req, b.nreq, rowcnt, rowoff, nheads + 2,
                                                          req_sorted);
            FA_BUILD_CUDA(cudaMemsetAsync(next_seg, 0, sizeof(int), st));
            FA_BUILD_CUDA(cudaGetLastError());
        }
        if (prof) FA_BUILD_CUDA(cudaEventRecord(ev[bi * 5 + 3], st));
        // persistent warps pull row segments; never more warps than requests
        int rgrid = (int)std::min<int64_t>(rev_ctas, (b.nreq + 32 * kReverseWarps - 1) /
                                                          (32 * kReverseWarps) + 1);
        if (exact)
            reverse_exact_kernel<<<rgrid, kReverseWarps * 32, smem_rev, st>>>(
                gb, req_sorted, b.nreq, heads, nheads, next_seg, ix->upper_owner, RL, ctr);
        else if (rc2)
            reverse_kernel<2><<<rgrid, kReverseWarps * 32, smem_rev, st>>>(
                gb, ix->d.sdt, sdtT, req_sorted, b.nreq, heads, nheads, next_seg,
                ix->upper_owner, RL, ctr, rev_sel, rev_sel_bytes);
        else
            reverse_kernel<kRowChunks><<<rgrid, kReverseWarps * 32, smem_rev, st>>>(
                gb, ix->d.sdt, sdtT, req_sorted, b.nreq, heads, nheads, next_seg,
                ix->upper_owner, RL, ctr, rev_sel, rev_sel_bytes);
        FA_BUILD_CUDA(cudaGetLastError());
        if (prof) FA_BUILD_CUDA(cudaEventRecord(ev[bi * 5 + 4], st));
        launches += 5;
    }
    unsigned long long hc[8];
    int herr = 0;
    FA_BUILD_CUDA(cudaMemcpyAsync(hc, ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
    FA_BUILD_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
    FA_BUILD_CUDA(cudaStreamSynchronize(st));
    if (prof) {
        double acc[4] = {0, 0, 0, 0};
        // FLASHANN_B200_BATCH_LOG=1: one stderr line per batch (diagnostics)
        const bool blog = getenv("FLASHANN_B200_BATCH_LOG") != nullptr;
        for (size_t bi = 0; bi < batches.size(); ++bi) {
            float bms[4] = {0.f, 0.f, 0.f, 0.f};
            for (int k = 0; k < 4; ++k) {
                FA_BUILD_CUDA(cudaEventElapsedTime(&bms[k], ev[bi * 5 + k], ev[bi * 5 + k + 1]));
                acc[k] += bms[k];
            }
            if (blog)
                fprintf(stderr, "[fa batch] %zu start %lld size %d nreq %lld ms %.4f %.4f %.4f %.4f\n",
                        bi, (long long)batches[bi].start, batches[bi].size,
                        (long long)batches[bi].nreq, bms[0], bms[1], bms[2], bms[3]);
        }
        for (auto &e : ev) cudaEventDestroy(e);
        res->ms_encode = acc[0];
        res->ms_search = acc[1];
        res->ms_sort = acc[2];
        res->ms_reverse = acc[3];
    }
    res->launches = launches;
#undef FA_BUILD_CUDA
    cleanup();
    if (herr) {
        set_error("visited-set overflow: an insertion search (C=%d) visited more vertices than "
                  "its 2^%d-entry global table holds", C, g.gvis_log2);
        return FA_EOVERFLOW;
    }
    ix->entry = ep;
    ix->max_layer = ml;
    ix->n_inserted = r1;
    res->entry_point = ep;
    res->max_layer = ml;
    res->n_batches = (int32_t)batches.size();
    res->dist_comps = (int64_t)hc[0];
    res->sym_comps = (int64_t)hc[1];
    res->kernel_calls = (int64_t)hc[2];
    res->visited = (int64_t)hc[3];
    res->reverse_prunes = (int64_t)hc[4];
    res->reverse_appends = (int64_t)hc[5];
    res->reverse_full_prunes = (int64_t)hc[6];
    return FA_OK;
}

static int run_query_encode(fa_index *ix, const float *qproj, int nq, uint8_t **adt_q,
                            cudaStream_t st) {
    FA_TRY(dev_alloc((void **)adt_q, (size_t)std::max(nq, 1) * ix->g.mpad * 16));
    int rc = launch_encode_adt(qproj, nq, ix->d.dproj, ix->d.cent, ix->d.dims, ix->d.offs, ix->g.m,
                               ix->d.dmax, ix->d.dist_min, ix->d.delta, nullptr, ix->g.mpad, *adt_q,
                               ix->g.mpad, st);
    if (rc) {
        pool_free(*adt_q);
        *adt_q = nullptr;
    }
    return rc;
}

extern "C" int fa_index_search(fa_index *ix, const float *queries, const float *qproj, int nq,
                               int ef, int k, int rerank_depth, int64_t entry, int max_layer,
                               int64_t *out_ids, double *out_d, int64_t *counters, void *stream) {
    FA_CHECK_ARG(ix, "null index");
    if (entry < 0) {
        set_error("cannot search an empty graph");
        return FA_EEMPTY;
    }
    FA_CHECK_ARG(entry < ix->g.n, "entry point out of range");
    FA_CHECK_ARG(ef >= 1 && ef <= 4096 && k >= 1, "need 1 <= k, 1 <= ef <= 4096");
    FA_CHECK_ARG(rerank_depth == 0 || (ix->d.vecs && queries), "rerank needs vectors and queries");
    const bool exact = ix->g.m == 0;
    FA_CHECK_ARG(!exact || queries, "the exact kind searches with the query vectors");
    cudaStream_t st = as_stream(stream);
    if (counters) memset(counters, 0, 4 * sizeof(int64_t));
    if (nq == 0) return FA_OK;
    const int capmax = std::max(ix->g.cap0, ix->g.capU);
    WarpLayout L;
    L.init(ix->g.mpad, ef, capmax,
           pick_hash_log2(ef, capmax, 1, ix->g.mpad, 0,
                          (size_t)8 * std::min(std::max(rerank_depth, 0), ef)),
           1, false, exact ? ix->d.dim * 4 : -1, (exact || ix->wide) ? 8 : 4);
    const int qw = search_warps_for(L.total);  // warps per CTA
    FA_CHECK_ARG(qw > 0, "search workspace %d B per warp exceeds shared memory", L.total);
    size_t smem = (size_t)qw * L.total;
    const QuerySearchFn qfn = query_search_variant(ef, exact, ix->wide);
    FA_CUDA(cudaFuncSetAttribute((const void *)qfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    FA_TRY(ensure_gvis(ix, (const void *)qfn, qw * 32, smem, ef, st));
    uint8_t *adt_q = nullptr;
    if (!exact) FA_TRY(run_query_encode(ix, qproj, nq, &adt_q, st));
    unsigned long long *ctr = nullptr;
    int *err = nullptr;
    int rc = dev_alloc((void **)&ctr, 8 * sizeof(unsigned long long));
    if (!rc) rc = dev_alloc((void **)&err, sizeof(int));
    unsigned long long hc[8] = {0};
    int herr = 0;
    if (!rc) {
        cudaMemsetAsync(ctr, 0, 8 * sizeof(unsigned long long), st);
        cudaMemsetAsync(err, 0, sizeof(int), st);
        int grid = (nq + qw - 1) / qw;
        Graph gq = ix->g;
        gq.tie = ix->search_tie;
        gq.expand = 1;
        qfn<<<grid, qw * 32, smem, st>>>(
            gq, adt_q, nq, (int)entry, max_layer, ef, k, rerank_depth, ix->d.vecs, ix->d.dim,
            queries, L, out_ids, out_d, ctr, err);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpyAsync(hc, ctr, sizeof(hc), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            set_error("query search: %s", cudaGetErrorString(e));
            rc = FA_ECUDA;
        }
    }
    pool_free(adt_q);
    pool_free(ctr);
    pool_free(err);
    if (rc) return rc;
    if (herr) {
        set_error("visited-set overflow in query search (ef=%d, table 2^%d)", ef,
                  ix->g.gvis_log2);
        return FA_EOVERFLOW;
    }
    if (counters)
        for (int i = 0; i < 4; ++i) counters[i] = (int64_t)hc[i];
    return FA_OK;
}

extern "C" int fa_index_search_layer(fa_index *ix, const float *qproj, int nq,
                                     const int64_t *entries, int width, int layer,
                                     int32_t *out_ids, double *out_d, int32_t *out_n,
                                     int64_t *counters, void *stream) {
    FA_CHECK_ARG(ix, "null index");
    FA_CHECK_ARG(width >= 1 && width <= 4096, "width=%d outside [1,4096]", width);
    FA_CHECK_ARG(layer >= 0, "layer < 0");
    cudaStream_t st = as_stream(stream);
    if (counters) memset(counters, 0, 4 * sizeof(int64_t));
    if (nq == 0) return FA_OK;
    // exact kind: qproj holds the query vectors (dim floats per row)
    const bool exact = ix->g.m == 0;
    const int capmax = std::max(ix->g.cap0, ix->g.capU);
    WarpLayout L;
    L.init(ix->g.mpad, width, capmax, pick_hash_log2(width, capmax, 1, ix->g.mpad, 0), 1, false,
           exact ? ix->d.dim * 4 : -1, (exact || ix->wide) ? 8 : 4);
    const int qw = search_warps_for(L.total);  // warps per CTA
    FA_CHECK_ARG(qw > 0, "search workspace %d B per warp exceeds shared memory", L.total);
    size_t smem = (size_t)qw * L.total;
    const LayerSearchFn lfn = layer_search_variant(width, exact, ix->wide);
    FA_CUDA(cudaFuncSetAttribute((const void *)lfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    FA_TRY(ensure_gvis(ix, (const void *)lfn, qw * 32, smem, width, st));
    uint8_t *adt_q = nullptr;
    if (!exact) FA_TRY(run_query_encode(ix, qproj, nq, &adt_q, st));
    unsigned long long *ctr = nullptr;
    int *err = nullptr;
    int rc = dev_alloc((void **)&ctr, 8 * sizeof(unsigned long long));
    if (!rc) rc = dev_alloc((void **)&err, sizeof(int));
    unsigned long long hc[8] = {0};
    int herr = 0;
    if (!rc) {
        cudaMemsetAsync(ctr, 0, 8 * sizeof(unsigned long long), st);
        cudaMemsetAsync(err, 0, sizeof(int), st);
        int grid = (nq + qw - 1) / qw;
        Graph gq = ix->g;
        gq.tie = ix->search_tie;
        gq.expand = 1;
        lfn<<<grid, qw * 32, smem, st>>>(
            gq, exact ? reinterpret_cast<const uint8_t *>(qproj) : adt_q, nq, entries, width,
            layer, L, out_ids, out_d, out_n, ctr, err);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpyAsync(hc, ctr, sizeof(hc), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            set_error("layer search: %s", cudaGetErrorString(e));
            rc = FA_ECUDA;
        }
    }
    pool_free(adt_q);
    pool_free(ctr);
    pool_free(err);
    if (rc) return rc;
    if (herr) {
        set_error("visited-set overflow in layer search (width=%d, table 2^%d)", width,
                  ix->g.gvis_log2);
        return FA_EOVERFLOW;
    }
    if (counters)
        for (int i = 0; i < 4; ++i) counters[i] = (int64_t)hc[i];
    return FA_OK;
}

extern "C" int fa_index_export_blocks(fa_index *ix, uint8_t *base_blocks, int64_t base_stride,
                                      uint8_t *upper_blocks, int64_t upper_stride, void *stream) {
    FA_CHECK_ARG(ix, "null index");
    const Graph &g = ix->g;
    const int nb0 = (g.cap0 + 15) / 16, nbU = (g.capU + 15) / 16;
    FA_CHECK_ARG(base_stride >= 4 + 4 * g.cap0 + nb0 * g.m * 16, "base stride too small");
    cudaStream_t st = as_stream(stream);
    if (g.n) {
        FA_TRY(launch_export(g, g.n, false, base_blocks, base_stride, g.cap0, g.cap0p, st));
    }
    if (g.nU) {
        FA_CHECK_ARG(upper_blocks && upper_stride >= 4 + 4 * g.capU + nbU * g.m * 16,
                     "upper stride too small");
        FA_TRY(launch_export(g, g.nU, true, upper_blocks, upper_stride, g.capU, g.capUp, st));
    }
    return FA_OK;
}

extern "C" int fa_index_export_rows(fa_index *ix, int32_t *base_rows, int32_t *upper_rows,
                                    void *stream) {
    FA_CHECK_ARG(ix, "null index");
    Graph g = ix->g;
    g.m = 0;  // count + ids only
    g.mpad = 0;
    cudaStream_t st = as_stream(stream);
    if (g.n)
        FA_TRY(launch_export(g, g.n, false, reinterpret_cast<uint8_t *>(base_rows),
                             4 + 4 * (int64_t)g.cap0, g.cap0, g.cap0p, st));
    if (g.nU) {
        FA_CHECK_ARG(upper_rows, "upper rows needed");
        FA_TRY(launch_export(g, g.nU, true, reinterpret_cast<uint8_t *>(upper_rows),
                             4 + 4 * (int64_t)g.capU, g.capU, g.capUp, st));
    }
    return FA_OK;
}

extern "C" int fa_index_import_blocks(fa_index *ix, const uint8_t *base_blocks, int64_t base_stride,
                                      const uint8_t *upper_blocks, int64_t upper_stride,
                                      void *stream) {
    FA_CHECK_ARG(ix, "null index");
    const Graph &g = ix->g;
    FA_CHECK_ARG(base_stride >= 4 + 4 * g.cap0, "base stride too small");
    cudaStream_t st = as_stream(stream);
    if (g.n) {
        import_kernel<<<1184, 256, 0, st>>>(g, g.n, false, base_blocks, base_stride, g.cap0, g.cap0p);
        FA_LAUNCH_CHECK();
    }
    if (g.nU) {
        FA_CHECK_ARG(upper_blocks && upper_stride >= 4 + 4 * g.capU, "upper stride too small");
        import_kernel<<<1184, 256, 0, st>>>(g, g.nU, true, upper_blocks, upper_stride, g.capU,
                                            g.capUp);
        FA_LAUNCH_CHECK();
    }
    return FA_OK;
}
