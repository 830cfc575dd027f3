// C-ABI plumbing: error strings, version, and the host-pointer drop-ins that
// mirror the reference core's blocking Cython entry points
// (build_graph _core.pyx:711-764, search_batch _core.pyx:817-888).
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <emmintrin.h>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace fa {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// RAII device buffer for the host drop-ins.
struct DevBuf {
    void *p = nullptr;
    ~DevBuf() { pool_free(p); }
    int alloc(size_t bytes) { return pool_alloc(&p, bytes); }
    int upload(const void *src, size_t bytes);
    template <typename T> T *as() const { return reinterpret_cast<T *>(p); }
};

// ---- pageable host <-> device copies --------------------------------------
// The drop-ins take the caller's (pageable) numpy buffers.  Large transfers
// go through per-worker pinned staging buffers: each worker thread moves its
// own chunks (DMA on its own stream + host memcpy), so the DMA of one chunk
// overlaps the host copies of the others and the host side runs on several
// cores.  The pinned pool is allocated once per process.
// chunk size (FLASHANN_B200_STAGE_MB, default 32)
static size_t stage_bytes() {
    static size_t b = 0;
    if (b == 0) {
        const char *e = getenv("FLASHANN_B200_STAGE_MB");
        b = (size_t)(e ? std::min(256, std::max(1, atoi(e))) : 32) << 20;
    }
    return b;
}
// worker threads (FLASHANN_B200_STAGE_WORKERS, default 8, at most 32)
static int stage_workers() {
    static int w = 0;
    if (w == 0) {
        const char *e = getenv("FLASHANN_B200_STAGE_WORKERS");
        w = e ? std::min(32, std::max(1, atoi(e))) : 8;
    }
    return w;
}
static std::mutex g_stage_mu;
static std::vector<void *> g_stage;

// Run fn(chunk, pinned buffer, stream) -> cudaError_t over chunks 0..nchunk-1
// on the staging workers (worker w takes chunks w, w + T, ...).
template <class F>
static int stage_run(size_t nchunk, const char *what, F fn, int workers = 0) {
    std::lock_guard<std::mutex> lk(g_stage_mu);  // one staged copy at a time
    const size_t kStageBytes = stage_bytes();
    const int T = (int)std::min<size_t>(workers > 0 ? workers : stage_workers(), nchunk);
    while ((int)g_stage.size() < T) {
        void *p = nullptr;
        cudaError_t e = cudaHostAlloc(&p, kStageBytes, cudaHostAllocDefault);
        if (e != cudaSuccess) {
            set_error("cudaHostAlloc(%zu): %s", kStageBytes, cudaGetErrorString(e));
            return FA_ENOMEM;
        }
        g_stage.push_back(p);
    }
    int device = 0;
    FA_CUDA(cudaGetDevice(&device));
    std::vector<cudaError_t> err(T, cudaSuccess);
    std::vector<std::thread> th;
    for (int w = 0; w < T; ++w)
        th.emplace_back([&, w]() {
            cudaError_t e = cudaSetDevice(device);
            cudaStream_t s = nullptr;
            if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
            uint8_t *buf = static_cast<uint8_t *>(g_stage[w]);
            for (size_t c = w; c < nchunk && e == cudaSuccess; c += T) e = fn(c, buf, s);
            if (s) cudaStreamDestroy(s);
            err[w] = e;
        });
    for (auto &t : th) t.join();
    for (cudaError_t e : err)
        if (e != cudaSuccess) {
            set_error("staged %s: %s", what, cudaGetErrorString(e));
            return FA_ECUDA;
        }
    return FA_OK;
}

static int staged_copy(void *host, void *dev, size_t bytes, bool d2h) {
    if (bytes == 0) return FA_OK;
    const size_t kStageBytes = stage_bytes();
    const size_t nchunk = (bytes + kStageBytes - 1) / kStageBytes;
    if (nchunk < 2) {
        FA_CUDA(d2h ? cudaMemcpy(host, dev, bytes, cudaMemcpyDeviceToHost)
                    : cudaMemcpy(dev, host, bytes, cudaMemcpyHostToDevice));
        return FA_OK;
    }
    return stage_run(nchunk, d2h ? "D2H copy" : "H2D copy",
                     [&](size_t c, uint8_t *buf, cudaStream_t s) {
                         const size_t off = c * kStageBytes, len = std::min(kStageBytes, bytes - off);
                         uint8_t *h = static_cast<uint8_t *>(host) + off;
                         uint8_t *d = static_cast<uint8_t *>(dev) + off;
                         cudaError_t e;
                         if (d2h) {
                             e = cudaMemcpyAsync(buf, d, len, cudaMemcpyDeviceToHost, s);
                             if (e == cudaSuccess) e = cudaStreamSynchronize(s);
                             if (e == cudaSuccess) memcpy(h, buf, len);
                         } else {
                             memcpy(buf, h, len);
                             e = cudaMemcpyAsync(d, buf, len, cudaMemcpyHostToDevice, s);
                             if (e == cudaSuccess) e = cudaStreamSynchronize(s);
                         }
                         return e;
                     });
}

// Upload the first row_bytes of each of `rows` strided host rows into a
// contiguous device array (rows x row_bytes): the workers gather the rows
// straight into their pinned buffers.  Used for the id part of reference
// blocks, whose inline code bytes the device index never reads.
static int staged_gather_rows(void *dev, const void *host, int64_t rows, int64_t src_stride,
                              size_t row_bytes) {
    if (rows == 0 || row_bytes == 0) return FA_OK;
    const size_t per = std::max<size_t>(1, stage_bytes() / row_bytes);
    const size_t nchunk = ((size_t)rows + per - 1) / per;
    return stage_run(nchunk, "row gather", [&](size_t c, uint8_t *buf, cudaStream_t s) {
        const size_t r0 = c * per, r1 = std::min<size_t>((size_t)rows, r0 + per);
        const uint8_t *h = static_cast<const uint8_t *>(host);
        for (size_t r = r0; r < r1; ++r)
            memcpy(buf + (r - r0) * row_bytes, h + r * (size_t)src_stride, row_bytes);
        cudaError_t e = cudaMemcpyAsync(static_cast<uint8_t *>(dev) + r0 * row_bytes, buf,
                                        (r1 - r0) * row_bytes, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        return e;
    });
}

int DevBuf::upload(const void *src, size_t bytes) {
    FA_TRY(alloc(bytes));
    return staged_copy(const_cast<void *>(src), p, bytes, false);
}

// A staged host-to-device copy on a helper thread (same device as the
// caller); join() returns its status and carries its error text over.
struct AsyncUpload {
    int rc = FA_OK;
    char err[sizeof(g_err)] = "";
    std::thread th;
    bool joined = false;
    AsyncUpload(const void *src, void *dst, size_t bytes) {
        int dev = 0;
        cudaGetDevice(&dev);
        th = std::thread([this, src, dst, bytes, dev]() {
            cudaError_t e = cudaSetDevice(dev);
            rc = e == cudaSuccess ? staged_copy(const_cast<void *>(src), dst, bytes, false)
                                  : FA_ECUDA;
            if (rc != FA_OK) snprintf(err, sizeof(err), "%s", g_err);
        });
    }
    int join() {
        if (!joined) {
            th.join();
            joined = true;
            if (rc != FA_OK) set_error("%s", err);
        }
        return rc;
    }
    ~AsyncUpload() {
        if (!joined) th.join();
    }
};
// Two staged host-to-device copies in sequence on one helper thread: the
// first part (rows the build needs at once), then the rest (rows it needs
// later).  wait_first() blocks until the first part is on the device.
struct TwoPartUpload {
    int rc1 = FA_OK, rc2 = FA_OK;
    char err[sizeof(g_err)] = "";
    bool done1 = false, joined = false;
    std::mutex mu;
    std::condition_variable cv;
    std::thread th;
    TwoPartUpload(const void *src, void *dst, size_t first, size_t total) {
        int dev = 0;
        cudaGetDevice(&dev);
        th = std::thread([this, src, dst, first, total, dev]() {
            int r = cudaSetDevice(dev) == cudaSuccess
                        ? staged_copy(const_cast<void *>(src), dst, first, false)
                        : FA_ECUDA;
            if (r != FA_OK) snprintf(err, sizeof(err), "%s", g_err);
            {
                std::lock_guard<std::mutex> lk(mu);
                rc1 = r;
                done1 = true;
            }
            cv.notify_all();
            if (r == FA_OK && total > first) {
                rc2 = staged_copy(static_cast<uint8_t *>(const_cast<void *>(src)) + first,
                                  static_cast<uint8_t *>(dst) + first, total - first, false);
                if (rc2 != FA_OK) snprintf(err, sizeof(err), "%s", g_err);
            }
        });
    }
    int wait_first() {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [this] { return done1; });
        if (rc1 != FA_OK) set_error("%s", err);
        return rc1;
    }
    int join() {
        if (!joined) {
            th.join();
            joined = true;
        }
        const int rc = rc1 != FA_OK ? rc1 : rc2;
        if (rc != FA_OK) set_error("%s", err);
        return rc;
    }
    ~TwoPartUpload() {
        if (!joined) th.join();
    }
};

// FA_TRY that first waits for an in-flight AsyncUpload (its buffers must
// outlive it)
#define FA_TRY_JOIN(up, call)      \
    do {                           \
        int _rc = (call);          \
        if (_rc != FA_OK) {        \
            (up).join();           \
            return _rc;            \
        }                          \
    } while (0)

// ---- reference blocks assembled on the host ---------------------------------
// The inline code bytes of a reference block (layout.py:1-45) repeat codes[]
// of its neighbours, so the host drop-in moves only (count, ids) rows over
// PCIe and writes the code batches here, from the caller's code table.  A
// 16-slot batch is a 16 x m byte transpose of 16 code rows: SSE2 unpacks on
// 16 x 16 tiles (scalar for an m % 16 tail).
static inline void transpose16(__m128i r[16]) {
    __m128i a[16], b[16], c[16];
    for (int k = 0; k < 8; ++k) {
        a[2 * k] = _mm_unpacklo_epi8(r[2 * k], r[2 * k + 1]);
        a[2 * k + 1] = _mm_unpackhi_epi8(r[2 * k], r[2 * k + 1]);
    }
    for (int g = 0; g < 4; ++g) {
        b[4 * g + 0] = _mm_unpacklo_epi16(a[4 * g + 0], a[4 * g + 2]);
        b[4 * g + 1] = _mm_unpackhi_epi16(a[4 * g + 0], a[4 * g + 2]);
        b[4 * g + 2] = _mm_unpacklo_epi16(a[4 * g + 1], a[4 * g + 3]);
        b[4 * g + 3] = _mm_unpackhi_epi16(a[4 * g + 1], a[4 * g + 3]);
    }
    for (int h = 0; h < 2; ++h)
        for (int q = 0; q < 4; ++q) {
            c[8 * h + 2 * q] = _mm_unpacklo_epi32(b[8 * h + q], b[8 * h + 4 + q]);
            c[8 * h + 2 * q + 1] = _mm_unpackhi_epi32(b[8 * h + q], b[8 * h + 4 + q]);
        }
    for (int p = 0; p < 8; ++p) {
        r[2 * p] = _mm_unpacklo_epi64(c[p], c[8 + p]);
        r[2 * p + 1] = _mm_unpackhi_epi64(c[p], c[8 + p]);
    }
}

// Copy len bytes with non-temporal 16-byte stores (no read-for-ownership of
// the destination lines; the caller's rows are 4 mod 16 aligned, so the
// head and tail go through ordinary stores).
static void stream_copy(uint8_t *dst, const uint8_t *src, size_t len) {
    size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
    if (head > len) head = len;
    memcpy(dst, src, head);
    size_t i = head;
    for (; i + 16 <= len; i += 16)
        _mm_stream_si128(reinterpret_cast<__m128i *>(dst + i),
                         _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + i)));
    memcpy(dst + i, src + i, len - i);
}

// rows r0 .. r1 - 1; rows0 = the (count, ids) row of r0.  Rows are built in
// a small (L1/L2-resident) bounce buffer, eight at a time, then streamed out.
static void assemble_range(uint8_t *blocks, int64_t r0, int64_t r1, int64_t stride, int cap,
                           int m, const int32_t *rows0, const uint8_t *codes, int64_t ncodes) {
    static const uint8_t zero[128 + 16] = {0};
    constexpr int kGroup = 8;
    constexpr int64_t kPrefetch = 4;  // rows
    const int nb = (cap + 15) / 16;
    const int m16 = m & ~15;
    std::vector<uint8_t> bounce((size_t)kGroup * stride);
    for (int64_t g0 = r0; g0 < r1; g0 += kGroup) {
        const int64_t g1 = std::min<int64_t>(r1, g0 + kGroup);
        for (int64_t r = g0; r < g1; ++r) {
            const int32_t *pr = rows0 + (r - r0) * (1 + (int64_t)cap);
            // the code rows of the row kPrefetch ahead: random 64-byte reads
            // from the n x m table are what bounds this loop
            if (r + kPrefetch < r1) {
                const int32_t *pf = pr + kPrefetch * (1 + (int64_t)cap);
                const int pc = std::min(std::max(pf[0], 0), cap);
                for (int j = 0; j < pc; ++j) {
                    const int u = pf[1 + j];
                    if (u >= 0 && u < ncodes)
                        for (int l = 0; l < m; l += 64)
                            _mm_prefetch(reinterpret_cast<const char *>(codes + (size_t)u * m + l),
                                         _MM_HINT_T0);
                }
            }
            uint8_t *b = bounce.data() + (r - g0) * stride;
            memcpy(b, pr, 4 * (size_t)(1 + cap));
            const int cnt = std::min(std::max(pr[0], 0), cap);
            uint8_t *region = b + 4 + 4 * (size_t)cap;
            uint8_t *region_end = b + stride;
            for (int bt = 0; bt < nb; ++bt) {
                const uint8_t *src[16];
                for (int ln = 0; ln < 16; ++ln) {
                    const int slot = bt * 16 + ln;
                    const int u = slot < cnt ? pr[1 + slot] : -1;
                    src[ln] = (u >= 0 && u < ncodes) ? codes + (size_t)u * m : zero;
                }
                uint8_t *out = region + (size_t)bt * m * 16;
                for (int i0 = 0; i0 < m16; i0 += 16) {
                    __m128i t[16];
                    for (int ln = 0; ln < 16; ++ln)
                        t[ln] = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src[ln] + i0));
                    transpose16(t);
                    for (int k = 0; k < 16; ++k)
                        _mm_storeu_si128(reinterpret_cast<__m128i *>(out + (size_t)(i0 + k) * 16),
                                         t[k]);
                }
                for (int i = m16; i < m; ++i)
                    for (int ln = 0; ln < 16; ++ln) out[(size_t)i * 16 + ln] = src[ln][i];
            }
            // bytes past the code region (a caller's wider stride) stay zero
            uint8_t *used = region + (size_t)nb * m * 16;
            if (used < region_end) memset(used, 0, (size_t)(region_end - used));
        }
        stream_copy(blocks + g0 * stride, bounce.data(), (size_t)(g1 - g0) * stride);
    }
    _mm_sfence();
}

// Device (count, ids) rows -> host reference blocks: each staging worker
// copies a chunk of rows into its pinned buffer and assembles those rows'
// blocks straight into the caller's array (all host cores).
static int staged_assemble(uint8_t *blocks, int64_t rows, int64_t stride, int cap, int m,
                           const int32_t *dev_rows, const uint8_t *codes, int64_t ncodes) {
    if (rows == 0) return FA_OK;
    const size_t rb = 4 * (size_t)(1 + cap);
    const size_t per = std::max<size_t>(1, std::min<size_t>(stage_bytes() / rb, 16384));
    const size_t nchunk = ((size_t)rows + per - 1) / per;
    const int T = std::max(stage_workers(), std::min(32, (int)std::thread::hardware_concurrency()));
    return stage_run(
        nchunk, "block assembly",
        [&](size_t c, uint8_t *buf, cudaStream_t s) {
            const size_t r0 = c * per, r1 = std::min<size_t>((size_t)rows, r0 + per);
            cudaError_t e = cudaMemcpyAsync(buf, reinterpret_cast<const uint8_t *>(dev_rows) + r0 * rb,
                                            (r1 - r0) * rb, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e == cudaSuccess)
                assemble_range(blocks, (int64_t)r0, (int64_t)r1, stride, cap, m,
                               reinterpret_cast<const int32_t *>(buf), codes, ncodes);
            return e;
        },
        T);
}

// rows of the projected vectors uploaded before the build starts (the batch
// schedule reaches them after ~60 batches: 0.2 x inserted per batch);
// FLASHANN_B200_EARLY_ROWS overrides (tests)
static int64_t early_rows() {
    const char *e = getenv("FLASHANN_B200_EARLY_ROWS");
    const long long v = e ? atoll(e) : 0;
    return v > 0 ? (int64_t)v : (int64_t)131072;
}

struct IndexGuard {
    fa_index *ix = nullptr;
    ~IndexGuard() { fa_index_destroy(ix); }
};

}  // namespace fa

using namespace fa;

extern "C" const char *fa_last_error(void) { return g_err; }
extern "C" int fa_version(void) { return 1; }

extern "C" int fa_assemble_blocks(uint8_t *blocks, int64_t rows, int64_t stride, int cap, int m,
                                  const int32_t *id_rows, const uint8_t *codes, int64_t ncodes) {
    FA_CHECK_ARG(rows >= 0 && cap >= 1 && m >= 0 && m <= 128, "bad block arguments");
    FA_CHECK_ARG(stride >= 4 + 4 * (int64_t)cap + (int64_t)((cap + 15) / 16) * m * 16,
                 "block stride too small");
    if (rows == 0) return FA_OK;
    const int T = (int)std::min<int64_t>(
        std::max(1, std::min(32, (int)std::thread::hardware_concurrency())),
        (rows + 4095) / 4096);
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([=]() {
            const int64_t r0 = rows * t / T, r1 = rows * (t + 1) / T;
            assemble_range(blocks, r0, r1, stride, cap, m, id_rows + r0 * (1 + (int64_t)cap), codes,
                           ncodes);
        });
    for (auto &x : th) x.join();
    return FA_OK;
}

// FLASHANN_B200_TIMING=1: per-phase wall times of the host drop-ins on stderr
struct PhaseTimer {
    bool on = getenv("FLASHANN_B200_TIMING") != nullptr;
    // constructed first, destroyed last: the mark covers the buffer frees
    ~PhaseTimer() { mark("teardown (frees)"); }
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char *what) {
        if (!on) return;
        cudaDeviceSynchronize();
        auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[fa timing] %-24s %8.2f ms\n", what,
                std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

extern "C" int fa_build_graph_host(int64_t n, int dim, const float *vecs, int dproj,
                                   const float *proj, uint8_t *codes, int m, const float *cent,
                                   int dmax, const int32_t *dims, const int32_t *offs,
                                   const uint8_t *sdt, double dist_min, double delta,
                                   const int32_t *levels, uint8_t *base_blocks, int64_t base_stride,
                                   const int64_t *uoff, uint8_t *upper_blocks, int64_t n_upper_rows,
                                   int64_t upper_stride, int C, int R, const fa_build_opts *opts,
                                   fa_build_result *res) {
    (void)vecs;
    (void)dim;
    FA_CHECK_ARG(n >= 0 && m >= 1 && R >= 1, "bad sizes");
    if (n == 0) {
        memset(res, 0, sizeof(*res));
        res->entry_point = -1;
        res->max_layer = -1;
        return FA_OK;
    }
    PhaseTimer tm;
    DevBuf dproj_b, dcent, ddims, doffs, dsdt, dlev, duoff, dbase, dupper;
    // the projected vectors (the one large input) upload on a helper thread:
    // the first rows while the model and layer arrays go up and the index is
    // created, the rest while the build's first batches run (they read only
    // the first rows; the build waits for the rest before the first batch
    // that needs them)
    FA_TRY(dproj_b.alloc(sizeof(float) * n * dproj));
    const int64_t early = std::min<int64_t>(n, early_rows());
    TwoPartUpload up(proj, dproj_b.p, sizeof(float) * early * dproj, sizeof(float) * n * dproj);
    FA_TRY_JOIN(up, dcent.upload(cent, sizeof(float) * (size_t)m * 16 * dmax));
    FA_TRY_JOIN(up, ddims.upload(dims, sizeof(int32_t) * m));
    FA_TRY_JOIN(up, doffs.upload(offs, sizeof(int32_t) * m));
    FA_TRY_JOIN(up, dsdt.upload(sdt, (size_t)m * 256));
    FA_TRY_JOIN(up, dlev.upload(levels, sizeof(int32_t) * n));
    FA_TRY_JOIN(up, duoff.upload(uoff, sizeof(int64_t) * n));
    fa_index_desc d;
    memset(&d, 0, sizeof(d));
    d.n = n; d.m = m; d.R = R; d.dim = 0; d.dproj = dproj; d.dmax = dmax;
    d.dist_min = dist_min; d.delta = delta;
    d.proj = dproj_b.as<float>(); d.cent = dcent.as<float>(); d.dims = ddims.as<int32_t>();
    d.offs = doffs.as<int32_t>(); d.sdt = dsdt.as<uint8_t>(); d.levels = dlev.as<int32_t>();
    d.uoff = duoff.as<int64_t>(); d.n_upper_rows = n_upper_rows;
    tm.mark("upload model/levels");
    IndexGuard guard;
    FA_TRY_JOIN(up, fa_index_create(&d, &guard.ix));
    FA_TRY_JOIN(up, up.wait_first());
    tm.mark("uploads + index create");
    FA_TRY_JOIN(up, index_encode_rows(guard.ix, 0, early, nullptr));
    if (early < n)
        index_set_late_rows(guard.ix, early, [&up, &guard, early, n](cudaStream_t st) {
            FA_TRY(up.join());
            return index_encode_rows(guard.ix, early, n, st);
        });
    FA_TRY_JOIN(up, fa_index_build(guard.ix, opts, res, nullptr));
    FA_TRY(up.join());
    tm.mark("encode + build");
    // codes[x] as the compiled core leaves them (prep_qctx overwrite)
    int cs = 0;
    const uint8_t *dcodes = fa_index_codes(guard.ix, &cs);
    FA_CUDA(cudaMemcpy2D(codes, m, dcodes, cs, m, n, cudaMemcpyDeviceToHost));
    tm.mark("codes D2H");
    // the graph leaves as (count, ids) rows; the blocks' inline code batches
    // are written on the host from codes[] (just read back above)
    const int cap0 = 2 * R;
    FA_TRY(dbase.alloc((size_t)n * 4 * (1 + cap0)));
    FA_TRY(dupper.alloc((size_t)n_upper_rows * 4 * (1 + R)));
    FA_TRY(fa_index_export_rows(guard.ix, dbase.as<int32_t>(), dupper.as<int32_t>(), nullptr));
    FA_CUDA(cudaDeviceSynchronize());
    tm.mark("export rows");
    FA_TRY(staged_assemble(base_blocks, n, base_stride, cap0, m, dbase.as<int32_t>(), codes, n));
    if (n_upper_rows)
        FA_TRY(staged_assemble(upper_blocks, n_upper_rows, upper_stride, R, m,
                               dupper.as<int32_t>(), codes, n));
    tm.mark("rows D2H + block assembly");
    return FA_OK;
}

extern "C" int fa_search_batch_host(int64_t n, int dim, const float *vecs, int dproj,
                                    const uint8_t *codes, int m, const float *cent, int dmax,
                                    const int32_t *dims, const int32_t *offs, const uint8_t *sdt,
                                    double dist_min, double delta, const int32_t *levels,
                                    const uint8_t *base_blocks, int64_t base_stride,
                                    const int64_t *uoff, const uint8_t *upper_blocks,
                                    int64_t n_upper_rows, int64_t upper_stride, int R,
                                    int64_t entry, int max_layer, const float *queries,
                                    const float *qproj, int nq, int ef, int k, int rerank_depth,
                                    int64_t *out_ids, double *out_d, int64_t *counters) {
    if (entry < 0) {
        set_error("cannot search an empty graph");
        return FA_EEMPTY;
    }
    FA_CHECK_ARG(n > 0 && m >= 1 && R >= 1 && k >= 1, "bad sizes");
    if (nq == 0) {
        if (counters) memset(counters, 0, 4 * sizeof(int64_t));
        return FA_OK;
    }
    PhaseTimer tm;
    DevBuf dvecs, dcent, ddims, doffs, dsdt, dlev, duoff, dbase, dupper, dq, dqp, dcodes, did, dd;
    if (rerank_depth > 0) {
        FA_TRY(dvecs.upload(vecs, sizeof(float) * n * dim));
        FA_TRY(dq.upload(queries, sizeof(float) * (size_t)nq * dim));
    }
    tm.mark("upload vecs + queries");
    FA_TRY(dqp.upload(qproj, sizeof(float) * (size_t)nq * dproj));
    FA_TRY(dcent.upload(cent, sizeof(float) * (size_t)m * 16 * dmax));
    FA_TRY(ddims.upload(dims, sizeof(int32_t) * m));
    FA_TRY(doffs.upload(offs, sizeof(int32_t) * m));
    FA_TRY(dsdt.upload(sdt, (size_t)m * 256));
    FA_TRY(dlev.upload(levels, sizeof(int32_t) * n));
    FA_TRY(duoff.upload(uoff, sizeof(int64_t) * n));
    // only the count + id prefix of each reference block: the inline code
    // bytes repeat codes[] (write_code_slot, _core.pyx:414-422) and the device
    // index reads codes from its own table
    const size_t row0 = 4 + 4 * (size_t)(2 * R), rowU = 4 + 4 * (size_t)R;
    FA_CHECK_ARG(base_stride >= (int64_t)row0 && (n_upper_rows == 0 || upper_stride >= (int64_t)rowU),
                 "block stride too small");
    tm.mark("upload model/levels");
    FA_TRY(dbase.alloc((size_t)n * row0));
    FA_TRY(staged_gather_rows(dbase.p, base_blocks, n, base_stride, row0));
    FA_TRY(dupper.alloc((size_t)n_upper_rows * rowU));
    FA_TRY(staged_gather_rows(dupper.p, upper_blocks, n_upper_rows, upper_stride, rowU));
    tm.mark("gather + upload id rows");
    FA_TRY(dcodes.upload(codes, (size_t)n * m));
    tm.mark("upload codes");
    FA_TRY(did.alloc(sizeof(int64_t) * (size_t)nq * k));
    FA_TRY(dd.alloc(sizeof(double) * (size_t)nq * k));
    fa_index_desc d;
    memset(&d, 0, sizeof(d));
    d.n = n; d.m = m; d.R = R; d.dim = dim; d.dproj = dproj; d.dmax = dmax;
    d.dist_min = dist_min; d.delta = delta;
    d.vecs = dvecs.as<float>(); d.cent = dcent.as<float>(); d.dims = ddims.as<int32_t>();
    d.offs = doffs.as<int32_t>(); d.sdt = dsdt.as<uint8_t>(); d.levels = dlev.as<int32_t>();
    d.uoff = duoff.as<int64_t>(); d.n_upper_rows = n_upper_rows;
    IndexGuard guard;
    FA_TRY(fa_index_create(&d, &guard.ix));
    FA_TRY(fa_index_set_codes(guard.ix, dcodes.as<uint8_t>(), m, nullptr));
    FA_TRY(fa_index_import_blocks(guard.ix, dbase.as<uint8_t>(), (int64_t)row0,
                                  dupper.as<uint8_t>(), (int64_t)rowU, nullptr));
    tm.mark("index create + import");
    FA_TRY(fa_index_search(guard.ix, dq.as<float>(), dqp.as<float>(), nq, ef, k, rerank_depth,
                           entry, max_layer, did.as<int64_t>(), dd.as<double>(), counters,
                           nullptr));
    tm.mark("search");
    FA_CUDA(cudaMemcpy(out_ids, did.p, sizeof(int64_t) * (size_t)nq * k, cudaMemcpyDeviceToHost));
    FA_CUDA(cudaMemcpy(out_d, dd.p, sizeof(double) * (size_t)nq * k, cudaMemcpyDeviceToHost));
    return FA_OK;
}

extern "C" int fa_build_graph_exact_host(int64_t n, int dim, const float *vecs,
                                         const int32_t *levels, uint8_t *base_blocks,
                                         int64_t base_stride, const int64_t *uoff,
                                         uint8_t *upper_blocks, int64_t n_upper_rows,
                                         int64_t upper_stride, int C, int R,
                                         const fa_build_opts *opts, fa_build_result *res) {
    FA_CHECK_ARG(n >= 0 && dim >= 1 && R >= 1, "bad sizes");
    if (n == 0) {
        memset(res, 0, sizeof(*res));
        res->entry_point = -1;
        res->max_layer = -1;
        return FA_OK;
    }
    DevBuf dvecs, dlev, duoff, dbase, dupper;
    FA_TRY(dvecs.upload(vecs, sizeof(float) * n * dim));
    FA_TRY(dlev.upload(levels, sizeof(int32_t) * n));
    FA_TRY(duoff.upload(uoff, sizeof(int64_t) * n));
    fa_index_desc d;
    memset(&d, 0, sizeof(d));
    d.n = n; d.m = 0; d.R = R; d.dim = dim; d.dproj = dim;
    d.vecs = dvecs.as<float>(); d.levels = dlev.as<int32_t>(); d.uoff = duoff.as<int64_t>();
    d.n_upper_rows = n_upper_rows;
    IndexGuard guard;
    FA_TRY(fa_index_create(&d, &guard.ix));
    FA_TRY(fa_index_build(guard.ix, opts, res, nullptr));
    FA_TRY(dbase.alloc((size_t)n * base_stride));
    FA_TRY(dupper.alloc((size_t)n_upper_rows * upper_stride));
    FA_TRY(fa_index_export_blocks(guard.ix, dbase.as<uint8_t>(), base_stride, dupper.as<uint8_t>(),
                                  upper_stride, nullptr));
    FA_CUDA(cudaDeviceSynchronize());
    FA_TRY(staged_copy(base_blocks, dbase.p, (size_t)n * base_stride, true));
    if (n_upper_rows)
        FA_TRY(staged_copy(upper_blocks, dupper.p, (size_t)n_upper_rows * upper_stride, true));
    return FA_OK;
}

extern "C" int fa_search_batch_exact_host(int64_t n, int dim, const float *vecs,
                                          const int32_t *levels, const uint8_t *base_blocks,
                                          int64_t base_stride, const int64_t *uoff,
                                          const uint8_t *upper_blocks, int64_t n_upper_rows,
                                          int64_t upper_stride, int R, int64_t entry,
                                          int max_layer, const float *queries, int nq, int ef,
                                          int k, int rerank_depth, int64_t *out_ids,
                                          double *out_d, int64_t *counters) {
    if (entry < 0) {
        set_error("cannot search an empty graph");
        return FA_EEMPTY;
    }
    FA_CHECK_ARG(n > 0 && dim >= 1 && R >= 1 && k >= 1, "bad sizes");
    if (nq == 0) {
        if (counters) memset(counters, 0, 4 * sizeof(int64_t));
        return FA_OK;
    }
    DevBuf dvecs, dlev, duoff, dbase, dupper, dq, did, dd;
    FA_TRY(dvecs.upload(vecs, sizeof(float) * n * dim));
    FA_TRY(dq.upload(queries, sizeof(float) * (size_t)nq * dim));
    FA_TRY(dlev.upload(levels, sizeof(int32_t) * n));
    FA_TRY(duoff.upload(uoff, sizeof(int64_t) * n));
    FA_TRY(dbase.upload(base_blocks, (size_t)n * base_stride));
    FA_TRY(dupper.upload(upper_blocks, (size_t)n_upper_rows * upper_stride));
    FA_TRY(did.alloc(sizeof(int64_t) * (size_t)nq * k));
    FA_TRY(dd.alloc(sizeof(double) * (size_t)nq * k));
    fa_index_desc d;
    memset(&d, 0, sizeof(d));
    d.n = n; d.m = 0; d.R = R; d.dim = dim; d.dproj = dim;
    d.vecs = dvecs.as<float>(); d.levels = dlev.as<int32_t>(); d.uoff = duoff.as<int64_t>();
    d.n_upper_rows = n_upper_rows;
    IndexGuard guard;
    FA_TRY(fa_index_create(&d, &guard.ix));
    FA_TRY(fa_index_import_blocks(guard.ix, dbase.as<uint8_t>(), base_stride, dupper.as<uint8_t>(),
                                  upper_stride, nullptr));
    FA_TRY(fa_index_search(guard.ix, dq.as<float>(), dq.as<float>(), nq, ef, k, rerank_depth,
                           entry, max_layer, did.as<int64_t>(), dd.as<double>(), counters,
                           nullptr));
    FA_CUDA(cudaMemcpy(out_ids, did.p, sizeof(int64_t) * (size_t)nq * k, cudaMemcpyDeviceToHost));
    FA_CUDA(cudaMemcpy(out_d, dd.p, sizeof(double) * (size_t)nq * k, cudaMemcpyDeviceToHost));
    return FA_OK;
}
