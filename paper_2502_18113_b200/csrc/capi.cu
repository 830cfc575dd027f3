// C-ABI plumbing: error strings, version, and the host-pointer drop-ins that
// mirror the reference core's blocking Cython entry points
// (build_graph _core.pyx:711-764, search_batch _core.pyx:817-888).
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
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
static int stage_run(size_t nchunk, const char *what, F fn) {
    std::lock_guard<std::mutex> lk(g_stage_mu);  // one staged copy at a time
    const size_t kStageBytes = stage_bytes();
    const int T = (int)std::min<size_t>(stage_workers(), nchunk);
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

struct IndexGuard {
    fa_index *ix = nullptr;
    ~IndexGuard() { fa_index_destroy(ix); }
};

}  // namespace fa

using namespace fa;

extern "C" const char *fa_last_error(void) { return g_err; }
extern "C" int fa_version(void) { return 1; }

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
    // the projected vectors (the one large input) upload on a helper thread
    // while the model and layer arrays go up and the index is created
    FA_TRY(dproj_b.alloc(sizeof(float) * n * dproj));
    AsyncUpload up(proj, dproj_b.p, sizeof(float) * n * dproj);
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
    FA_TRY(up.join());
    tm.mark("uploads + index create");
    FA_TRY(fa_index_encode(guard.ix, nullptr));
    FA_TRY(fa_index_build(guard.ix, opts, res, nullptr));
    tm.mark("encode + build");
    // codes[x] as the compiled core leaves them (prep_qctx overwrite)
    int cs = 0;
    const uint8_t *dcodes = fa_index_codes(guard.ix, &cs);
    FA_CUDA(cudaMemcpy2D(codes, m, dcodes, cs, m, n, cudaMemcpyDeviceToHost));
    tm.mark("codes D2H");
    FA_TRY(dbase.alloc((size_t)n * base_stride));
    FA_TRY(dupper.alloc((size_t)n_upper_rows * upper_stride));
    FA_TRY(fa_index_export_blocks(guard.ix, dbase.as<uint8_t>(), base_stride, dupper.as<uint8_t>(),
                                  upper_stride, nullptr));
    FA_CUDA(cudaDeviceSynchronize());
    tm.mark("export");
    FA_TRY(staged_copy(base_blocks, dbase.p, (size_t)n * base_stride, true));
    if (n_upper_rows)
        FA_TRY(staged_copy(upper_blocks, dupper.p, (size_t)n_upper_rows * upper_stride, true));
    tm.mark("blocks D2H");
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
