#include <cstdlib>
#include <atomic>
// extern "C" boundary (include/sparseoracle_b200.h): argument validation with
// the reference's error types/messages, H2D/D2H staging between the
// reference's host layout (int64 indices, row-major ELL) and the device
// layout, and the per-device context.
#include <algorithm>
#include <chrono>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "features.cuh"
#include "forest.cuh"

namespace sob {

// model.cu
so_forest* forest_upload(int32_t kind, int32_t n_trees, const int64_t* node_off, const int32_t* feature,
                         const double* threshold, const int32_t* left, const int32_t* right, const int32_t* cls,
                         cudaStream_t s);
void predict_rows(const so_forest& f, const double* rows_dev, int64_t n, int32_t* out_dev, cudaStream_t s);
void predict_rows_blocked(const so_forest& f, const double* rows_dev, int64_t n, int32_t* out_dev, cudaStream_t s);
void enqueue_tune_predict(const so_forest& f, const FeatState* st, const so_conversion_config& cfg, int active,
                          so_tune_outcome* out_dev, cudaStream_t s);

struct TunePlan {
    uint64_t forest_uid = 0;
    so_conversion_config cfg{};
    FeatState* st = nullptr;
    so_tune_outcome* out = nullptr;      // pinned, mapped: the predict kernel writes it over the link
    so_tune_outcome* out_dev = nullptr;  // device view of `out`
    cudaEvent_t e0 = nullptr, e1 = nullptr;  // plan build: timing the two CSR sweeps
    // private stream the graph is captured and replayed on: a capture on the
    // shared context stream would swallow other threads' work (and the
    // replay would re-run it); nothing but this plan ever uses it
    cudaStream_t ps = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::unique_ptr<FeatWorkspace> ws;
    bool matches(uint64_t uid, const so_conversion_config& c) const {
        return uid == forest_uid && c.kh_override == cfg.kh_override && c.true_diag_ratio == cfg.true_diag_ratio &&
               c.max_padding_factor == cfg.max_padding_factor && c.max_padded_entries == cfg.max_padded_entries;
    }
};

void destroy_tune_plan(TunePlan* p) {
    if (!p) return;
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->st) cudaFree(p->st);
    if (p->out) cudaFreeHost(p->out);
    if (p->e0) cudaEventDestroy(p->e0);
    if (p->e1) cudaEventDestroy(p->e1);
    p->ws.reset();
    if (p->ps) cudaStreamDestroy(p->ps);
    delete p;
}

namespace {
thread_local std::string g_err;
std::mutex g_mu;
Context g_ctx[64];
bool g_ready[64];
thread_local int g_dev = -1;
}  // namespace

void set_error(const std::string& m) { g_err = m; }

Context& ctx(int d) {
    if (d < 0 || d >= 64) fail(SO_INVALID_INPUT, "bad device ordinal");
    std::lock_guard<std::mutex> lk(g_mu);
    Context& c = g_ctx[d];
    if (!g_ready[d]) {
        SOB_CUDA(cudaSetDevice(d));
        c.device = d;
        SOB_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
        SOB_CUDA(cudaStreamCreateWithFlags(&c.copy_in, cudaStreamNonBlocking));
        SOB_CUDA(cudaStreamCreateWithFlags(&c.copy_out, cudaStreamNonBlocking));
        SOB_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, d));
        int l2 = 0;
        SOB_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, d));
        c.l2_bytes = l2;
        // keep freed pool memory cached: conversions and scratch are stream-
        // ordered allocations, reuse must not go back to the driver
        cudaMemPool_t pool;
        SOB_CUDA(cudaDeviceGetDefaultMemPool(&pool, d));
        uint64_t thresh = UINT64_MAX;
        SOB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
        g_ready[d] = true;
    }
    return c;
}

Context& current_ctx() {
    if (g_dev < 0) {
        int d = 0;
        SOB_CUDA(cudaGetDevice(&d));
        g_dev = d;
    }
    SOB_CUDA(cudaSetDevice(g_dev));
    return ctx(g_dev);
}

namespace {

// ------------------------------------------------------------ staging kernels

__global__ void narrow_idx(const int64_t* __restrict__ in, int32_t* __restrict__ out, int64_t n, int64_t hi,
                           int allow_sentinel, int* __restrict__ bad) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t v = in[i];
    const bool ok = (v >= 0 && v < hi) || (allow_sentinel && v == -1);
    if (!ok) atomicExch(bad, 1);
    out[i] = int32_t(v);
}

__global__ void widen_idx(const int32_t* __restrict__ in, int64_t* __restrict__ out, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i];
}

// row-major [n][K] (int64 / f64) <-> column-major [K][n] (int32 / f64)
__global__ void ell_to_colmajor(const int64_t* __restrict__ col_rm, const double* __restrict__ val_rm, int64_t n,
                                int64_t K, int64_t ncols, int32_t* __restrict__ col_cm, double* __restrict__ val_cm,
                                int* __restrict__ bad) {
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // row-major index
    if (idx >= n * K) return;
    const int64_t i = idx / K, k = idx - i * K;
    const int64_t c = col_rm[idx];
    if (!((c >= 0 && c < ncols) || c == -1)) atomicExch(bad, 1);
    col_cm[k * n + i] = int32_t(c);
    val_cm[k * n + i] = val_rm[idx];
}

__global__ void ell_to_rowmajor(const int32_t* __restrict__ col_cm, const double* __restrict__ val_cm, int64_t n,
                                int64_t K, int64_t* __restrict__ col_rm, double* __restrict__ val_rm) {
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // column-major index
    if (idx >= n * K) return;
    const int64_t k = idx / n, i = idx - k * n;
    col_rm[i * K + k] = col_cm[idx];
    val_rm[i * K + k] = val_cm[idx];
}

__global__ void check_row_ptr(const int64_t* __restrict__ rp, int64_t n, int64_t nnz, int* __restrict__ bad) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i > n) return;
    if (i == 0 && rp[0] != 0) atomicExch(bad, 1);
    if (i == n && rp[n] != nnz) atomicExch(bad, 1);
    if (i < n && rp[i + 1] < rp[i]) atomicExch(bad, 1);
}

__global__ void check_cols(const int32_t* __restrict__ col, int64_t n, int64_t ncols, int* __restrict__ bad) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && (col[i] < 0 || col[i] >= ncols)) atomicExch(bad, 1);
}

__global__ void ell_short_rows(const int32_t* __restrict__ col_cm, int64_t n, int64_t K,
                               unsigned long long* __restrict__ out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    bool s = i < n && K > 0 && col_cm[(K - 1) * n + i] == -1;
    const unsigned b = __ballot_sync(0xffffffffu, s);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(out, (unsigned long long)__popc(b));
}

unsigned grid1(int64_t n) { return unsigned(ceil_div(n > 0 ? n : 1, 256)); }

void check_dims(int64_t nrows, int64_t ncols) {
    if (nrows < 0 || ncols < 0) fail(SO_INVALID_INPUT, "negative dimension");
    if (nrows >= (int64_t(1) << 31) || ncols >= (int64_t(1) << 31) || nrows + ncols >= (int64_t(1) << 31))
        fail(SO_INVALID_INPUT, "device layout needs nrows + ncols < 2^31");
}

template <typename T>
void h2d(DBuf<T>& buf, const T* src, int64_t n, cudaStream_t s) {
    buf.alloc(n, s);
    if (n > 0) {
        if (!src) fail(SO_INVALID_INPUT, "null host array");
        SOB_CUDA(cudaMemcpyAsync(buf.get(), src, sizeof(T) * size_t(n), cudaMemcpyHostToDevice, s));
    }
}

template <typename T>
void d2h(T* dst, const DBuf<T>& buf, int64_t n, cudaStream_t s) {
    if (n > 0 && dst) SOB_CUDA(cudaMemcpyAsync(dst, buf.get(), sizeof(T) * size_t(n), cudaMemcpyDeviceToHost, s));
}

struct BadFlag {
    DBuf<int> f;
    cudaStream_t s;
    explicit BadFlag(cudaStream_t st) : f(1, st), s(st) { SOB_CUDA(cudaMemsetAsync(f.get(), 0, sizeof(int), s)); }
    int* get() { return f.get(); }
    void raise_if(so_status st, const char* msg) {
        if (d2h_scalar(f.get(), s)) fail(st, msg);
    }
};

void upload_idx(DBuf<int32_t>& out, const int64_t* src, int64_t n, int64_t hi, bool sentinel, BadFlag& bad,
                cudaStream_t s) {
    DBuf<int64_t> stage;
    h2d(stage, src, n, s);
    out.alloc(n, s);
    if (n > 0) {
        narrow_idx<<<grid1(n), 256, 0, s>>>(stage.get(), out.get(), n, hi, sentinel ? 1 : 0, bad.get());
        SOB_LAUNCH("narrow_idx");
    }
}

void download_idx(int64_t* dst, const DBuf<int32_t>& src, int64_t n, cudaStream_t s) {
    if (n <= 0 || !dst) return;
    DBuf<int64_t> stage(n, s);
    widen_idx<<<grid1(n), 256, 0, s>>>(src.get(), stage.get(), n);
    SOB_LAUNCH("widen_idx");
    d2h(dst, stage, n, s);
    SOB_CUDA(cudaStreamSynchronize(s));
}

void upload_csr_part(CsrPart& c, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rp, const int64_t* col,
                     const double* val, cudaStream_t s) {
    BadFlag bad(s);
    c.nnz = nnz;
    h2d(c.row_ptr, rp, nrows + 1, s);
    check_row_ptr<<<grid1(nrows + 1), 256, 0, s>>>(c.row_ptr.get(), nrows, nnz, bad.get());
    SOB_LAUNCH("check_row_ptr");
    upload_idx(c.col, col, nnz, ncols, false, bad, s);
    h2d(c.val, val, nnz, s);
    bad.raise_if(SO_INVALID_INPUT, "CSR arrays inconsistent (row_ptr or column index out of range)");
    build_row_blocks(c, nrows, s);
}

void upload_dia_part(DiaPart& d, int64_t nrows, int64_t ncols, int64_t ndiags, const int64_t* offsets,
                     const double* values, int64_t stored, cudaStream_t s) {
    for (int64_t k = 0; k < ndiags; ++k) {
        if (offsets[k] < -(nrows - 1) || offsets[k] > ncols - 1)
            fail(SO_INVALID_INPUT, "DIA offset outside [-(nrows-1), ncols-1]");
        if (k > 0 && offsets[k] <= offsets[k - 1]) fail(SO_INVALID_INPUT, "DIA offsets must be strictly increasing");
    }
    d.ndiags = ndiags;
    d.stored_nnz = stored;
    h2d(d.offsets, offsets, ndiags, s);
    h2d(d.values, values, ndiags * nrows, s);
}

void upload_ell_part(EllPart& e, int64_t nrows, int64_t ncols, int64_t width, const int64_t* col, const double* val,
                     int64_t stored, cudaStream_t s) {
    BadFlag bad(s);
    e.width = width;
    e.stored_nnz = stored;
    DBuf<int64_t> scol;
    DBuf<double> sval;
    h2d(scol, col, nrows * width, s);
    h2d(sval, val, nrows * width, s);
    e.col.alloc(nrows * width, s);
    e.val.alloc(nrows * width, s);
    if (nrows * width > 0) {
        ell_to_colmajor<<<grid1(nrows * width), 256, 0, s>>>(scol.get(), sval.get(), nrows, width, ncols, e.col.get(),
                                                             e.val.get(), bad.get());
        SOB_LAUNCH("ell_to_colmajor");
    }
    bad.raise_if(SO_INVALID_INPUT, "ELL column index out of range");
}

void upload_coo_part(CooPart& c, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* row, const int64_t* col,
                     const double* val, cudaStream_t s) {
    BadFlag bad(s);
    c.nnz = nnz;
    upload_idx(c.row, row, nnz, nrows, false, bad, s);
    upload_idx(c.col, col, nnz, ncols, false, bad, s);
    h2d(c.val, val, nnz, s);
    bad.raise_if(SO_INVALID_INPUT, "COO index out of range");
}

so_matrix* new_host_matrix(int32_t fmt, int64_t nrows, int64_t ncols) {
    check_dims(nrows, ncols);
    Context& c = current_ctx();
    auto* m = new so_matrix();
    m->device = c.device;
    m->format = fmt;
    m->nrows = nrows;
    m->ncols = ncols;
    return m;
}

cudaStream_t on_device(const so_matrix* m) {
    if (!m) fail(SO_INVALID_INPUT, "null matrix");
    SOB_CUDA(cudaSetDevice(m->device));
    g_dev = m->device;
    return ctx(m->device).stream;
}

template <typename F>
so_status make(so_matrix** out, F&& f) {
    return guard([&] {
        if (!out) fail(SO_INVALID_INPUT, "null out pointer");
        *out = nullptr;
        std::unique_ptr<so_matrix> m(f());
        SOB_CUDA(cudaStreamSynchronize(ctx(m->device).stream));
        *out = m.release();
    });
}

so_conversion_config cfg_or_default(const so_conversion_config* c) {
    if (c) return *c;
    return so_conversion_config{0, 0.2, 10.0, 0};
}

void check_ratio(const so_matrix& m, double ratio) {  // features.cpp:86-91
    if (m.nrows < 1 || m.ncols < 1) fail(SO_EMPTY_MATRIX, "extract_features: matrix has a zero dimension");
    if (!(ratio > 0.0) || ratio > 1.0) fail(SO_INVALID_INPUT, "extract_features: true_diag_ratio must be in (0, 1]");
}

void check_x(const so_matrix& m, int64_t xlen) {  // spmv.cpp:12-19
    if (xlen != m.ncols)
        fail(SO_DIMENSION_MISMATCH, "spmv: vector length " + std::to_string(xlen) + " does not match ncols " +
                                        std::to_string(m.ncols));
}

}  // namespace

static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace sob

namespace sob {
namespace {

// events owned by a scope (or a thread): destroyed on every exit path
struct EventSet {
    std::vector<cudaEvent_t> ev;
    unsigned flags;
    EventSet(size_t n, unsigned f) : flags(f) { grow(n); }
    void grow(size_t n) {
        while (ev.size() < n) {
            cudaEvent_t e;
            SOB_CUDA(cudaEventCreateWithFlags(&e, flags));
            ev.push_back(e);
        }
    }
    ~EventSet() {
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
    }
    EventSet(const EventSet&) = delete;
    EventSet& operator=(const EventSet&) = delete;
};

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// device-visible address of pinned, mapped host memory (UVA: usually p itself), else null
const void* mapped_ptr(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// Row-chunk pipeline of spmv(m, x) for matrices whose rows only read a known
// column window (DIA, HDC with an empty CSR part): x is uploaded in the
// windows the chunks need (copy engine, copy_in), chunk k's rows run on the
// compute stream as soon as its window has landed, and chunk k's y is read
// back on copy_out while later chunks upload and compute -- the host<->device
// transfers of both directions overlap each other and the kernels.  Results
// are identical to the one-shot path (same kernel per row).
constexpr int64_t kPipeRows = 1 << 18;

}  // namespace

void ensure_dia_window(const so_matrix& m, cudaStream_t s) {
    if (m.dia_window_known.load(std::memory_order_acquire) || m.dia.ndiags == 0) return;
    std::vector<int64_t> off(size_t(m.dia.ndiags));
    d2h(off.data(), m.dia.offsets, m.dia.ndiags, s);
    SOB_CUDA(cudaStreamSynchronize(s));
    m.dia_omin.store(*std::min_element(off.begin(), off.end()), std::memory_order_relaxed);
    m.dia_omax.store(*std::max_element(off.begin(), off.end()), std::memory_order_relaxed);
    m.dia_window_known.store(true, std::memory_order_release);
}

namespace {

bool spmv_pipelined(const so_matrix& m, const double* x, double* y, cudaStream_t s) {
    const bool dia_only = m.format == SO_DIA || (m.format == SO_HDC && m.csr.nnz == 0);
    if (!dia_only || m.dia.ndiags == 0 || m.nrows < 2 * kPipeRows) return false;
    // y overlapping x (in-place calls through the C-ABI): x must be read in
    // full before any y lands -- the one-shot path does exactly that
    const auto xa = reinterpret_cast<uintptr_t>(x), ya = reinterpret_cast<uintptr_t>(y);
    if (xa < ya + sizeof(double) * size_t(m.nrows) && ya < xa + sizeof(double) * size_t(m.ncols)) return false;
    if (!is_pinned(x) || !is_pinned(y)) return false;
    ensure_dia_window(m, s);
    // narrow windows: one kernel over the host link, no copy engine
    static const bool zc_off = std::getenv("SOB_NO_ZERO_COPY") != nullptr;  // diagnostic knob
    if (!zc_off) {
        const double* xm = static_cast<const double*>(mapped_ptr(x));
        double* ym = static_cast<double*>(const_cast<void*>(mapped_ptr(y)));
        // x up on the copy engine with the kernel following it, y over the SMs
        // (config 2: 0.87 -> 0.70 ms per call); else x and y both over the SMs
        if (ym && spmv_dia_follow(m, x, ym, s, ctx(m.device).copy_in)) return true;
        if (xm && ym && spmv_dia_zero_copy(m, xm, ym, s)) return true;
    }
    Context& c = ctx(m.device);
    const int64_t n = m.nrows, nc = m.ncols;
    static const int64_t max_chunks = [] {
        const char* e = std::getenv("SOB_PIPE_CHUNKS");  // tuning knob (default 16)
        return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t(16);
    }();
    const int64_t nchunks = std::min<int64_t>(max_chunks, ceil_div(n, kPipeRows));
    const int64_t rows_per = ceil_div(n, nchunks);
    DBuf<double> dx(nc, s), dy(n, s);
    thread_local EventSet pool(0, cudaEventDisableTiming);
    pool.grow(size_t(2 * nchunks + 1));
    std::vector<cudaEvent_t>& ev = pool.ev;
    // buffers come from the compute stream's pool: the copy streams wait on it
    SOB_CUDA(cudaEventRecord(ev[0], s));
    SOB_CUDA(cudaStreamWaitEvent(c.copy_in, ev[0], 0));
    SOB_CUDA(cudaStreamWaitEvent(c.copy_out, ev[0], 0));
    // every x window goes up first (the copy engine never waits on the host
    // enqueueing kernels and read-backs), then chunk k's rows run as soon as
    // their window has landed and chunk k's y goes down behind them
    int64_t x_hi = 0;
    for (int64_t k = 0; k < nchunks; ++k) {
        const int64_t a = k * rows_per, b = std::min(n, a + rows_per);
        if (a >= b) break;
        const int64_t need = std::min(nc, std::max<int64_t>(0, b + m.dia_omax));
        const int64_t want = k + 1 == nchunks ? nc : need;
        if (want > x_hi) {
            SOB_CUDA(cudaMemcpyAsync(dx.get() + x_hi, x + x_hi, sizeof(double) * size_t(want - x_hi),
                                     cudaMemcpyHostToDevice, c.copy_in));
            x_hi = want;
        }
        SOB_CUDA(cudaEventRecord(ev[1 + 2 * k], c.copy_in));
    }
    for (int64_t k = 0; k < nchunks; ++k) {
        const int64_t a = k * rows_per, b = std::min(n, a + rows_per);
        if (a >= b) break;
        SOB_CUDA(cudaStreamWaitEvent(s, ev[1 + 2 * k], 0));
        spmv_device_rows(m, dx.get(), dy.get(), a, b, s);
        SOB_CUDA(cudaEventRecord(ev[2 + 2 * k], s));
        SOB_CUDA(cudaStreamWaitEvent(c.copy_out, ev[2 + 2 * k], 0));
        SOB_CUDA(cudaMemcpyAsync(y + a, dy.get() + a, sizeof(double) * size_t(b - a), cudaMemcpyDeviceToHost,
                                 c.copy_out));
    }
    // the buffers are released on s: order s after the last read-back
    SOB_CUDA(cudaEventRecord(ev[0], c.copy_out));
    SOB_CUDA(cudaStreamWaitEvent(s, ev[0], 0));
    return true;
}

}  // namespace
}  // namespace sob

using namespace sob;

extern "C" {

const char* so_last_error(void) { return g_err.c_str(); }
const char* so_version(void) { return "sparseoracle-b200 0.1 (sm_100a)"; }

int64_t so_kernel_launches(void) { return sob::g_launches.load(std::memory_order_relaxed); }

so_status so_set_device(int device) {
    return guard([&] {
        SOB_CUDA(cudaSetDevice(device));
        g_dev = device;
        ctx(device);
    });
}

so_status so_get_device(int* device) {
    return guard([&] {
        if (!device) fail(SO_INVALID_INPUT, "null out pointer");
        *device = current_ctx().device;
    });
}

so_status so_device_sync(void) {
    return guard([&] { SOB_CUDA(cudaStreamSynchronize(current_ctx().stream)); });
}

void* so_default_stream(void) {
    try {
        return reinterpret_cast<void*>(current_ctx().stream);
    } catch (...) {
        return nullptr;
    }
}

// ---------------------------------------------------------------- uploads

so_status so_matrix_upload_coo(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* row, const int64_t* col,
                               const double* val, so_matrix** out) {
    return make(out, [&] {
        SOB_RANGE("so_matrix_upload_coo");
        std::unique_ptr<so_matrix> m(new_host_matrix(SO_COO, nrows, ncols));
        upload_coo_part(m->coo, nrows, ncols, nnz, row, col, val, ctx(m->device).stream);
        return m.release();
    });
}

so_status so_matrix_upload_csr(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* row_ptr, const int64_t* col,
                               const double* val, so_matrix** out) {
    return make(out, [&] {
        SOB_RANGE("so_matrix_upload_csr");
        std::unique_ptr<so_matrix> m(new_host_matrix(SO_CSR, nrows, ncols));
        upload_csr_part(m->csr, nrows, ncols, nnz, row_ptr, col, val, ctx(m->device).stream);
        return m.release();
    });
}

so_status so_matrix_upload_dia(int64_t nrows, int64_t ncols, int64_t ndiags, const int64_t* offsets,
                               const double* values, int64_t stored_nnz, so_matrix** out) {
    return make(out, [&] {
        SOB_RANGE("so_matrix_upload_dia");
        std::unique_ptr<so_matrix> m(new_host_matrix(SO_DIA, nrows, ncols));
        upload_dia_part(m->dia, nrows, ncols, ndiags, offsets, values, stored_nnz, ctx(m->device).stream);
        return m.release();
    });
}

so_status so_matrix_upload_ell(int64_t nrows, int64_t ncols, int64_t width, const int64_t* col, const double* val,
                               int64_t stored_nnz, so_matrix** out) {
    return make(out, [&] {
        SOB_RANGE("so_matrix_upload_ell");
        std::unique_ptr<so_matrix> m(new_host_matrix(SO_ELL, nrows, ncols));
        upload_ell_part(m->ell, nrows, ncols, width, col, val, stored_nnz, ctx(m->device).stream);
        return m.release();
    });
}

so_status so_matrix_upload_hyb(int64_t nrows, int64_t ncols, int64_t width, const int64_t* ell_col,
                               const double* ell_val, int64_t ell_stored_nnz, int64_t coo_nnz, const int64_t* coo_row,
                               const int64_t* coo_col, const double* coo_val, int64_t kh, so_matrix** out) {
    return make(out, [&] {
        SOB_RANGE("so_matrix_upload_hyb");
        std::unique_ptr<so_matrix> m(new_host_matrix(SO_HYB, nrows, ncols));
        cudaStream_t s = ctx(m->device).stream;
        upload_ell_part(m->ell, nrows, ncols, width, ell_col, ell_val, ell_stored_nnz, s);
        upload_coo_part(m->coo, nrows, ncols, coo_nnz, coo_row, coo_col, coo_val, s);
        m->kh = kh;
        return m.release();
    });
}

so_status so_matrix_upload_hdc(int64_t nrows, int64_t ncols, int64_t ndiags, const int64_t* offsets,
                               const double* values, int64_t dia_stored_nnz, int64_t csr_nnz, const int64_t* row_ptr,
                               const int64_t* col, const double* val, int64_t threshold, so_matrix** out) {
    return make(out, [&] {
        SOB_RANGE("so_matrix_upload_hdc");
        std::unique_ptr<so_matrix> m(new_host_matrix(SO_HDC, nrows, ncols));
        cudaStream_t s = ctx(m->device).stream;
        upload_dia_part(m->dia, nrows, ncols, ndiags, offsets, values, dia_stored_nnz, s);
        upload_csr_part(m->csr, nrows, ncols, csr_nnz, row_ptr, col, val, s);
        m->threshold = threshold;
        return m.release();
    });
}

so_status so_coo_from_triplets(int64_t nrows, int64_t ncols, int64_t n, const int64_t* row, const int64_t* col,
                               const double* val, so_matrix** out) {
    return make(out, [&] {
        SOB_RANGE("so_coo_from_triplets");
        check_dims(nrows, ncols);
        if (n > 0 && (!row || !col || !val)) fail(SO_INVALID_INPUT, "null host array");
        return coo_from_triplets_device(nrows, ncols, n, row, col, val, current_ctx().stream);
    });
}

so_status so_read_matrix_market(const char* path, so_matrix** out) {
    return make(out, [&] {
        SOB_RANGE("so_read_matrix_market");
        if (!path) fail(SO_INVALID_INPUT, "null path");
        return read_matrix_market(std::string(path), current_ctx().stream);
    });
}

so_status so_write_matrix_market(const so_matrix* m, const char* path) {
    return guard([&] {
        SOB_RANGE("so_write_matrix_market");
        if (!path) fail(SO_INVALID_INPUT, "null path");
        cudaStream_t s = on_device(m);
        if (m->format != SO_COO) fail(SO_INVALID_INPUT, "write_matrix_market: expects a COO matrix");
        if (!coo_is_canonical(*m, s)) fail(SO_INVALID_INPUT, "write_matrix_market: matrix is not canonical");
        const int64_t z = m->coo.nnz;
        std::vector<int32_t> r32(static_cast<size_t>(z)), c32(static_cast<size_t>(z));
        std::vector<double> v(static_cast<size_t>(z));
        d2h(r32.data(), m->coo.row, z, s);
        d2h(c32.data(), m->coo.col, z, s);
        d2h(v.data(), m->coo.val, z, s);
        SOB_CUDA(cudaStreamSynchronize(s));
        std::vector<int64_t> r(r32.begin(), r32.end()), c(c32.begin(), c32.end());
        write_matrix_market(m->nrows, m->ncols, z, r.data(), c.data(), v.data(), std::string(path));
    });
}

so_status so_matrix_import_csr_device(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* row_ptr_dev,
                                      const int32_t* col_dev, const double* val_dev, so_matrix** out) {
    return make(out, [&] {
        std::unique_ptr<so_matrix> m(new_host_matrix(SO_CSR, nrows, ncols));
        cudaStream_t s = ctx(m->device).stream;
        CsrPart& c = m->csr;
        c.nnz = nnz;
        c.row_ptr.alloc(nrows + 1, s);
        c.col.alloc(nnz, s);
        c.val.alloc(nnz, s);
        SOB_CUDA(cudaMemcpyAsync(c.row_ptr.get(), row_ptr_dev, c.row_ptr.bytes(), cudaMemcpyDeviceToDevice, s));
        if (nnz > 0) {
            SOB_CUDA(cudaMemcpyAsync(c.col.get(), col_dev, c.col.bytes(), cudaMemcpyDeviceToDevice, s));
            SOB_CUDA(cudaMemcpyAsync(c.val.get(), val_dev, c.val.bytes(), cudaMemcpyDeviceToDevice, s));
        }
        BadFlag bad(s);
        check_row_ptr<<<grid1(nrows + 1), 256, 0, s>>>(c.row_ptr.get(), nrows, nnz, bad.get());
        SOB_LAUNCH("check_row_ptr");
        if (nnz > 0) {
            check_cols<<<grid1(nnz), 256, 0, s>>>(c.col.get(), nnz, ncols, bad.get());
            SOB_LAUNCH("check_cols");
        }
        bad.raise_if(SO_INVALID_INPUT, "device CSR arrays inconsistent (row_ptr or column index out of range)");
        build_row_blocks(c, nrows, s);
        return m.release();
    });
}

void so_matrix_free(so_matrix* m) {
    if (!m) return;
    try {
        cudaSetDevice(m->device);
    } catch (...) {
    }
    delete m;
}

so_status so_matrix_info_get(const so_matrix* m, so_matrix_info* out) {
    return guard([&] {
        if (!m || !out) fail(SO_INVALID_INPUT, "null argument");
        out->format = m->format;
        out->device = m->device;
        out->nrows = m->nrows;
        out->ncols = m->ncols;
        out->nnz = m->nnz();
        out->coo_nnz = m->coo.nnz;
        out->csr_nnz = m->csr.nnz;
        out->ndiags = m->dia.ndiags;
        out->dia_stored_nnz = m->dia.stored_nnz;
        out->ell_width = m->ell.width;
        out->ell_stored_nnz = m->ell.stored_nnz;
        out->kh = m->kh;
        out->true_diag_threshold = m->threshold;
    });
}

so_status so_matrix_download(const so_matrix* m, const so_host_arrays* a) {
    return guard([&] {
        SOB_RANGE("so_matrix_download");
        if (!a) fail(SO_INVALID_INPUT, "null host arrays");
        cudaStream_t s = on_device(m);
        const int64_t n = m->nrows;
        const bool coo = m->format == SO_COO || m->format == SO_HYB;
        const bool csr = m->format == SO_CSR || m->format == SO_HDC;
        const bool dia = m->format == SO_DIA || m->format == SO_HDC;
        const bool ell = m->format == SO_ELL || m->format == SO_HYB;
        if (coo) {
            download_idx(a->coo_row, m->coo.row, m->coo.nnz, s);
            download_idx(a->coo_col, m->coo.col, m->coo.nnz, s);
            d2h(a->coo_val, m->coo.val, m->coo.nnz, s);
        }
        if (csr) {
            d2h(a->csr_row_ptr, m->csr.row_ptr, n + 1, s);
            download_idx(a->csr_col, m->csr.col, m->csr.nnz, s);
            d2h(a->csr_val, m->csr.val, m->csr.nnz, s);
        }
        if (dia) {
            d2h(a->dia_offsets, m->dia.offsets, m->dia.ndiags, s);
            d2h(a->dia_values, m->dia.values, m->dia.ndiags * n, s);
        }
        if (ell) {
            const int64_t tot = n * m->ell.width;
            if (tot > 0 && (a->ell_col || a->ell_val)) {
                DBuf<int64_t> c(tot, s);
                DBuf<double> v(tot, s);
                ell_to_rowmajor<<<grid1(tot), 256, 0, s>>>(m->ell.col.get(), m->ell.val.get(), n, m->ell.width, c.get(),
                                                           v.get());
                SOB_LAUNCH("ell_to_rowmajor");
                d2h(a->ell_col, c, tot, s);
                d2h(a->ell_val, v, tot, s);
                SOB_CUDA(cudaStreamSynchronize(s));
            }
        }
        SOB_CUDA(cudaStreamSynchronize(s));
    });
}

// ------------------------------------------------------------ conversions

so_status so_from_coo(const so_matrix* coo, int32_t target, const so_conversion_config* cfg, so_matrix** out) {
    return make(out, [&]() -> so_matrix* {
        SOB_RANGE("so_from_coo");
        cudaStream_t s = on_device(coo);
        if (coo->format != SO_COO) fail(SO_INVALID_INPUT, "from_coo: source is not a COO matrix");
        if (target < 0 || target > 5)
            fail(SO_INVALID_INPUT, "format id " + std::to_string(target) + " outside 0..5");
        if (!coo_is_canonical(*coo, s)) fail(SO_INVALID_INPUT, "from_coo: source matrix is not canonical COO");
        if (target == SO_COO) return clone_matrix(*coo, s);
        std::unique_ptr<so_matrix> csr(coo_to_csr_device(*coo, s));
        if (target == SO_CSR) return csr.release();
        so_matrix* r = csr_to_format(*csr, target, cfg_or_default(cfg), s);
        SOB_CUDA(cudaStreamSynchronize(s));
        return r;
    });
}

so_status so_convert(const so_matrix* src, int32_t target, const so_conversion_config* cfg, so_matrix** out) {
    return make(out, [&]() -> so_matrix* {
        SOB_RANGE("so_convert");
        cudaStream_t s = on_device(src);
        if (target < 0 || target > 5)
            fail(SO_INVALID_INPUT, "format id " + std::to_string(target) + " outside 0..5");
        if (src->format == target) return clone_matrix(*src, s);
        if (src->format == SO_CSR && csr_rows_canonical(*src, s)) {
            so_matrix* r = csr_to_format(*src, target, cfg_or_default(cfg), s);  // no canonicalizing copy
            SOB_CUDA(cudaStreamSynchronize(s));
            return r;
        }
        std::unique_ptr<so_matrix> csr(any_to_csr(*src, s));
        if (target == SO_CSR) return csr.release();
        so_matrix* r = csr_to_format(*csr, target, cfg_or_default(cfg), s);
        SOB_CUDA(cudaStreamSynchronize(s));
        return r;
    });
}

so_status so_to_coo(const so_matrix* src, so_matrix** out) {
    return make(out, [&]() -> so_matrix* {
        SOB_RANGE("so_to_coo");
        cudaStream_t s = on_device(src);
        if (src->format == SO_COO) return clone_matrix(*src, s);  // formats.cpp:436-437
        std::unique_ptr<so_matrix> csr(any_to_csr(*src, s));
        so_matrix* r = csr_to_coo(*csr, s);
        SOB_CUDA(cudaStreamSynchronize(s));
        return r;
    });
}

int32_t so_format_feasible(int32_t target, const so_feature_vector* f, const so_conversion_config* cfgp) {
    const so_conversion_config cfg = cfg_or_default(cfgp);
    const int64_t cap = padded_entry_cap(cfg, f->nnz);  // tuners.cpp:26-45
    switch (target) {
        case SO_COO:
        case SO_CSR:
            return 1;
        case SO_DIA:
            return f->ndiags * f->nrows <= cap;
        case SO_ELL:
            return f->max_nnz_per_row * f->nrows <= cap;
        case SO_HYB: {
            const int64_t kh = effective_kh(cfg, f->nnz, f->nrows);
            return std::min(kh, f->max_nnz_per_row) * f->nrows <= cap;
        }
        case SO_HDC:
            return f->ntrue_diags * f->nrows <= cap;
    }
    return 0;
}

// ------------------------------------------------------------------ SpMV

so_status so_spmv_device(const so_matrix* m, const double* x_dev, double* y_dev, void* stream) {
    return guard([&] {
        SOB_RANGE("so_spmv_device");
        on_device(m);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx(m->device).stream;
        spmv_device(*m, x_dev, y_dev, s);
    });
}

so_status so_spmv_device_rows(const so_matrix* m, const double* x_dev, double* y_dev, int64_t row_lo,
                              int64_t row_hi, void* stream) {
    return guard([&] {
        SOB_RANGE("so_spmv_device_rows");
        on_device(m);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx(m->device).stream;
        spmv_device_rows(*m, x_dev, y_dev, row_lo, row_hi, s);
    });
}

so_status so_spmv_rows_push(const so_matrix* m, const double* x_dev, double* y_dev, int64_t row_lo, int64_t row_hi,
                            double* remote_dev, unsigned* ticket_dev, unsigned long long* remote_flag,
                            unsigned long long flag_value, void* stream) {
    return guard([&] {
        SOB_RANGE("so_spmv_rows_push");
        on_device(m);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx(m->device).stream;
        spmv_rows_push(*m, x_dev, y_dev, row_lo, row_hi, remote_dev, ticket_dev, remote_flag, flag_value, s);
    });
}

so_status so_wait_flag(const unsigned long long* flag_dev, unsigned long long value, void* stream) {
    return guard([&] {
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : current_ctx().stream;
        wait_flag(flag_dev, value, s);
    });
}

int64_t so_wait_flag_timeouts(void) {
    int64_t v = -1;
    guard([&] {
        current_ctx();
        v = int64_t(wait_flag_timeouts());
    });
    return v;
}

so_status so_ipc_alloc(int64_t bytes, void** dev_ptr, so_ipc_handle* handle) {
    return guard([&] {
        if (bytes <= 0 || !dev_ptr || !handle) fail(SO_INVALID_INPUT, "ipc_alloc: bad arguments");
        current_ctx();
        void* p = nullptr;
        const cudaError_t e = cudaMalloc(&p, size_t(bytes));  // IPC needs a plain cudaMalloc allocation
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            fail(SO_OUT_OF_MEMORY, "ipc_alloc: out of device memory");
        }
        SOB_CUDA(e);
        SOB_CUDA(cudaMemset(p, 0, size_t(bytes)));
        cudaIpcMemHandle_t h;
        SOB_CUDA(cudaIpcGetMemHandle(&h, p));
        static_assert(sizeof(h) <= sizeof(handle->bytes), "IPC handle size");
        std::memcpy(handle->bytes, &h, sizeof(h));
        *dev_ptr = p;
    });
}

so_status so_ipc_open(const so_ipc_handle* handle, void** dev_ptr) {
    return guard([&] {
        if (!handle || !dev_ptr) fail(SO_INVALID_INPUT, "ipc_open: bad arguments");
        current_ctx();
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle->bytes, sizeof(h));
        SOB_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

so_status so_ipc_close(void* dev_ptr) {
    return guard([&] { SOB_CUDA(cudaIpcCloseMemHandle(dev_ptr)); });
}

so_status so_ipc_free(void* dev_ptr) {
    return guard([&] { SOB_CUDA(cudaFree(dev_ptr)); });
}

so_status so_gen_stencil27_dia(int64_t g, int64_t row_lo, int64_t row_hi, int64_t col_lo, int64_t col_hi,
                               uint64_t seed, so_matrix** out) {
    return make(out, [&] {
        const int64_t n = g * g * g;
        if (g < 1 || row_lo < 0 || row_hi > n || row_lo > row_hi || col_lo < 0 || col_hi > n || col_lo > col_hi)
            fail(SO_INVALID_INPUT, "stencil slice outside the g^3 grid");
        check_dims(row_hi - row_lo, col_hi - col_lo);
        return gen_stencil27_dia(g, row_lo, row_hi, col_lo, col_hi, seed, current_ctx().stream);
    });
}

so_status so_spmv(const so_matrix* m, const double* x, int64_t xlen, double* y) {
    return guard([&] {
        SOB_RANGE("so_spmv");
        cudaStream_t s = on_device(m);
        check_x(*m, xlen);
        if (m->nrows > 0 && spmv_pipelined(*m, x, y, s)) {
            SOB_CUDA(cudaStreamSynchronize(s));
            return;
        }
        // pageable buffers (the reference API's std::vector): staged through
        // pinned memory by host threads, overlapped with the device work;
        // pinned buffers the follow path declined go straight to the copy
        // engines (the staging copies would only add host traffic)
        static const bool pinned_staged = std::getenv("SOB_PINNED_STAGED") != nullptr;  // diagnostic knob (A/B)
        const bool both_pinned = !pinned_staged && is_pinned(x) && is_pinned(y);
        if (both_pinned && m->nrows >= 2 * kPipeRows) {
            // CSR: the kernels follow one upload of x and store y into mapped host memory
            const auto xa = reinterpret_cast<uintptr_t>(x), ya = reinterpret_cast<uintptr_t>(y);
            const bool overlap = xa < ya + sizeof(double) * size_t(m->nrows) && ya < xa + sizeof(double) * size_t(m->ncols);
            double* ym = static_cast<double*>(const_cast<void*>(mapped_ptr(y)));
            if (!overlap && ym && spmv_csr_follow(*m, x, ym, s, ctx(m->device).copy_in)) return;
        }
        if (m->nrows > 0 && !both_pinned && spmv_pageable(*m, x, y, s)) return;
        DBuf<double> dx, dy(m->nrows, s);
        h2d(dx, x, xlen, s);
        spmv_device(*m, dx.get(), dy.get(), s);
        d2h(y, dy, m->nrows, s);
        SOB_CUDA(cudaStreamSynchronize(s));
    });
}

so_status so_spmv_new(const so_matrix* m, const double* x, int64_t xlen, so_make_output make_y, void* make_ctx) {
    return guard([&] {
        SOB_RANGE("so_spmv_new");
        if (!make_y) fail(SO_INVALID_INPUT, "spmv: null output allocator");
        cudaStream_t s = on_device(m);
        check_x(*m, xlen);
        const std::function<double*()> mk = [&]() -> double* { return make_y(make_ctx, m->nrows); };
        // pageable x: y is built on this thread while the device works
        static const bool eager = std::getenv("SOB_EAGER_Y") != nullptr;  // diagnostic knob (A/B)
        if (!eager && m->nrows > 0 && spmv_pageable(*m, x, nullptr, s, &mk)) return;
        double* y = mk();
        if (!y && m->nrows > 0) fail(SO_OUT_OF_MEMORY, "spmv: output vector allocation failed");
        if (m->nrows > 0 && spmv_pipelined(*m, x, y, s)) {
            SOB_CUDA(cudaStreamSynchronize(s));
            return;
        }
        if (m->nrows > 0 && spmv_pageable(*m, x, y, s)) return;
        DBuf<double> dx, dy(m->nrows, s);
        h2d(dx, x, xlen, s);
        spmv_device(*m, dx.get(), dy.get(), s);
        d2h(y, dy, m->nrows, s);
        SOB_CUDA(cudaStreamSynchronize(s));
    });
}

so_status so_time_spmv(const so_matrix* m, const double* x, int64_t xlen, int64_t reps, double* per_rep,
                       double* total) {
    return guard([&] {
        SOB_RANGE("so_time_spmv");
        if (reps < 1) fail(SO_INVALID_INPUT, "time_spmv: repetitions must be >= 1");  // spmv.cpp:223-225
        cudaStream_t s = on_device(m);
        check_x(*m, xlen);
        DBuf<double> dx, dy(m->nrows, s);
        h2d(dx, x, xlen, s);
        spmv_device(*m, dx.get(), dy.get(), s);  // warm-up, untimed (spmv.cpp:231)
        EventSet evs(size_t(reps) + 1, 0);
        std::vector<cudaEvent_t>& ev = evs.ev;
        SOB_CUDA(cudaEventRecord(ev[0], s));
        for (int64_t r = 0; r < reps; ++r) {
            spmv_device(*m, dx.get(), dy.get(), s);
            SOB_CUDA(cudaEventRecord(ev[size_t(r) + 1], s));
        }
        SOB_CUDA(cudaStreamSynchronize(s));
        double sum = 0.0;
        for (int64_t r = 0; r < reps; ++r) {
            float ms = 0.f;
            SOB_CUDA(cudaEventElapsedTime(&ms, ev[size_t(r)], ev[size_t(r) + 1]));
            per_rep[r] = double(ms) * 1e-3;
            sum += per_rep[r];
        }
        *total = sum;
    });
}

int64_t so_spmv_bytes(const so_matrix* m) {
    int64_t bytes = -1;
    guard([&] {
        cudaStream_t s = on_device(m);
        const int64_t n = m->nrows, nc = m->ncols;
        int64_t b = 8 * nc + 8 * n;  // x read once, y written once
        auto dia_bytes = [&]() {
            std::vector<int64_t> off(size_t(m->dia.ndiags));
            d2h(off.data(), m->dia.offsets, m->dia.ndiags, s);
            SOB_CUDA(cudaStreamSynchronize(s));
            int64_t cells = 0;
            for (int64_t o : off) {
                const int64_t lo = std::max<int64_t>(0, -o), hi = std::min(n, nc - o);
                if (hi > lo) cells += hi - lo;
            }
            return 8 * cells + 8 * m->dia.ndiags;
        };
        auto ell_bytes = [&]() {
            DBuf<unsigned long long> c(1, s);
            SOB_CUDA(cudaMemsetAsync(c.get(), 0, sizeof(unsigned long long), s));
            if (n > 0) {
                ell_short_rows<<<grid1(n), 256, 0, s>>>(m->ell.col.get(), n, m->ell.width, c.get());
                SOB_LAUNCH("ell_short_rows");
            }
            const int64_t shortr = int64_t(d2h_scalar(c.get(), s));
            return m->ell.stored_nnz * 12 + 4 * shortr;
        };
        switch (m->format) {
            case SO_COO: b += m->coo.nnz * 16; break;
            case SO_CSR: b += m->csr.nnz * 12 + (n + 1) * 8; break;
            case SO_DIA: b += dia_bytes(); break;
            case SO_ELL: b += ell_bytes(); break;
            case SO_HYB: b += ell_bytes() + m->coo.nnz * 16; break;
            // an empty CSR part is never touched (the DIA kernel runs alone)
            case SO_HDC: b += dia_bytes() + (m->csr.nnz > 0 ? m->csr.nnz * 12 + (n + 1) * 8 : 0); break;
        }
        bytes = b;
    });
    return bytes;
}

// -------------------------------------------------------------- features

so_status so_extract_features(const so_matrix* m, double ratio, so_feature_vector* out, so_scan_stats* stats) {
    return guard([&] {
        SOB_RANGE("so_extract_features");
        cudaStream_t s = on_device(m);
        check_ratio(*m, ratio);
        DBuf<FeatState> st(1, s);
        enqueue_features(*m, ratio, st.get(), s);
        FeatState h;
        SOB_CUDA(cudaMemcpyAsync(&h, st.get(), sizeof(FeatState), cudaMemcpyDeviceToHost, s));
        SOB_CUDA(cudaStreamSynchronize(s));
        if (out) *out = h.out;
        if (stats) {
            stats->entry_visits = int64_t(h.visits);
            stats->structure_reads = int64_t(h.structure);
        }
    });
}

// ----------------------------------------------------------------- model

so_status so_forest_upload(int32_t kind, int32_t n_trees, const int64_t* node_off, const int32_t* feature,
                           const double* threshold, const int32_t* left, const int32_t* right, const int32_t* cls,
                           so_forest** out) {
    return guard([&] {
        SOB_RANGE("so_forest_upload");
        *out = nullptr;
        *out = forest_upload(kind, n_trees, node_off, feature, threshold, left, right, cls, current_ctx().stream);
    });
}

void so_forest_free(so_forest* f) { delete f; }

namespace sob {
namespace {
so_status predict_host_rows(const so_forest* f, int64_t n, const double* rows, int32_t* out, bool blocked) {
    return guard([&] {
        SOB_RANGE("so_predict_rows");
        if (!f) fail(SO_INVALID_INPUT, "null forest");
        if (n < 0 || (n > 0 && (!rows || !out))) fail(SO_INVALID_INPUT, "bad rows");
        SOB_CUDA(cudaSetDevice(f->device));
        g_dev = f->device;
        cudaStream_t s = ctx(f->device).stream;
        DBuf<double> dr;
        h2d(dr, rows, n * 10, s);
        DBuf<int32_t> dout(n, s);
        if (blocked)
            predict_rows_blocked(*f, dr.get(), n, dout.get(), s);
        else
            predict_rows(*f, dr.get(), n, dout.get(), s);
        d2h(out, dout, n, s);
        SOB_CUDA(cudaStreamSynchronize(s));
    });
}
}  // namespace
}  // namespace sob

so_status so_predict_rows(const so_forest* f, int64_t n, const double* rows, int32_t* out) {
    return predict_host_rows(f, n, rows, out, false);
}

so_status so_predict_rows_latency(const so_forest* f, int64_t n, const double* rows, int32_t* out) {
    return predict_host_rows(f, n, rows, out, true);
}

so_status so_predict(const so_forest* f, const so_feature_vector* x, int32_t* out) {
    if (!x) {
        set_error("null feature vector");
        return SO_INVALID_INPUT;
    }
    double row[10] = {double(x->nrows),          double(x->ncols),          double(x->nnz),
                      x->avg_nnz_per_row,        x->density,                double(x->max_nnz_per_row),
                      double(x->min_nnz_per_row), x->nnz_row_spread,        double(x->ndiags),
                      double(x->ntrue_diags)};
    // one row: the blocked warp walk of the fused tuner (latency path)
    return so_predict_rows_latency(f, 1, row, out);
}

// tune_ml with the feature pipeline (about ten kernels + stream-ordered
// scratch allocations) captured once per (matrix, forest, ratio, caps) as a
// CUDA graph and replayed with a single launch, so small matrices pay one
// launch instead of ten; the predict/feasibility kernel follows on the same
// stream.  The outcome lands in a persistent device buffer (one small D2H).
so_status so_tune_ml(const so_matrix* m, const so_forest* f, double ratio, const so_conversion_config* cfgp,
                     so_tune_outcome* out) {
    const auto t_entry = std::chrono::steady_clock::now();
    return guard([&] {
        SOB_RANGE("so_tune_ml");
        if (!f || !out) fail(SO_INVALID_INPUT, "null argument");
        cudaStream_t s = on_device(m);
        if (f->device != m->device) fail(SO_INVALID_INPUT, "forest and matrix live on different devices");
        check_ratio(*m, ratio);
        so_conversion_config cfg = cfg_or_default(cfgp);
        cfg.true_diag_ratio = ratio;  // TunerConfig::effective_conversion (tuners.hpp:21-25)
        // the cached plan (graph, workspace, events, stream) belongs to the
        // matrix: concurrent tune_ml calls on one const matrix take turns,
        // different matrices tune concurrently
        std::lock_guard<std::mutex> plan_lock(m->tune_mu);
        TunePlan* plan = m->tune_plan.get();
        if (!plan || !plan->matches(f->uid, cfg)) {
            m->tune_plan.reset();
            std::unique_ptr<TunePlan, TunePlanDeleter> np(new TunePlan());
            np->forest_uid = f->uid;
            np->cfg = cfg;
            SOB_CUDA(cudaStreamCreateWithFlags(&np->ps, cudaStreamNonBlocking));
            SOB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&np->st), sizeof(FeatState), s));
            SOB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&np->out), sizeof(so_tune_outcome), cudaHostAllocMapped));
            SOB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&np->out_dev), np->out, 0));
            SOB_CUDA(cudaEventCreate(&np->e0));
            SOB_CUDA(cudaEventCreate(&np->e1));
            np->ws.reset(new FeatWorkspace(*m, s));
            np->ws->enable_fork();  // the graph gets the bins branch beside the spread chain
            SOB_CUDA(cudaStreamSynchronize(s));
            cudaStream_t ps = np->ps;
            // which CSR sweep suits this matrix depends on how its diagonal
            // keys repeat (banded/stencil rows: the lockstep sweep's slot
            // cache; scattered keys: the entry-parallel sweep, e.g. a 172K-row
            // uniform matrix 88 -> 80 us, or straight global atomics): time
            // the three once, keep the fastest
            if ((m->format == SO_CSR || m->format == SO_HDC) && m->csr.nblk > 0 && m->nrows > 0 &&
                !std::getenv("SOB_FEAT_ENTRY")) {
                float best[3] = {1e30f, 1e30f, 1e30f};
                auto time_mode = [&](int mode) {
                    np->ws->sweep = mode;
                    SOB_CUDA(cudaEventRecord(np->e0, ps));
                    enqueue_features(*m, ratio, np->st, ps, np->ws.get());
                    SOB_CUDA(cudaEventRecord(np->e1, ps));
                    SOB_CUDA(cudaEventSynchronize(np->e1));
                    float ms = 0.f;
                    SOB_CUDA(cudaEventElapsedTime(&ms, np->e0, np->e1));
                    best[mode] = std::min(best[mode], ms);
                };
                time_mode(0);
                // straight global atomics only pay off when keys barely repeat
                // (R-MAT: ~9 entries per diagonal); on banded / stencil rows
                // every entry of a diagonal would hit one address (config 2:
                // 36 ms), so that mode is not even timed there
                so_feature_vector fv{};
                SOB_CUDA(cudaMemcpy(&fv, reinterpret_cast<const char*>(np->st) + offsetof(FeatState, out), sizeof(fv),
                                    cudaMemcpyDeviceToHost));
                const bool try_direct = fv.ndiags > 0 && fv.nnz <= 64 * fv.ndiags;
                for (int rep = 0; rep < 2; ++rep)
                    for (int mode = 0; mode < 3; ++mode)
                        if (mode != 2 || try_direct) time_mode(mode);
                np->ws->sweep = int(std::min_element(best, best + 3) - best);
            }
            cudaGraph_t g = nullptr;
            // one graph: features, predict + feasibility; T_FE / T_PRED are
            // device intervals taken by the kernels themselves (%globaltimer
            // stamps: first feature kernel -> finalize -> vote), so the graph
            // carries no event nodes and the host no event queries
            SOB_CUDA(cudaStreamBeginCapture(ps, cudaStreamCaptureModeThreadLocal));
            try {
                enqueue_features(*m, ratio, np->st, ps, np->ws.get());
                enqueue_tune_predict(*f, np->st, cfg, m->format, np->out_dev, ps);
            } catch (...) {
                cudaStreamEndCapture(ps, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            SOB_CUDA(cudaStreamEndCapture(ps, &g));
            SOB_CUDA(cudaGraphInstantiate(&np->exec, g, 0));
            cudaGraphDestroy(g);
            plan = np.get();
            m->tune_plan = std::move(np);
        }
        // every call that produces or changes a matrix synchronises before it
        // returns (make(), conversions), so the matrix arrays are complete:
        // the replay needs no ordering against the context stream
        static const bool trace = std::getenv("SOB_TUNE_TRACE") != nullptr;  // diagnostic knob: host phases
        const auto t_plan = std::chrono::steady_clock::now();
        SOB_CUDA(cudaGraphLaunch(plan->exec, plan->ps));
        const auto t_launch = std::chrono::steady_clock::now();
        SOB_CUDA(cudaStreamSynchronize(plan->ps));
        const auto t_sync = std::chrono::steady_clock::now();
        so_tune_outcome h = *plan->out;  // written by the predict kernel (mapped host memory), times included
        const double fe = h.feature_time_seconds * 1e3, pr = h.predict_time_seconds * 1e3;
        const auto t_end = std::chrono::steady_clock::now();
        h.wall_time_seconds = std::chrono::duration<double>(t_end - t_entry).count();
        if (trace) {
            auto us = [&](std::chrono::steady_clock::time_point t) {
                return std::chrono::duration<double, std::micro>(t - t_entry).count();
            };
            std::fprintf(stderr, "[tune] plan %.1f launch %.1f sync %.1f end %.1f us; fe %.1f pred %.1f us\n",
                         us(t_plan), us(t_launch), us(t_sync), us(t_end), fe * 1e3, pr * 1e3);
        }
        *out = h;
    });
}

}  // extern "C"
