// spmv(m, x) with pageable host buffers -- the reference API's own call
// (spmv.hpp:20, spmv.cpp:203-219: x is a std::vector, y comes back as a fresh
// std::vector).  The device cannot DMA pageable memory directly; the driver's
// pageable copies bounce through a small internal buffer one piece at a time.
// Here host threads copy x into a cached pinned (mapped) staging buffer in
// chunks, and the device starts on each chunk as soon as it has landed:
//
//   * DIA-window matrices (DIA, HDC with an empty CSR part, diagonal window
//     <= 256): the zero-copy kernel reads x straight from the staging buffer
//     and writes y straight into the pinned y staging buffer, row blocks
//     launched as soon as the x prefix their window needs is staged;
//   * every other matrix: chunk k of x goes up on the copy engine as soon as
//     it is staged, the kernel runs on the full x, y comes back in chunks.
//
// In both cases the same host threads copy y out of the staging buffer chunk
// by chunk as the device finishes it (a CUDA event per chunk), so the host
// copies of x and y overlap the link transfers and the kernel.  Results are
// bit-identical to the one-shot path (same kernels).
//
// Lazy y (so_spmv_new, the C++ spmv(m, x) returning a fresh std::vector): the
// caller's thread builds y -- the vector's value-initialisation, a 32 MB
// single-threaded zero fill on config 2 -- while a pool thread orchestrates
// the device work and the others stage x; the y copies start once y exists.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <immintrin.h>
#include <sys/resource.h>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "matrix.cuh"

namespace sob {

namespace {

// Persistent host copy pool: workers sleep on a condition variable between
// calls and spin (briefly) during one.
class CopyPool {
  public:
    static CopyPool& get() {
        static CopyPool pool;
        return pool;
    }
    int size() const { return int(th_.size()); }
    // run fn(worker) on every worker and on the caller (worker id size());
    // returns when all are done
    void run(const std::function<void(int)>& fn, const std::function<void()>& caller) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            pending_ = int(th_.size());
            ++gen_;
        }
        cv_.notify_all();
        caller();
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }

  private:
    CopyPool() {
        int n = int(std::thread::hardware_concurrency());
        if (const char* e = std::getenv("SOB_HOST_THREADS")) n = std::atoi(e);  // tuning knob
        n = std::max(1, std::min(n, 32));  // all host threads: 16 beat 8 by 1.3x on the B200 hosts (32 MB x + y)
        for (int i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    void loop(int id) {
        uint64_t seen = 0;
        while (true) {
            const std::function<void(int)>* fn;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                fn = fn_;
            }
            if (fn) (*fn)(id);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* fn_ = nullptr;
    uint64_t gen_ = 0;
    int pending_ = 0;
    bool stop_ = false;
};

// Pinned, mapped staging buffers per device (grow-only, one pageable call at
// a time per device).
struct Staging {
    std::mutex mu;
    double* x = nullptr;
    double* y = nullptr;
    size_t capx = 0, capy = 0;
    std::vector<cudaEvent_t> ev;
    void reserve(size_t nx, size_t ny) {
        auto grow = [](double*& p, size_t& cap, size_t want) {
            if (cap >= want) return;
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            SOB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p), want * sizeof(double),
                                   cudaHostAllocMapped | cudaHostAllocPortable));
            cap = want;
        };
        grow(x, capx, std::max<size_t>(nx, 1));
        grow(y, capy, std::max<size_t>(ny, 1));
    }
    void events(size_t n) {
        while (ev.size() < n) {
            cudaEvent_t e;
            SOB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ev.push_back(e);
        }
    }
};
Staging g_stage[64];

// Host copy with non-temporal (streaming) stores: the destination is not
// read first (no read-for-ownership) and does not evict the source from the
// caches -- x lands in pinned memory that only the device reads next, y in a
// buffer the caller reads later.  AVX2 when the CPU has it, else memcpy.
__attribute__((target("avx2"))) void copy_nt_avx2(double* dst, const double* src, size_t n) {
    size_t i = 0;
    while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31)) {
        dst[i] = src[i];
        ++i;
    }
    for (; i + 16 <= n; i += 16) {
        const __m256d a = _mm256_loadu_pd(src + i), b = _mm256_loadu_pd(src + i + 4);
        const __m256d c = _mm256_loadu_pd(src + i + 8), d = _mm256_loadu_pd(src + i + 12);
        _mm256_stream_pd(dst + i, a);
        _mm256_stream_pd(dst + i + 4, b);
        _mm256_stream_pd(dst + i + 8, c);
        _mm256_stream_pd(dst + i + 12, d);
    }
    for (; i < n; ++i) dst[i] = src[i];
    _mm_sfence();
}

// want_nt = false: plain stores -- for a y the caller's thread has just
// value-initialised (lazy y), whose lines are still cache-resident: streaming
// stores would first have to evict them (config 2: 3.1 -> 2.1 ms per call)
void copy_host(double* dst, const double* src, size_t n, bool want_nt = true) {
    static const bool nt = [] {
        if (std::getenv("SOB_NO_NT_COPY")) return false;  // diagnostic knob
        __builtin_cpu_init();
        return bool(__builtin_cpu_supports("avx2"));
    }();
    if (nt && want_nt)
        copy_nt_avx2(dst, src, n);
    else
        std::memcpy(dst, src, n * sizeof(double));
}

struct Task {
    double* dst;  // x tasks; y tasks copy to y + off (y may not exist yet)
    const double* src;
    size_t n;
    int chunk;  // x chunk (>= 0) or -(y chunk) - 1
    int64_t off;
};

constexpr int64_t kMinStaged = int64_t(1) << 18;  // elements of x + y below which the one-shot path wins
constexpr int64_t kTaskElems = int64_t(1) << 16;  // 512 KB per host copy task

}  // namespace

bool spmv_pageable(const so_matrix& m, const double* x, double* y, cudaStream_t s,
                   const std::function<double*()>* make_y) {
    static const bool off = std::getenv("SOB_NO_PAGEABLE_STAGING") != nullptr;  // diagnostic knob
    const int64_t n = m.nrows, nc = m.ncols;
    if (off || n + nc < kMinStaged || !x || (!y && !make_y)) return false;
    // in-place calls: x must be read in full before any y lands (one-shot path)
    const auto xa = reinterpret_cast<uintptr_t>(x), ya = reinterpret_cast<uintptr_t>(y);
    if (!make_y && xa < ya + sizeof(double) * size_t(n) && ya < xa + sizeof(double) * size_t(nc)) return false;
    static const bool trace = std::getenv("SOB_STAGE_TRACE") != nullptr;  // diagnostic knob: phase times
    const auto t_entry = std::chrono::steady_clock::now();
    std::atomic<int64_t> t_launched{0}, t_yready{0}, t_ycopied{0};
    auto stamp = [&](std::atomic<int64_t>& t) {
        if (trace)
            t.store(std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t_entry).count());
    };
    const int dev = m.device;
    Staging& st = g_stage[dev];
    std::lock_guard<std::mutex> lk(st.mu);
    st.reserve(size_t(nc), size_t(n));
    double* X = st.x;
    double* Y = st.y;
    double *Xd = nullptr, *Yd = nullptr;
    SOB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&Xd), X, 0));
    SOB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&Yd), Y, 0));

    const bool dia_only = (m.format == SO_DIA || (m.format == SO_HDC && m.csr.nnz == 0)) && m.dia.ndiags > 0;
    if (dia_only) ensure_dia_window(m, s);
    const int64_t zr = zero_copy_rows_per_block();
    // x chunks of ~1/8 of x (>= 1 MB), y chunks aligned to zero-copy blocks
    const int64_t cx = std::max<int64_t>(int64_t(1) << 17, ceil_div(nc, 8));
    const int64_t nxc = ceil_div(nc, cx);
    const int64_t cy = std::max<int64_t>(ceil_div(int64_t(1) << 17, zr), ceil_div(ceil_div(n, 8), zr)) * zr;
    const int64_t nyc = ceil_div(n, cy);
    st.events(size_t(nyc));
    std::atomic<bool> follow{false};  // narrow DIA windows: the follow-the-copy kernel (one launch per y chunk)
    FollowToken ftok;

    // the task list: every x chunk (in order), then every y chunk
    std::vector<Task> tasks;
    std::vector<int> per_x(size_t(nxc), 0), per_y(size_t(nyc), 0);
    for (int64_t k = 0; k < nxc; ++k)
        for (int64_t a = k * cx, e = std::min(nc, a + cx); a < e; a += kTaskElems, ++per_x[size_t(k)])
            tasks.push_back(Task{X + a, x + a, size_t(std::min(e, a + kTaskElems) - a), int(k), a});
    for (int64_t j = 0; j < nyc; ++j)
        for (int64_t a = j * cy, e = std::min(n, a + cy); a < e; a += kTaskElems, ++per_y[size_t(j)])
            tasks.push_back(Task{nullptr, Y + a, size_t(std::min(e, a + kTaskElems) - a), -int(j) - 1, a});
    std::unique_ptr<std::atomic<int>[]> xdone(new std::atomic<int>[size_t(nxc)]);
    std::unique_ptr<std::atomic<int>[]> ygate(new std::atomic<int>[size_t(nyc)]);  // y chunk's event recorded
    for (int64_t k = 0; k < nxc; ++k) xdone[size_t(k)].store(0);
    for (int64_t j = 0; j < nyc; ++j) ygate[size_t(j)].store(0);
    std::atomic<size_t> next{0};
    std::atomic<int> failed{0};
    std::atomic<double*> yptr{make_y ? nullptr : y};
    std::mutex ymu;
    std::condition_variable ycv;
    std::exception_ptr err, yerr;
    std::function<void()> orchestrate;

    auto worker = [&](int id) {
        cudaSetDevice(dev);
        if (make_y && id == 0) orchestrate();  // the caller is building y
        // After a failure the y copies are skipped but every x chunk is
        // still staged: the orchestrator waits for each (wait_x) before it
        // can finish, so abandoning one would hang the call (a failed y
        // allocation raced the x tasks this way).
        auto y_ready = [&](const Task& k, double*& dst) -> bool {
            const int j = -k.chunk - 1;
            if (!(dst = yptr.load(std::memory_order_acquire))) {
                // y is being built on the caller's thread: sleep, do not
                // spin (spinning workers take its core and its memory
                // bandwidth: config 2 zero fill 0.9 -> 2.0 ms)
                std::unique_lock<std::mutex> lk(ymu);
                ycv.wait(lk, [&] { return yptr.load(std::memory_order_acquire) || failed.load(); });
                dst = yptr.load(std::memory_order_acquire);
                if (!dst) return false;
            }
            dst += k.off;
            while (!ygate[size_t(j)].load(std::memory_order_acquire)) {
                if (failed.load(std::memory_order_relaxed)) return false;
                std::this_thread::yield();
            }
            while (true) {
                const cudaError_t q = cudaEventQuery(st.ev[size_t(j)]);
                if (q == cudaSuccess) return !failed.load(std::memory_order_relaxed);
                if (q != cudaErrorNotReady) {
                    failed.store(1);
                    return false;
                }
                std::this_thread::yield();
            }
        };
        while (true) {
            const size_t t = next.fetch_add(1);
            if (t >= tasks.size()) return;
            const Task& k = tasks[t];
            double* dst = k.dst;
            if (k.chunk < 0 && (failed.load(std::memory_order_relaxed) || !y_ready(k, dst))) continue;
            copy_host(dst, k.src, k.n, k.chunk >= 0 || !make_y);
            if (k.chunk >= 0) xdone[size_t(k.chunk)].fetch_add(1, std::memory_order_release);
            if (trace && t + 1 == tasks.size()) stamp(t_ycopied);
        }
    };

    orchestrate = [&]() {
        try {
            auto wait_x = [&](int64_t k) {
                while (xdone[size_t(k)].load(std::memory_order_acquire) < per_x[size_t(k)]) std::this_thread::yield();
            };
            // narrow DIA windows: each staged x chunk goes up on the copy
            // engine while a kernel per y chunk follows the copy front
            // (spmv.cu dia_follow_kernel); an event after each launch gates
            // that chunk's copy-out
            if (dia_only && cy % zr == 0) {
                cudaStream_t copy = ctx(dev).copy_in;
                const std::function<void(int64_t)> after = [&](int64_t j) {
                    SOB_CUDA(cudaEventRecord(st.ev[size_t(j)], s));
                    ygate[size_t(j)].store(1, std::memory_order_release);
                };
                const bool launched = follow_launch(m, Yd, s, copy, cy, &after, [&](double* dx) {
                    for (int64_t k = 0; k < nxc; ++k) {
                        wait_x(k);
                        const int64_t a = k * cx, e = std::min(nc, a + cx);
                        SOB_CUDA(cudaMemcpyAsync(dx + a, X + a, sizeof(double) * size_t(e - a), cudaMemcpyHostToDevice,
                                                 copy));
                    }
                }, ftok);
                if (launched) {
                    follow.store(true, std::memory_order_release);
                    stamp(t_launched);
                    return;
                }
            }
            // CSR / ELL / COO / HYB: the same with one launch of the FOLLOW
            // kernels.  CSR / ELL store y into Yd: one event after them gates
            // every y chunk's copy-out.  COO parts leave y in device memory:
            // it comes down chunk by chunk, an event after each chunk's copy
            // (one copy of all of y was slower than the staged path: config 2
            // COO 1.85 -> 1.80 ms, the HYB-shaped matrix COO 1.68 -> 1.81,
            // HYB 1.62 -> 1.82; profiles/r02ao_coo_follow.txt)
            static const bool coo_staged = std::getenv("SOB_PAGEABLE_COO_STAGED") != nullptr;  // A/B knob
            const bool coo_part = (m.format == SO_COO || m.format == SO_HYB) && m.coo.nnz > 0;
            if (!dia_only && !(coo_part && coo_staged)) {
                cudaStream_t copy = ctx(dev).copy_in;
                const std::function<void(const double*)> after = [&](const double* ydev) {
                    for (int64_t j = 0; j < nyc; ++j) {
                        if (ydev) {
                            const int64_t a = j * cy, e = std::min(n, a + cy);
                            SOB_CUDA(cudaMemcpyAsync(Yd + a, ydev + a, sizeof(double) * size_t(e - a),
                                                     cudaMemcpyDefault, s));
                        }
                        SOB_CUDA(cudaEventRecord(st.ev[size_t(j)], s));
                        if (ydev) ygate[size_t(j)].store(1, std::memory_order_release);
                    }
                    if (!ydev)
                        for (int64_t j = 0; j < nyc; ++j) ygate[size_t(j)].store(1, std::memory_order_release);
                };
                const bool launched = follow_launch_rows(m, Yd, s, copy, &after, [&](double* dx) {
                    for (int64_t k = 0; k < nxc; ++k) {
                        wait_x(k);
                        const int64_t a = k * cx, e = std::min(nc, a + cx);
                        SOB_CUDA(cudaMemcpyAsync(dx + a, X + a, sizeof(double) * size_t(e - a), cudaMemcpyHostToDevice,
                                                 copy));
                    }
                }, ftok);
                if (launched) {
                    follow.store(true, std::memory_order_release);
                    stamp(t_launched);
                    return;
                }
            }
            // an empty launch range probes eligibility (window <= 256, offsets fit)
            const bool zc = dia_only && spmv_dia_zero_copy(m, Xd, Yd, s, 0, 0);
            if (zc) {
                // zero-copy row blocks as their x window is staged
                const int64_t nblk = ceil_div(n, zr);
                const int64_t omax = m.dia_omax;
                int64_t blk_done = 0, yrec = 0;
                for (int64_t k = 0; k < nxc; ++k) {
                    wait_x(k);
                    const int64_t P = std::min(nc, (k + 1) * cx);
                    // block b reads x up to min(nc, (b+1)*zr + omax)
                    int64_t hi = P >= nc ? nblk : std::max<int64_t>(0, (P - omax) / zr);
                    hi = std::min(hi, nblk);
                    if (hi > blk_done) {
                        spmv_dia_zero_copy(m, Xd, Yd, s, blk_done, hi);
                        blk_done = hi;
                        // y chunks whose rows are all launched
                        while (yrec < nyc && std::min(n, (yrec + 1) * cy) <= std::min(n, blk_done * zr)) {
                            SOB_CUDA(cudaEventRecord(st.ev[size_t(yrec)], s));
                            ygate[size_t(yrec)].store(1, std::memory_order_release);
                            ++yrec;
                        }
                    }
                }
                while (yrec < nyc) {
                    SOB_CUDA(cudaEventRecord(st.ev[size_t(yrec)], s));
                    ygate[size_t(yrec)].store(1, std::memory_order_release);
                    ++yrec;
                }
                stamp(t_launched);
                return;
            }
            // generic: x chunks up on the copy engine as staged, kernel, y down in chunks
            DBuf<double> dx(nc, s), dy(n, s);
            for (int64_t k = 0; k < nxc; ++k) {
                wait_x(k);
                const int64_t a = k * cx, e = std::min(nc, a + cx);
                SOB_CUDA(cudaMemcpyAsync(dx.get() + a, X + a, sizeof(double) * size_t(e - a), cudaMemcpyHostToDevice, s));
            }
            spmv_device(m, dx.get(), dy.get(), s);
            stamp(t_launched);
            for (int64_t j = 0; j < nyc; ++j) {
                const int64_t a = j * cy, e = std::min(n, a + cy);
                SOB_CUDA(cudaMemcpyAsync(Y + a, dy.get() + a, sizeof(double) * size_t(e - a), cudaMemcpyDeviceToHost, s));
                SOB_CUDA(cudaEventRecord(st.ev[size_t(j)], s));
                ygate[size_t(j)].store(1, std::memory_order_release);
            }
        } catch (...) {
            err = std::current_exception();
            failed.store(1);
        }
    };
    CopyPool& pool = CopyPool::get();
    pool.run(worker, [&] {
        if (make_y) {
            try {
                struct rusage ru0, ru1;
                if (trace) getrusage(RUSAGE_THREAD, &ru0);
                double* p = (*make_y)();
                if (trace) {
                    getrusage(RUSAGE_THREAD, &ru1);
                    std::fprintf(stderr, "[stage] make_y minor faults %ld\n", ru1.ru_minflt - ru0.ru_minflt);
                }
                if (!p) fail(SO_OUT_OF_MEMORY, "spmv: output vector allocation failed");
                {
                    std::lock_guard<std::mutex> lk(ymu);
                    yptr.store(p, std::memory_order_release);
                }
                stamp(t_yready);
            } catch (...) {
                yerr = std::current_exception();
                std::lock_guard<std::mutex> lk(ymu);
                failed.store(1);
            }
            ycv.notify_all();
        } else {
            orchestrate();
        }
        worker(pool.size());  // then help with the y copies
    });
    if (err) {  // the copy stream may still read the staging buffers: drain both before they are released
        cudaStreamSynchronize(s);
        cudaStreamSynchronize(ctx(dev).copy_in);
        std::rethrow_exception(err);
    }
    if (yerr) {  // as above: the staged x may still be going up on the copy stream
        cudaStreamSynchronize(s);
        cudaStreamSynchronize(ctx(dev).copy_in);
        std::rethrow_exception(yerr);
    }
    if (follow.load()) {
        SOB_CUDA(cudaStreamSynchronize(s));
        if (!follow_finish(ftok)) {
            // the copy never reached the kernel (a serialising tool): y is
            // recomputed on the one-shot path into whatever y exists now
            double* yy = yptr.load();
            if (!yy) fail(SO_CUDA_ERROR, "pageable spmv: follow kernel timed out before y existed");
            SOB_CUDA(cudaStreamSynchronize(ctx(dev).copy_in));
            DBuf<double> dx(nc, s), dy(n, s);
            SOB_CUDA(cudaMemcpyAsync(dx.get(), x, sizeof(double) * size_t(nc), cudaMemcpyHostToDevice, s));
            spmv_device(m, dx.get(), dy.get(), s);
            SOB_CUDA(cudaMemcpyAsync(yy, dy.get(), sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, s));
            SOB_CUDA(cudaStreamSynchronize(s));
            return true;
        }
    }
    if (failed.load()) {
        cudaStreamSynchronize(s);
        fail(SO_CUDA_ERROR, "pageable spmv: staging copy failed");
    }
    SOB_CUDA(cudaStreamSynchronize(s));
    if (trace) {
        const int64_t t_end =
            std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t_entry).count();
        std::fprintf(stderr, "[stage] launched %lld us, y ready %lld us, last y copy %lld us, end %lld us (%s)\n",
                     (long long)t_launched.load(), (long long)t_yready.load(), (long long)t_ycopied.load(),
                     (long long)t_end, make_y ? "lazy y" : "caller y");
    }
    return true;
}

}  // namespace sob
