// Shared device/host plumbing for the sm_100a hot path: status handling,
// stream-ordered allocation, warp primitives and a hand-written scan.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <utility>

#include "sparseoracle_b200.h"

namespace sob {

// ---------------------------------------------------------------- errors ----

// Internal exception carrying an so_status; converted at the C-ABI edge.
struct Fail : std::runtime_error {
    so_status status;
    Fail(so_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(so_status s, const std::string& m) { throw Fail(s, m); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    so_status s = (e == cudaErrorMemoryAllocation) ? SO_OUT_OF_MEMORY : SO_CUDA_ERROR;
    fail(s, std::string(what) + ": " + cudaGetErrorString(e));
}

#define SOB_CUDA(call) ::sob::cuda_check((call), #call)
// every kernel launch of the library goes through this check; it also counts
// launches (so_kernel_launches, used by bench.py's gpu_launches)
void count_launch();
#define SOB_LAUNCH(what) (::sob::count_launch(), ::sob::cuda_check(cudaGetLastError(), what))

void set_error(const std::string& m);

// Programmatic dependent launch (sm_90+): a kernel launched with
// launch_pdl may be scheduled while its predecessor on the stream is still
// running; pdl_enter() -- the first statement of every such kernel -- waits
// for the predecessor's completion and memory (griddepcontrol.wait) and lets
// the NEXT kernel be scheduled as soon as all of this kernel's CTAs have
// started (griddepcontrol.launch_dependents).  A no-op for kernels launched
// without the attribute.  Used for the feature / tune chain, where the
// kernels are short and the launch latency between them is a large share.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" :::);
}
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cuda_check(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

// NVTX range over a C-ABI call (convert / features / predict / tune / SpMV /
// dist iterate), visible in nsys / ncu --nvtx timelines; header-only NVTX v3,
// a no-op unless a tool is attached (SURVEY §5 tracing).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define SOB_RANGE(name) ::sob::NvtxRange sob_nvtx_range_(name)

template <typename F>
so_status guard(F&& f) {
    try {
        f();
        return SO_OK;
    } catch (const Fail& e) {
        set_error(e.what());
        return e.status;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return SO_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        set_error(e.what());
        return SO_ERROR;
    }
}

// ---------------------------------------------------------------- context ---

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    // copy-engine streams of the pipelined host spmv (capi.cu so_spmv)
    cudaStream_t copy_in = nullptr, copy_out = nullptr;
    int num_sms = 148;
    int64_t l2_bytes = 0;
};

// Per-device context (created lazily; the non-blocking stream every host-facing
// call is ordered on).
Context& ctx(int device);
Context& current_ctx();

// RAII device buffer, stream-ordered (cudaMallocAsync from the device pool).
template <typename T>
struct DBuf {
    T* p = nullptr;
    int64_t n = 0;
    cudaStream_t s = nullptr;

    DBuf() = default;
    DBuf(int64_t count, cudaStream_t stream) { alloc(count, stream); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept { swap(o); }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            swap(o);
        }
        return *this;
    }
    ~DBuf() { release(); }

    void swap(DBuf& o) noexcept {
        std::swap(p, o.p);
        std::swap(n, o.n);
        std::swap(s, o.s);
    }
    void alloc(int64_t count, cudaStream_t stream) {
        release();
        s = stream;
        n = count;
        if (count > 0) SOB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * size_t(count), stream));
    }
    void release() noexcept {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return sizeof(T) * size_t(n); }
    T* get() const { return p; }
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Grid sizing: a multiple of the SM count (148 on B200) times resident CTAs,
// capped by the work available.
inline int grid_for(int64_t work_items, int block, int per_sm = 8) {
    Context& c = current_ctx();
    int64_t want = ceil_div(work_items, block);
    int64_t cap = int64_t(c.num_sms) * per_sm;
    if (want < 1) want = 1;
    return int(want < cap ? want : cap);
}

// ------------------------------------------------------------ device utils --

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}
// inclusive prefix sum within a warp
template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T w = __shfl_up_sync(0xffffffffu, v, o);
        if (lane_id() >= unsigned(o)) v += w;
    }
    return v;
}

// Streaming loads: bypass L1 allocation for read-once matrix arrays.
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int ld_stream(const int* p) {
    int v;
    asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// 256-bit streaming loads (sm_100: LDG.E.ENL2.256): one instruction moves 32
// contiguous bytes per lane, so a warp covers 1 KB with no L1 allocation.
// The pointer must be 32-byte aligned.
__device__ __forceinline__ void ld_stream_v8(const int* p, int (&v)[8]) {
    asm("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
        : "l"(p));
}
__device__ __forceinline__ void ld_stream_v4(const double* p, double* v) {
    asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
        : "l"(p));
}

// ----------------------------------------------------------- host helpers ---

// Exclusive scan of int64 counts in place-out (out[0..n]), out[n] = total.
// Hand-written 3-phase reduce-then-scan; returns nothing, total stays on device.
void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s);
// Exclusive scan of int32 flags/counts into int64 positions (out has n+1 slots).
void exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, cudaStream_t s);

template <typename T>
T d2h_scalar(const T* dptr, cudaStream_t s) {
    T v{};
    SOB_CUDA(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, s));
    SOB_CUDA(cudaStreamSynchronize(s));
    return v;
}

}  // namespace sob
