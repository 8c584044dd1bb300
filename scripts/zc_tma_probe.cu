// Diagnostic: host-buffer DIA spmv (config-2 shape: n = 4M, offsets -13..13)
// with the x windows pulled from mapped pinned host memory by the bulk-copy
// engine (cp.async.bulk, mbarrier completion) into a shared-memory ring of a
// persistent CTA, instead of per-thread 16-byte loads (the product's
// dia_zc_kernel).  Also: copy-engine reference numbers and a read-only
// bulk-copy bandwidth sweep.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o build/zc_tma_probe scripts/zc_tma_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>

constexpr int H = 13, ND = 2 * H + 1;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(b)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// persistent CTA, TR rows per tile, S-stage ring of x windows; y either
// stored per thread (YB = 0) or staged in shared memory and bulk-stored (YB = 1)
template <int TR, int S, int YB>
__global__ void __launch_bounds__(TR, 1) dia_tma(int n, const double* __restrict__ vals, const double* x, double* y) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int W = TR + 2 * H + 4;  // window doubles, even-aligned start
    double* xs = reinterpret_cast<double*>(smem);
    double* ys = xs + S * W;  // [2][TR] when YB
    __shared__ uint64_t bar[S];
    const int ntiles = (n + TR - 1) / TR;
    auto issue = [&](int k) {  // k-th tile of this CTA into stage k % S
        const int t = blockIdx.x + k * gridDim.x;
        if (t >= ntiles) return;
        const int i0 = t * TR;
        const int w0 = max(0, i0 - H) & ~1;
        const int w1 = min(n, i0 + TR + H);
        const uint32_t bytes = uint32_t((w1 - w0 + 1) & ~1) * 8u;
        mbar_expect_tx(&bar[k % S], bytes);
        bulk_g2s(xs + (k % S) * W, x + w0, bytes, &bar[k % S]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int k = 0; k < S; ++k) issue(k);
    }
    __syncthreads();
    for (int k = 0;; ++k) {
        const int t = blockIdx.x + k * gridDim.x;
        if (t >= ntiles) break;
        const int i0 = t * TR, i = i0 + threadIdx.x;
        const int w0 = max(0, i0 - H) & ~1;
        double v[ND];
#pragma unroll
        for (int d = 0; d < ND; ++d) v[d] = i < n ? __ldcs(vals + size_t(d) * n + i) : 0.0;
        mbar_wait(&bar[k % S], (k / S) & 1);
        const double* xw = xs + (k % S) * W;
        double acc = 0.0;
#pragma unroll
        for (int d = 0; d < ND; ++d) {
            const int c = i + d - H;
            acc = __dadd_rn(acc, (unsigned)c < (unsigned)n ? __dmul_rn(v[d], xw[c - w0]) : -0.0);
        }
        if (YB) {
            double* yb = ys + (k & 1) * TR;
            if (threadIdx.x == 0) bulk_wait_read<1>();  // the store issued from this buffer 2 tiles ago
            __syncthreads();
            if (i < n) yb[threadIdx.x] = acc;
            fence_async_smem();
        } else if (i < n) {
            y[i] = acc;
        }
        __syncthreads();  // stage k % S free, y buffer complete
        if (threadIdx.x == 0) {
            issue(k + S);
            if (YB) {
                const int cnt = min(TR, n - i0);
                bulk_s2g(y + i0, ys + (k & 1) * TR, uint32_t(cnt) * 8u);
                bulk_commit();
            }
        }
    }
    if (YB && threadIdx.x == 0) bulk_wait_read<0>();
    if (YB && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// read-only bulk-copy bandwidth from x (host or device), CH bytes per copy
template <int S>
__global__ void __launch_bounds__(32, 1) bulk_read(const char* x, size_t total, uint32_t ch, unsigned long long* sink) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bar[S];
    const size_t nch = total / ch;
    if (threadIdx.x != 0) return;
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    int k = 0;
    for (; k < S; ++k) {
        const size_t c = blockIdx.x + size_t(k) * gridDim.x;
        if (c >= nch) break;
        mbar_expect_tx(&bar[k], ch);
        bulk_g2s(smem + size_t(k) * ch, x + c * ch, ch, &bar[k]);
    }
    unsigned long long acc = 0;
    for (int j = 0;; ++j) {
        const size_t c = blockIdx.x + size_t(j) * gridDim.x;
        if (c >= nch) break;
        mbar_wait(&bar[j % S], (j / S) & 1);
        acc += smem[size_t(j % S) * ch];
        const size_t cn = blockIdx.x + size_t(j + S) * gridDim.x;
        if (cn < nch) {
            mbar_expect_tx(&bar[j % S], ch);
            bulk_g2s(smem + size_t(j % S) * ch, x + cn * ch, ch, &bar[j % S]);
        }
    }
    if (acc == 0xffffffffull) *sink = acc;
}

// the product's scheme (per-thread 16-byte window loads, y stored per thread)
template <int TT>
__global__ void __launch_bounds__(TT) dia_zc2(int n, const double* __restrict__ vals, const double* x, double* y) {
    __shared__ double2 xs2[(TT + 2 * H + 4) / 2];
    const double* xs = reinterpret_cast<const double*>(xs2);
    const int i0 = blockIdx.x * TT, i = i0 + threadIdx.x;
    const int w0 = (i0 - H) & ~1;
    const int nw = (TT + 2 * H + 4) / 2;
    for (int j = threadIdx.x; j < nw; j += TT) {
        const int c = w0 + 2 * j;
        double2 v;
        if (c >= 0 && c + 1 < n) v = *reinterpret_cast<const double2*>(x + c);
        else {
            v.x = (c >= 0 && c < n) ? x[c] : 0.0;
            v.y = (c + 1 >= 0 && c + 1 < n) ? x[c + 1] : 0.0;
        }
        xs2[j] = v;
    }
    __syncthreads();
    if (i >= n) return;
    const int base = i - H - w0;
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
        const int c = i + d - H;
        const double v = __ldcs(vals + size_t(d) * n + i);
        acc = __dadd_rn(acc, (unsigned)c < (unsigned)n ? __dmul_rn(v, xs[base + d]) : -0.0);
    }
    y[i] = acc;
}

template <class F>
float best_of(int reps, F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float t;
        cudaEventElapsedTime(&t, a, b);
        best = std::min(best, t);
    }
    return best;
}

int main() {
    const int n = 4000000;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *vals, *xh, *yh, *xd, *yd, *xm, *ym, *yref;
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    cudaMalloc(&vals, size_t(ND) * n * 8);
    cudaHostAlloc(&xh, n * 8, cudaHostAllocMapped);
    cudaHostAlloc(&yh, n * 8, cudaHostAllocMapped);
    cudaHostAlloc(&yref, n * 8, 0);
    cudaHostGetDevicePointer(&xm, xh, 0);
    cudaHostGetDevicePointer(&ym, yh, 0);
    cudaMalloc(&xd, n * 8);
    cudaMalloc(&yd, n * 8);
    {
        double* hv = (double*)malloc(size_t(ND) * n * 8);
        for (size_t k = 0; k < size_t(ND) * n; ++k) hv[k] = 0.5 + double((k * 2654435761u) % 1000) / 700.0;
        cudaMemcpy(vals, hv, size_t(ND) * n * 8, cudaMemcpyHostToDevice);
        free(hv);
    }
    for (int i = 0; i < n; ++i) xh[i] = 1.0 + double(i % 17) / 16.0;
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    const size_t B = size_t(n) * 8;
    printf("copy engine: H2D %.3f ms, D2H %.3f ms\n",
           best_of(5, [&] { cudaMemcpyAsync(xd, xh, B, cudaMemcpyHostToDevice, 0); }),
           best_of(5, [&] { cudaMemcpyAsync(yh, yd, B, cudaMemcpyDeviceToHost, 0); }));
    printf("copy engine duplex: %.3f ms\n", best_of(5, [&] {
               cudaEvent_t e;
               cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
               cudaEventRecord(e, 0);
               cudaStreamWaitEvent(s1, e, 0);
               cudaStreamWaitEvent(s2, e, 0);
               cudaMemcpyAsync(xd, xh, B, cudaMemcpyHostToDevice, s1);
               cudaMemcpyAsync(yh, yd, B, cudaMemcpyDeviceToHost, s2);
               cudaEventRecord(e, s1);
               cudaStreamWaitEvent(0, e, 0);
               cudaEventRecord(e, s2);
               cudaStreamWaitEvent(0, e, 0);
           }));
    // reference y (device-resident inputs)
    dia_zc2<1024><<<(n + 1023) / 1024, 1024>>>(n, vals, xd, yd);
    cudaMemcpy(yref, yd, B, cudaMemcpyDeviceToHost);
    printf("product scheme zc2<1024> x,y host: %.3f ms\n",
           best_of(6, [&] { dia_zc2<1024><<<(n + 1023) / 1024, 1024>>>(n, vals, xm, ym); }));
    for (int S : {2, 4, 8})
        for (uint32_t ch : {4096u, 16384u, 65536u})
            for (int per : {1, 2, 4}) {
                const int g = sms * per;
                float t = 0;
                if (S == 2) {
                    cudaFuncSetAttribute(bulk_read<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * ch);
                    t = best_of(4, [&] { bulk_read<2><<<g, 32, 2 * ch>>>((const char*)xm, B, ch, sink); });
                } else if (S == 4) {
                    if (4 * ch > 200000) continue;
                    cudaFuncSetAttribute(bulk_read<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * ch);
                    t = best_of(4, [&] { bulk_read<4><<<g, 32, 4 * ch>>>((const char*)xm, B, ch, sink); });
                } else {
                    if (8 * ch > 200000) continue;
                    cudaFuncSetAttribute(bulk_read<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * ch);
                    t = best_of(4, [&] { bulk_read<8><<<g, 32, 8 * ch>>>((const char*)xm, B, ch, sink); });
                }
                printf("bulk read host S=%d ch=%6u grid=%4d: %.3f ms %.1f GB/s (%s)\n", S, ch, g, t, B / t / 1e6,
                       cudaGetErrorString(cudaGetLastError()));
            }
    auto check = [&](const char* tag) {
        cudaDeviceSynchronize();
        size_t bad = 0;
        for (int i = 0; i < n; ++i) bad += yh[i] != yref[i];
        printf("  %s: bad=%zu (%s)\n", tag, bad, cudaGetErrorString(cudaGetLastError()));
    };
#define RUN_TMA(TR, S, YB, PER)                                                                        \
    {                                                                                                  \
        const size_t sm = size_t(S) * (TR + 2 * H + 4) * 8 + (YB ? 2 * TR * 8 : 0);                   \
        cudaFuncSetAttribute(dia_tma<TR, S, YB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)); \
        const int g = std::min((n + TR - 1) / TR, sms * PER);                                          \
        memset(yh, 0, B);                                                                              \
        float t = best_of(6, [&] { dia_tma<TR, S, YB><<<g, TR, sm>>>(n, vals, xm, ym); });             \
        printf("dia_tma TR=%d S=%d YB=%d per=%d: %.3f ms\n", TR, S, YB, PER, t);                       \
        check("host x,y");                                                                             \
        t = best_of(6, [&] { dia_tma<TR, S, YB><<<g, TR, sm>>>(n, vals, xm, yd); });                   \
        printf("  x host only: %.3f ms\n", t);                                                         \
    }
    RUN_TMA(1024, 2, 0, 1)
    RUN_TMA(1024, 4, 0, 1)
    RUN_TMA(1024, 4, 1, 1)
    RUN_TMA(512, 4, 0, 2)
    RUN_TMA(512, 8, 0, 2)
    RUN_TMA(512, 8, 1, 2)
    RUN_TMA(256, 8, 0, 4)
    RUN_TMA(256, 8, 1, 4)
    RUN_TMA(1024, 8, 0, 1)
    RUN_TMA(1024, 8, 1, 1)
    return 0;
}
