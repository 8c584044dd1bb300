// Microbenchmark: DIA SpMV kernel variants on the config-2 shape
// (n = 4M rows, 27 diagonals -13..13), fp64.  Standalone, not the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/diav scripts/dia_variants.cu && /tmp/diav
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ double lds(const double* p) {
    double v; asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v;
}

// (a) one row per thread, U diagonals loaded before accumulation
template <int U>
__global__ void __launch_bounds__(256) dia_a(int64_t n, int D, const int64_t* __restrict__ off,
                                             const double* __restrict__ v, const double* __restrict__ x, double* __restrict__ y) {
    __shared__ int64_t so[64];
    if (threadIdx.x < D) so[threadIdx.x] = off[threadIdx.x];
    __syncthreads();
    int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    int d0 = 0;
    for (; d0 + U <= D; d0 += U) {
        double a[U], b[U]; bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int64_t c = i + so[d0 + u];
            ok[u] = c >= 0 && c < n;
            int64_t cc = c < 0 ? 0 : (c >= n ? n - 1 : c);
            a[u] = lds(v + int64_t(d0 + u) * n + i);
            b[u] = __ldg(x + cc);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, ok[u] ? __dmul_rn(a[u], b[u]) : -0.0);
    }
    for (; d0 < D; ++d0) {
        int64_t c = i + so[d0];
        if (c >= 0 && c < n) acc = __dadd_rn(acc, __dmul_rn(lds(v + int64_t(d0) * n + i), __ldg(x + c)));
    }
    y[i] = acc;
}

// (a') masked tail: every chunk is a full U-wide batch of loads
template <int U>
__global__ void __launch_bounds__(256) dia_am(int64_t n, int D, const int64_t* __restrict__ off,
                                              const double* __restrict__ v, const double* __restrict__ x, double* __restrict__ y) {
    __shared__ int64_t so[64];
    if (threadIdx.x < D) so[threadIdx.x] = off[threadIdx.x];
    __syncthreads();
    int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    for (int d0 = 0; d0 < D; d0 += U) {
        double a[U], b[U]; bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int d = d0 + u < D ? d0 + u : D - 1;
            int64_t c = i + so[d];
            ok[u] = d0 + u < D && c >= 0 && c < n;
            int64_t cc = c < 0 ? 0 : (c >= n ? n - 1 : c);
            a[u] = lds(v + int64_t(d) * n + i);
            b[u] = __ldg(x + cc);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc = __dadd_rn(acc, ok[u] ? __dmul_rn(a[u], b[u]) : -0.0);
    }
    y[i] = acc;
}

// (b) two consecutive rows per thread, 16-byte value loads
__global__ void __launch_bounds__(256) dia_b(int64_t n, int D, const int64_t* __restrict__ off,
                                             const double* __restrict__ v, const double* __restrict__ x, double* __restrict__ y) {
    __shared__ int64_t so[64];
    if (threadIdx.x < D) so[threadIdx.x] = off[threadIdx.x];
    __syncthreads();
    int64_t i = 2 * (int64_t(blockIdx.x) * 256 + threadIdx.x);
    if (i >= n) return;  // n even here
    double a0 = 0.0, a1 = 0.0;
    constexpr int U = 8;
    int d0 = 0;
    for (; d0 + U <= D; d0 += U) {
        double2 a[U]; double b0[U], b1[U]; bool o0[U], o1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int64_t c = i + so[d0 + u];
            o0[u] = c >= 0 && c < n;
            o1[u] = c + 1 >= 0 && c + 1 < n;
            int64_t c0 = c < 0 ? 0 : (c >= n ? n - 1 : c);
            int64_t c1 = c + 1 < 0 ? 0 : (c + 1 >= n ? n - 1 : c + 1);
            a[u] = __ldcs(reinterpret_cast<const double2*>(v + int64_t(d0 + u) * n + i));
            b0[u] = __ldg(x + c0);
            b1[u] = __ldg(x + c1);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            a0 = __dadd_rn(a0, o0[u] ? __dmul_rn(a[u].x, b0[u]) : -0.0);
            a1 = __dadd_rn(a1, o1[u] ? __dmul_rn(a[u].y, b1[u]) : -0.0);
        }
    }
    for (; d0 < D; ++d0) {
        int64_t c = i + so[d0];
        double2 a = __ldcs(reinterpret_cast<const double2*>(v + int64_t(d0) * n + i));
        if (c >= 0 && c < n) a0 = __dadd_rn(a0, __dmul_rn(a.x, __ldg(x + c)));
        if (c + 1 >= 0 && c + 1 < n) a1 = __dadd_rn(a1, __dmul_rn(a.y, __ldg(x + c + 1)));
    }
    reinterpret_cast<double2*>(y)[i / 2] = make_double2(a0, a1);
}

// (c) TMA bulk copies (cp.async.bulk) of each diagonal's R-row slice into a
// 2-stage shared-memory ring, mbarrier completion, persistent CTAs.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n"
                 ::"r"(smem_u32(b)), "r"(phase) : "memory");
}

template <int R, int DMAX>
__global__ void __launch_bounds__(R) dia_c(int64_t n, int D, const int64_t* __restrict__ off,
                                           const double* __restrict__ v, const double* __restrict__ x, double* __restrict__ y) {
    extern __shared__ __align__(128) unsigned char sm[];
    double* buf = reinterpret_cast<double*>(sm);          // [2][DMAX][R]
    uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 2 * DMAX * R);
    __shared__ int64_t so[64];
    if (threadIdx.x < D) so[threadIdx.x] = off[threadIdx.x];
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t ntiles = n / R;  // full tiles only (tail handled separately)
    auto issue = [&](int64_t tile, int s) {
        mbar_expect(&bar[s], uint32_t(D) * R * 8);
        for (int d = 0; d < D; ++d)
            bulk_g2s(buf + (s * DMAX + d) * R, v + int64_t(d) * n + tile * R, R * 8, &bar[s]);
    };
    int64_t t = blockIdx.x;
    if (threadIdx.x == 0 && t < ntiles) issue(t, 0);
    uint32_t ph[2] = {0, 0};
    int s = 0;
    for (; t < ntiles; t += gridDim.x) {
        const int64_t tn = t + gridDim.x;
        if (threadIdx.x == 0 && tn < ntiles) issue(tn, s ^ 1);
        mbar_wait(&bar[s], ph[s]);
        ph[s] ^= 1;
        const int64_t i = t * R + threadIdx.x;
        double acc = 0.0;
        const double* col = buf + s * DMAX * R + threadIdx.x;
#pragma unroll 9
        for (int d = 0; d < D; ++d) {
            int64_t c = i + so[d];
            bool ok = c >= 0 && c < n;
            int64_t cc = c < 0 ? 0 : (c >= n ? n - 1 : c);
            double xv = __ldg(x + cc);
            acc = __dadd_rn(acc, ok ? __dmul_rn(col[d * R], xv) : -0.0);
        }
        y[i] = acc;
        __syncthreads();  // everyone done with stage s before it is refilled
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        s ^= 1;
    }
}

int main() {
    const int64_t n = 4000000;
    const int D = 27;
    std::vector<int64_t> off(D);
    for (int d = 0; d < D; ++d) off[d] = d - 13;
    std::vector<double> hv(size_t(D) * n), hx(n);
    uint64_t st = 12345;
    auto rnd = [&]() { st = st * 6364136223846793005ULL + 1442695040888963407ULL; return double(st >> 11) * 0x1.0p-53; };
    for (auto& a : hv) a = 0.5 + 1.5 * rnd();
    for (auto& a : hx) a = rnd() - 0.5;
    int64_t *doff; double *dv, *dx, *dy, *dy2;
    CK(cudaMalloc(&doff, D * 8)); CK(cudaMalloc(&dv, hv.size() * 8)); CK(cudaMalloc(&dx, n * 8));
    CK(cudaMalloc(&dy, n * 8)); CK(cudaMalloc(&dy2, n * 8));
    CK(cudaMemcpy(doff, off.data(), D * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dv, hv.data(), hv.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dx, hx.data(), n * 8, cudaMemcpyHostToDevice));
    char* flush; size_t fl = size_t(512) << 20; CK(cudaMalloc(&flush, fl));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double bytes = 8.0 * (double(D) * n - 13 * 14) + 8.0 * D + 16.0 * n;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        float best = 1e9, tot = 0; int reps = 20;
        for (int r = 0; r < reps + 3; ++r) {
            CK(cudaMemsetAsync(flush, r, fl));
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 3) { tot += ms; if (ms < best) best = ms; }
        }
        CK(cudaGetLastError());
        std::vector<double> a(n), b(n);
        CK(cudaMemcpy(a.data(), dy, n * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(b.data(), dy2, n * 8, cudaMemcpyDeviceToHost));
        int64_t bad = 0; for (int64_t i = 0; i < n; ++i) bad += a[i] != b[i];
        printf("%-28s best %8.1f us avg %8.1f us  %7.0f GB/s (avg)  mismatches vs (a): %lld\n", name, best * 1e3,
               tot / reps * 1e3, bytes / (tot / reps * 1e-3) / 1e9, (long long)bad);
    };
    dia_a<8><<<(n + 255) / 256, 256>>>(n, D, doff, dv, dx, dy2);  // reference result in dy2
    CK(cudaDeviceSynchronize());
    run("a: 1 row/thr U=8", [&] { dia_a<8><<<(n + 255) / 256, 256>>>(n, D, doff, dv, dx, dy); });
    run("am: masked U=6", [&] { dia_am<6><<<(n + 255) / 256, 256>>>(n, D, doff, dv, dx, dy); });
    run("am: masked U=7", [&] { dia_am<7><<<(n + 255) / 256, 256>>>(n, D, doff, dv, dx, dy); });
    run("am: masked U=8", [&] { dia_am<8><<<(n + 255) / 256, 256>>>(n, D, doff, dv, dx, dy); });
    run("am: masked U=9", [&] { dia_am<9><<<(n + 255) / 256, 256>>>(n, D, doff, dv, dx, dy); });
    run("am: masked U=10", [&] { dia_am<10><<<(n + 255) / 256, 256>>>(n, D, doff, dv, dx, dy); });
    run("am: masked U=14", [&] { dia_am<14><<<(n + 255) / 256, 256>>>(n, D, doff, dv, dx, dy); });
    run("a: 1 row/thr U=16", [&] { dia_a<16><<<(n + 255) / 256, 256>>>(n, D, doff, dv, dx, dy); });
    run("a: 1 row/thr U=27", [&] { dia_a<27><<<(n + 255) / 256, 256>>>(n, D, doff, dv, dx, dy); });
    run("b: 2 rows/thr v2", [&] { dia_b<<<(n / 2 + 255) / 256, 256>>>(n, D, doff, dv, dx, dy); });
    {
        constexpr int R = 256, DM = 27;
        size_t smem = size_t(2) * DM * R * 8 + 64;
        CK(cudaFuncSetAttribute(dia_c<R, DM>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        for (int per : {1, 2}) {
            char nm[64]; snprintf(nm, 64, "c: TMA bulk R=256 %dCTA/SM", per);
            run(nm, [&] { dia_c<R, DM><<<sms * per, R, smem>>>(n, D, doff, dv, dx, dy); });
        }
    }
    {
        constexpr int R = 128, DM = 27;
        size_t smem = size_t(2) * DM * R * 8 + 64;
        CK(cudaFuncSetAttribute(dia_c<R, DM>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        for (int per : {2, 4}) {
            char nm[64]; snprintf(nm, 64, "c: TMA bulk R=128 %dCTA/SM", per);
            run(nm, [&] { dia_c<R, DM><<<sms * per, R, smem>>>(n, D, doff, dv, dx, dy); });
        }
    }
    // streaming-read calibration: same bytes, no compute
    return 0;
}
