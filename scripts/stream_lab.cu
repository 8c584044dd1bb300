// Stream lab (not the product): the fastest cold read of B bytes (+ a write of
// W bytes) one kernel achieves on this B200, for the byte counts of the config
// 1 matrices (56-96 MB: 10-15 us kernels) up to config 2 (0.9-1.8 GB).  This is
// the size-matched floor the small-matrix SpMV numbers are compared against
// (DESIGN.md §7): at 10 us, launch, ramp-up and tail are a visible share.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/stream_lab scripts/stream_lab.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ void ld256(const double* p, double (&v)[4]) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}

// each thread reads U 32-byte vectors (grid-stride) and writes one double per
// `wratio` doubles read (the y stream of an SpMV)
template <int U>
__global__ void __launch_bounds__(256) stream_read(const double* __restrict__ a, int64_t n4, double* __restrict__ y,
                                                   int64_t ny) {
    double acc = 0.0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n4; i += U * stride) {
        double v[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) ld256(a + 4 * (i + u * stride), v[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u][0] + v[u][1] + v[u][2] + v[u][3];
    }
    for (; i < n4; i += stride) {
        double v[4];
        ld256(a + 4 * i, v);
        acc += v[0] + v[1] + v[2] + v[3];
    }
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < ny; j += stride) y[j] = acc;
}

// L2 eviction without dirty lines (a write flush leaves ~L2 of dirty lines
// that are written back during the next kernel)
__global__ void flush_kernel(const double* p, int64_t n, double* sink) {
    double s = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        s += p[i];  // plain loads: allocate in L2 and evict what was there
    if (s == 1.2345) *sink = s;
}

int main() {
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t kFlush = size_t(512) << 20;
    double* flush; CK(cudaMalloc(&flush, kFlush));
    CK(cudaMemset(flush, 0, kFlush));
    double* big; const size_t kBig = size_t(2000) << 20; CK(cudaMalloc(&big, kBig));
    CK(cudaMemset(big, 0, kBig));
    double* y; CK(cudaMalloc(&y, size_t(64) << 20));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const double peak = getenv("LAB_PEAK") ? atof(getenv("LAB_PEAK")) : 6539.5;
    // (read MB, write MB): config 1 DIA 48+8, CSR 72+8, COO 88+8, config 2 DIA 896+32
    const double cases[][2] = {{8, 8}, {24, 8}, {48, 8}, {64, 8}, {88, 8}, {200, 32}, {896, 32}, {1760, 32}};
    printf("cold = after a 512 MB read flush; best grid of {1,2,4,8,16} CTAs/SM x U in {2,4}\n");
    for (auto& c : cases) {
        const int64_t n4 = int64_t(c[0] * (1 << 20) / 32), ny = int64_t(c[1] * (1 << 20) / 8);
        float best = 1e9; int bb = 0, bu = 0;
        for (int per : {1, 2, 4, 8, 16})
            for (int U : {2, 4}) {
                float tot = 0; const int reps = 10;
                for (int r = 0; r < reps + 2; ++r) {
                    flush_kernel<<<sms * 4, 256>>>(flush, int64_t(kFlush / 8), y);
                    cudaEventRecord(e0);
                    if (U == 2) stream_read<2><<<sms * per, 256>>>(big, n4, y, ny);
                    else stream_read<4><<<sms * per, 256>>>(big, n4, y, ny);
                    cudaEventRecord(e1);
                    CK(cudaEventSynchronize(e1));
                    float ms; cudaEventElapsedTime(&ms, e0, e1);
                    if (r >= 2) tot += ms;
                }
                const float t = tot / reps;
                if (t < best) { best = t; bb = per; bu = U; }
            }
        const double bytes = (c[0] + c[1]) * (1 << 20);
        printf("  read %6.0f MB + write %4.0f MB: %8.2f us  %7.0f GB/s  %.3f of peak  (%d CTAs/SM, U=%d)\n", c[0], c[1],
               best * 1e3, bytes / (best * 1e-3) / 1e9, bytes / (best * 1e-3) / 1e9 / peak, bb, bu);
    }
    CK(cudaGetLastError());
    return 0;
}
