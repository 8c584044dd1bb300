// Diagnostic: DIA spmv (config-2 shape: n = 4M, offsets -13..13) reading x
// straight from mapped pinned host memory and writing y straight into it
// (no copy engine), vs the device-resident kernel.  Variants: direct x loads
// (relies on caching of sysmem lines) and a per-CTA shared-memory window.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/zc_probe scripts/zc_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>
#include <algorithm>

constexpr int H = 13, ND = 2 * H + 1, T = 256;

// x window of a CTA with 16-byte loads (window start rounded down to even)
template <int TT>
__global__ void __launch_bounds__(TT) dia_zc2(int n, const double* __restrict__ vals, const double* x, double* y) {
    __shared__ double2 xs2[(TT + 2 * H + 4) / 2];
    const double* xs = reinterpret_cast<const double*>(xs2);
    const int i0 = blockIdx.x * TT, i = i0 + threadIdx.x;
    const int w0 = (i0 - H) & ~1;  // even
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

// as dia_zc2, but the 27 values are loaded into registers BEFORE the x
// window (PCIe latency overlaps the HBM latency)
template <int TT, int MINB>
__global__ void __launch_bounds__(TT, MINB) dia_zc3(int n, const double* __restrict__ vals, const double* x, double* y) {
    __shared__ double2 xs2[(TT + 2 * H + 4) / 2];
    const double* xs = reinterpret_cast<const double*>(xs2);
    const int i0 = blockIdx.x * TT, i = i0 + threadIdx.x;
    double v[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) v[d] = i < n ? __ldcs(vals + size_t(d) * n + i) : 0.0;
    const int w0 = (i0 - H) & ~1;
    const int nw = (TT + 2 * H + 4) / 2;
    for (int j = threadIdx.x; j < nw; j += TT) {
        const int c = w0 + 2 * j;
        double2 t;
        if (c >= 0 && c + 1 < n) t = *reinterpret_cast<const double2*>(x + c);
        else {
            t.x = (c >= 0 && c < n) ? x[c] : 0.0;
            t.y = (c + 1 >= 0 && c + 1 < n) ? x[c + 1] : 0.0;
        }
        xs2[j] = t;
    }
    __syncthreads();
    if (i >= n) return;
    const int base = i - H - w0;
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
        const int c = i + d - H;
        acc = __dadd_rn(acc, (unsigned)c < (unsigned)n ? __dmul_rn(v[d], xs[base + d]) : -0.0);
    }
    y[i] = acc;
}

template <int TT>
__global__ void __launch_bounds__(TT, 4) dia_zc_rows(int n, int lo, int hi, const double* __restrict__ vals,
                                                    const double* x, double* y) {
    __shared__ double2 xs2[(TT + 2 * H + 4) / 2];
    const double* xs = reinterpret_cast<const double*>(xs2);
    const int i0 = lo + blockIdx.x * TT, i = i0 + threadIdx.x;
    double v[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) v[d] = i < hi ? __ldcs(vals + size_t(d) * n + i) : 0.0;
    const int w0 = (i0 - H) & ~1;
    const int nw = (TT + 2 * H + 4) / 2;
    for (int j = threadIdx.x; j < nw; j += TT) {
        const int c = w0 + 2 * j;
        double2 t;
        if (c >= 0 && c + 1 < n) t = *reinterpret_cast<const double2*>(x + c);
        else {
            t.x = (c >= 0 && c < n) ? x[c] : 0.0;
            t.y = (c + 1 >= 0 && c + 1 < n) ? x[c + 1] : 0.0;
        }
        xs2[j] = t;
    }
    __syncthreads();
    if (i >= hi) return;
    const int base = i - H - w0;
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
        const int c = i + d - H;
        acc = __dadd_rn(acc, (unsigned)c < (unsigned)n ? __dmul_rn(v[d], xs[base + d]) : -0.0);
    }
    y[i] = acc;
}

template <int TT>
__global__ void __launch_bounds__(TT) dia_rows(int n, int lo, int hi, const double* __restrict__ vals,
                                              const double* __restrict__ x, double* y) {
    const int i = lo + blockIdx.x * TT + threadIdx.x;
    if (i >= hi) return;
    double v[ND], xv[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) {
        const int c = i + d - H;
        v[d] = __ldcs(vals + size_t(d) * n + i);
        xv[d] = __ldg(x + ((unsigned)c < (unsigned)n ? c : 0));
    }
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
        const int c = i + d - H;
        acc = __dadd_rn(acc, (unsigned)c < (unsigned)n ? __dmul_rn(v[d], xv[d]) : -0.0);
    }
    y[i] = acc;
}

template <int MODE>  // 0 direct, 1 smem window
__global__ void __launch_bounds__(T) dia_zc(int n, const double* __restrict__ vals, const double* x, double* y) {
    __shared__ double xs[T + 2 * H];
    const int i0 = blockIdx.x * T, i = i0 + threadIdx.x;
    if (MODE == 1) {
        for (int j = threadIdx.x; j < T + 2 * H; j += T) {
            const int c = i0 - H + j;
            xs[j] = (c >= 0 && c < n) ? x[c] : 0.0;
        }
        __syncthreads();
    }
    if (i >= n) return;
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
        const int c = i + d - H;
        const double v = __ldcs(vals + size_t(d) * n + i);
        const double xv = MODE == 1 ? xs[threadIdx.x + d] : ((unsigned)c < (unsigned)n ? x[c] : 0.0);
        acc = __dadd_rn(acc, (unsigned)c < (unsigned)n ? __dmul_rn(v, xv) : -0.0);
    }
    y[i] = acc;
}

int main() {
    const int n = 4000000;
    double *vals, *xh, *yh, *xd, *yd, *xm, *ym;
    cudaMalloc(&vals, size_t(ND) * n * 8);
    cudaMemset(vals, 0, size_t(ND) * n * 8);
    cudaHostAlloc(&xh, n * 8, cudaHostAllocMapped);
    cudaHostAlloc(&yh, n * 8, cudaHostAllocMapped);
    cudaHostGetDevicePointer(&xm, xh, 0);
    cudaHostGetDevicePointer(&ym, yh, 0);
    cudaMalloc(&xd, n * 8);
    cudaMalloc(&yd, n * 8);
    for (int i = 0; i < n; ++i) xh[i] = 1.0;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = (n + T - 1) / T;
    for (int v = 0; v < 16; ++v) {
        float best = 1e9;
        for (int rep = 0; rep < 6; ++rep) {
            cudaEventRecord(a);
            switch (v) {
                case 0: dia_zc<0><<<grid, T>>>(n, vals, xd, yd); break;  // device resident
                case 1: dia_zc<1><<<grid, T>>>(n, vals, xd, yd); break;
                case 2: dia_zc<0><<<grid, T>>>(n, vals, xm, ym); break;  // zero-copy x and y
                case 3: dia_zc<1><<<grid, T>>>(n, vals, xm, ym); break;
                case 4: dia_zc<1><<<grid, T>>>(n, vals, xm, yd); break;  // zero-copy x only
                case 5: dia_zc<1><<<grid, T>>>(n, vals, xd, ym); break;  // zero-copy y only
                case 6: dia_zc2<256><<<grid, 256>>>(n, vals, xm, ym); break;
                case 7: dia_zc2<256><<<grid, 256>>>(n, vals, xm, yd); break;
                case 8: dia_zc2<512><<<(n + 511) / 512, 512>>>(n, vals, xm, ym); break;
                case 9: dia_zc2<1024><<<(n + 1023) / 1024, 1024>>>(n, vals, xm, ym); break;
                case 10: dia_zc3<256, 4><<<grid, 256>>>(n, vals, xm, ym); break;
                case 11: dia_zc3<256, 3><<<grid, 256>>>(n, vals, xm, ym); break;
                case 12: dia_zc3<128, 8><<<(n + 127) / 128, 128>>>(n, vals, xm, ym); break;
                case 13: dia_zc3<256, 4><<<grid, 256>>>(n, vals, xm, yd); break;
                case 14: dia_zc3<256, 4><<<grid, 256>>>(n, vals, xd, ym); break;
                case 15: dia_zc3<512, 2><<<(n + 511) / 512, 512>>>(n, vals, xm, ym); break;
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float t;
            cudaEventElapsedTime(&t, a, b);
            if (t < best) best = t;
        }
        printf("variant %d: %.3f ms  (%s)\n", v, best, cudaGetErrorString(cudaGetLastError()));
    }
    // chunked: x up on the copy engine in K pieces, kernel k waits for its
    // piece and writes y straight to mapped host memory (ymode 1) or to the
    // device with a D2H copy per chunk (ymode 0)
    cudaStream_t s0, ci, co;
    cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&ci, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&co, cudaStreamNonBlocking);
    std::vector<cudaEvent_t> ev(80);
    for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    for (int ymode = 0; ymode < 2; ++ymode)
        for (int K : {2, 4, 8, 16, 32}) {
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                cudaDeviceSynchronize();
                cudaEventRecord(a, s0);
                cudaStreamWaitEvent(ci, a, 0);
                cudaStreamWaitEvent(co, a, 0);
                const int per = (n + K - 1) / K;
                int xhi = 0;
                for (int k = 0; k < K; ++k) {
                    const int hi = k + 1 == K ? n : std::min(n, (k + 1) * per + H);
                    cudaMemcpyAsync(xd + xhi, xh + xhi, size_t(hi - xhi) * 8, cudaMemcpyHostToDevice, ci);
                    xhi = hi;
                    cudaEventRecord(ev[k], ci);
                }
                for (int k = 0; k < K; ++k) {
                    const int lo = k * per, hi = std::min(n, lo + per);
                    cudaStreamWaitEvent(s0, ev[k], 0);
                    dia_rows<256><<<(hi - lo + 255) / 256, 256, 0, s0>>>(n, lo, hi, vals, xd, ymode ? ym : yd);
                    if (!ymode) {
                        cudaEventRecord(ev[40 + k], s0);
                        cudaStreamWaitEvent(co, ev[40 + k], 0);
                        cudaMemcpyAsync(yh + lo, yd + lo, size_t(hi - lo) * 8, cudaMemcpyDeviceToHost, co);
                    }
                }
                cudaEventRecord(ev[39], co);
                cudaStreamWaitEvent(s0, ev[39], 0);
                cudaEventRecord(b, s0);
                cudaEventSynchronize(b);
                float t;
                cudaEventElapsedTime(&t, a, b);
                if (t < best) best = t;
            }
            printf("chunked ymode %d K %2d: %.3f ms (%s)\n", ymode, K, best, cudaGetErrorString(cudaGetLastError()));
        }
    // split: rows [0, f*n) read x from host (zero copy) while the copy engine
    // uploads x[f*n - H, n); rows [f*n, n) then run on the device copy; y
    // written to mapped host memory throughout
    for (int pct : {20, 30, 40, 50, 60, 70}) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, s0);
            cudaStreamWaitEvent(ci, a, 0);
            const int cut = int(int64_t(n) * pct / 100);
            const int x0 = std::max(0, cut - H);
            cudaMemcpyAsync(xd + x0, xh + x0, size_t(n - x0) * 8, cudaMemcpyHostToDevice, ci);
            cudaEventRecord(ev[0], ci);
            dia_zc_rows<256><<<(cut + 255) / 256, 256, 0, s0>>>(n, 0, cut, vals, xm, ym);
            cudaStreamWaitEvent(s0, ev[0], 0);
            dia_rows<256><<<(n - cut + 255) / 256, 256, 0, s0>>>(n, cut, n, vals, xd, ym);
            cudaEventRecord(b, s0);
            cudaEventSynchronize(b);
            float t;
            cudaEventElapsedTime(&t, a, b);
            if (t < best) best = t;
        }
        printf("split %d%%: %.3f ms (%s)\n", pct, best, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
