// Diagnostic: the pinned-buffer spmv pipeline (capi.cu spmv_pipelined)
// rebuilt outside the library with timing events on every stage, on the
// config-2 DIA matrix (27 diagonals, n = 4M) generated on the device.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -Iinclude -o build/pipe_probe scripts/pipe_probe.cu \
//        -Lpaper_2303_05098_b200/lib -lsparseoracle_b200 -Xlinker -rpath,'$ORIGIN/../paper_2303_05098_b200/lib'
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

#include "sparseoracle_b200.h"

int main() {
    const int64_t n = 4000000, h = 13, nd = 2 * h + 1;
    std::vector<int64_t> off(nd);
    for (int d = 0; d < nd; ++d) off[d] = d - h;
    std::vector<double> vals(size_t(nd) * n, 1.0);
    so_matrix* m = nullptr;
    if (so_matrix_upload_dia(n, n, nd, off.data(), vals.data(), nd * n, &m) != SO_OK) {
        printf("upload: %s\n", so_last_error());
        return 1;
    }
    double *x, *y, *dx, *dy;
    cudaHostAlloc(&x, n * 8, 0);
    cudaHostAlloc(&y, n * 8, 0);
    cudaMalloc(&dx, n * 8);
    cudaMalloc(&dy, n * 8);
    for (int64_t i = 0; i < n; ++i) x[i] = 1.0;
    cudaStream_t s, ci, co;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&ci, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&co, cudaStreamNonBlocking);
    {  // plain duplex: one 32 MB copy each way, concurrently, synced per rep
        cudaEvent_t a, b1, b2;
        cudaEventCreate(&a); cudaEventCreate(&b1); cudaEventCreate(&b2);
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(a, s);
            cudaStreamWaitEvent(ci, a, 0);
            cudaStreamWaitEvent(co, a, 0);
            cudaMemcpyAsync(dx, x, n * 8, cudaMemcpyHostToDevice, ci);
            cudaMemcpyAsync(y, dy, n * 8, cudaMemcpyDeviceToHost, co);
            cudaEventRecord(b1, ci);
            cudaEventRecord(b2, co);
            cudaEventSynchronize(b1);
            cudaEventSynchronize(b2);
            float t1, t2;
            cudaEventElapsedTime(&t1, a, b1);
            cudaEventElapsedTime(&t2, a, b2);
            printf("duplex 32+32 MB: h2d %.3f ms, d2h %.3f ms\n", t1, t2);
        }
        for (int rep = 0; rep < 2; ++rep) {  // chunked, no dependencies
            cudaEventRecord(a, s);
            cudaStreamWaitEvent(ci, a, 0);
            cudaStreamWaitEvent(co, a, 0);
            for (int k = 0; k < 16; ++k) {
                cudaMemcpyAsync(dx + k * (n / 16), x + k * (n / 16), (n / 16) * 8, cudaMemcpyHostToDevice, ci);
                cudaMemcpyAsync(y + k * (n / 16), dy + k * (n / 16), (n / 16) * 8, cudaMemcpyDeviceToHost, co);
            }
            cudaEventRecord(b1, ci);
            cudaEventRecord(b2, co);
            cudaEventSynchronize(b1);
            cudaEventSynchronize(b2);
            float t1, t2;
            cudaEventElapsedTime(&t1, a, b1);
            cudaEventElapsedTime(&t2, a, b2);
            printf("duplex 16x(2+2) MB: h2d %.3f ms, d2h %.3f ms\n", t1, t2);
        }
    }
    {  // chunked with dependencies but no kernels: d2h k waits on h2d k
        cudaEvent_t a, b1, b2;
        cudaEventCreate(&a); cudaEventCreate(&b1); cudaEventCreate(&b2);
        std::vector<cudaEvent_t> e(16);
        for (auto& q : e) cudaEventCreateWithFlags(&q, cudaEventDisableTiming);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a, s);
            cudaStreamWaitEvent(ci, a, 0);
            cudaStreamWaitEvent(co, a, 0);
            for (int k = 0; k < 16; ++k) {
                cudaMemcpyAsync(dx + k * (n / 16), x + k * (n / 16), (n / 16) * 8, cudaMemcpyHostToDevice, ci);
                cudaEventRecord(e[k], ci);
            }
            for (int k = 0; k < 16; ++k) {
                cudaStreamWaitEvent(co, e[k], 0);
                cudaMemcpyAsync(y + k * (n / 16), dy + k * (n / 16), (n / 16) * 8, cudaMemcpyDeviceToHost, co);
            }
            cudaEventRecord(b1, ci);
            cudaEventRecord(b2, co);
            cudaEventSynchronize(b1);
            cudaEventSynchronize(b2);
            float t1, t2;
            cudaEventElapsedTime(&t1, a, b1);
            cudaEventElapsedTime(&t2, a, b2);
            printf("dep-chunked no kernels: h2d %.3f ms, d2h %.3f ms\n", t1, t2);
        }
    }
    double* ymapped = nullptr;
    cudaHostGetDevicePointer((void**)&ymapped, y, 0);
    printf("y %p mapped %p\n", (void*)y, (void*)ymapped);
    for (int mode = 0; mode < 3; ++mode)
    for (int nch : {1, 4, 8, 16, 32}) {
        const int64_t rows = (n + nch - 1) / nch;
        std::vector<cudaEvent_t> ein(nch), ek(nch);
        for (auto& e : ein) cudaEventCreate(&e);
        for (auto& e : ek) cudaEventCreate(&e);
        cudaEvent_t t0, tin, tk, tout;
        cudaEventCreate(&t0);
        cudaEventCreate(&tin);
        cudaEventCreate(&tk);
        cudaEventCreate(&tout);
        for (int rep = 0; rep < 4; ++rep) {
            auto w0 = std::chrono::steady_clock::now();
            cudaEventRecord(t0, s);
            cudaStreamWaitEvent(ci, t0, 0);
            cudaStreamWaitEvent(co, t0, 0);
            int64_t xh = 0;
            for (int k = 0; k < nch; ++k) {
                const int64_t b = std::min(n, (k + 1) * rows);
                const int64_t want = k + 1 == nch ? n : std::min(n, b + h);
                cudaMemcpyAsync(dx + xh, x + xh, (want - xh) * 8, cudaMemcpyHostToDevice, ci);
                xh = want;
                cudaEventRecord(ein[k], ci);
            }
            cudaEventRecord(tin, ci);
            for (int k = 0; k < nch; ++k) {
                const int64_t a = k * rows, b = std::min(n, a + rows);
                cudaStreamWaitEvent(s, ein[k], 0);
                if (mode == 2) {  // rows written straight into the mapped host y (no read-back copy)
                    so_spmv_device_rows(m, dx, ymapped, a, b, s);
                    continue;
                }
                so_spmv_device_rows(m, dx, dy, a, b, s);
                if (mode == 0) {  // read-back on its own copy stream
                    cudaEventRecord(ek[k], s);
                    cudaStreamWaitEvent(co, ek[k], 0);
                    cudaMemcpyAsync(y + a, dy + a, (b - a) * 8, cudaMemcpyDeviceToHost, co);
                } else {  // read-back on the compute stream
                    cudaMemcpyAsync(y + a, dy + a, (b - a) * 8, cudaMemcpyDeviceToHost, s);
                }
            }
            cudaEventRecord(tk, s);
            if (mode == 0) cudaEventRecord(tout, co); else cudaEventRecord(tout, s);
            if (mode == 2 && rep == 3) {
                cudaEventSynchronize(tout);
                double bad = 0;
                for (int64_t i = 0; i < n; ++i) bad += (y[i] != (i < h || i >= n - h ? y[i] : 27.0));
                printf("  mapped y check: %g mismatches (interior rows == 27)\n", bad);
            }
            auto w1 = std::chrono::steady_clock::now();
            cudaEventSynchronize(tout);
            auto w2 = std::chrono::steady_clock::now();
            float a1, a2, a3;
            cudaEventElapsedTime(&a1, t0, tin);
            cudaEventElapsedTime(&a2, t0, tk);
            cudaEventElapsedTime(&a3, t0, tout);
            printf("mode %d chunks %2d: h2d done %.3f  kernels done %.3f  d2h done %.3f ms | host enqueue %.3f ms, wall %.3f ms\n",
                   mode, nch, a1, a2, a3, std::chrono::duration<double, std::milli>(w1 - w0).count(),
                   std::chrono::duration<double, std::milli>(w2 - w0).count());
        }
    }
    return 0;
}
