// Diagnostic: does an HBM-saturating kernel slow concurrent PCIe copies?
// A 32 MB H2D and a 32 MB D2H (pinned) run beside a grid-stride streaming
// read of a 1 GB buffer launched on `sms` SMs (0 = no kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/hog_probe scripts/hog_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__global__ void hog(const double2* __restrict__ a, size_t n, int reps, double* out) {
    double s = 0;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
            const double2 v = __ldcs(a + i);
            s += v.x + v.y;
        }
    if (s == 12345.0) *out = s;
}

// persistent variant: block b handles slice b of every chunk; waits for the
// chunk's x flag (written by the copy stream), reads its data slice and x
// (through L2: the copy engine wrote it), writes y (device or mapped host),
// then counts itself done for the chunk (the read-back stream waits on it)
__global__ void pipe_kernel(const double2* __restrict__ a, size_t ck, const double* x, size_t cx, double* y,
                            const unsigned* flags, unsigned* done, unsigned epoch) {
    for (int k = 0; k < 16; ++k) {
        if (threadIdx.x == 0) {
            unsigned f;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(flags + k) : "memory");
            } while (f < epoch);
        }
        __syncthreads();
        double s = 0;
        const double2* ak = a + k * ck;
        for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < ck; i += size_t(gridDim.x) * blockDim.x) {
            const double2 v = __ldcs(ak + i);
            s += v.x + v.y;
        }
        for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < cx; i += size_t(gridDim.x) * blockDim.x)
            y[k * cx + i] = s + __ldcg(x + k * cx + i);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();
            atomicAdd(done + k, 1u);
        }
    }
}

int main() {
    const size_t nx = 4000000, nb = (size_t(1) << 30) / sizeof(double2);
    double *x, *y, *dx, *dy, *o;
    double2* big;
    cudaHostAlloc(&x, nx * 8, 0);
    cudaHostAlloc(&y, nx * 8, 0);
    cudaMalloc(&dx, nx * 8);
    cudaMalloc(&dy, nx * 8);
    cudaMalloc(&o, 8);
    cudaMalloc(&big, nb * sizeof(double2));
    cudaMemset(big, 0, nb * sizeof(double2));
    cudaStream_t s, ci, co;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&ci, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&co, cudaStreamNonBlocking);
    cudaEvent_t a, b1, b2, k0, k1;
    cudaEventCreate(&a); cudaEventCreate(&b1); cudaEventCreate(&b2);
    cudaEventCreate(&k0); cudaEventCreate(&k1);
    const int sms_list[] = {0, 8, 16, 32, 64, 148, 296, 888};
    for (int sms : sms_list) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, s);
            cudaStreamWaitEvent(ci, a, 0);
            cudaStreamWaitEvent(co, a, 0);
            cudaEventRecord(k0, s);
            if (sms) hog<<<sms, 512, 0, s>>>(big, nb, sms >= 148 ? 6 : 1, o);
            cudaEventRecord(k1, s);
            cudaMemcpyAsync(dx, x, nx * 8, cudaMemcpyHostToDevice, ci);
            cudaMemcpyAsync(y, dy, nx * 8, cudaMemcpyDeviceToHost, co);
            cudaEventRecord(b1, ci);
            cudaEventRecord(b2, co);
            cudaDeviceSynchronize();
            float t1, t2, tk;
            cudaEventElapsedTime(&t1, a, b1);
            cudaEventElapsedTime(&t2, a, b2);
            cudaEventElapsedTime(&tk, k0, k1);
            if (rep == 2)
                printf("hog ctas %4d: kernel %.3f ms (%.0f GB/s)  h2d %.3f ms  d2h %.3f ms\n", sms, tk,
                       sms ? (sms >= 148 ? 6.0 : 1.0) * nb * 16 / tk / 1e6 : 0.0, t1, t2);
        }
    }
    // the spmv pipeline's shape: 16 x-chunks up on ci, a 58 MB streaming
    // kernel per chunk on s (waiting for its chunk when `dep`), 16 y-chunks
    // down on co behind each kernel; kernel grid = `ctas`
    std::vector<cudaEvent_t> ev(64);
    for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    const size_t cx = nx / 16, ck = size_t(928) * 1000000 / 16 / sizeof(double2);
    for (int dep = 0; dep < 2; ++dep)
        for (int ctas : {148, 296, 592, 888, 1776}) {
            float t1 = 0, t2 = 0;
            for (int rep = 0; rep < 3; ++rep) {
                cudaDeviceSynchronize();
                cudaEventRecord(a, s);
                cudaStreamWaitEvent(ci, a, 0);
                cudaStreamWaitEvent(co, a, 0);
                for (int k = 0; k < 16; ++k) {
                    cudaMemcpyAsync(dx + k * cx, x + k * cx, cx * 8, cudaMemcpyHostToDevice, ci);
                    cudaEventRecord(ev[k], ci);
                }
                cudaEventRecord(b1, ci);
                for (int k = 0; k < 16; ++k) {
                    if (dep) cudaStreamWaitEvent(s, ev[k], 0);
                    hog<<<ctas, 512, 0, s>>>(big + k * ck, ck, 1, o);
                    cudaEventRecord(ev[16 + k], s);
                    cudaStreamWaitEvent(co, ev[16 + k], 0);
                    cudaMemcpyAsync(y + k * cx, dy + k * cx, cx * 8, cudaMemcpyDeviceToHost, co);
                }
                cudaEventRecord(b2, co);
                cudaDeviceSynchronize();
                cudaEventElapsedTime(&t1, a, b1);
                cudaEventElapsedTime(&t2, a, b2);
            }
            printf("pipeline dep=%d ctas %4d: h2d done %.3f ms, all done %.3f ms\n", dep, ctas, t1, t2);
        }
    {
        unsigned *flags, *done, *hflag;
        double* ymap;
        cudaMalloc(&flags, 64 * 4);
        cudaMalloc(&done, 64 * 4);
        cudaMemset(flags, 0, 64 * 4);
        cudaMemset(done, 0, 64 * 4);
        cudaHostAlloc(&hflag, 64 * 4, 0);
        cudaHostAlloc(&ymap, nx * 8, cudaHostAllocMapped);
        double* ymap_d;
        cudaHostGetDevicePointer(&ymap_d, ymap, 0);
        unsigned epoch = 0;
        for (int mode = 0; mode < 3; ++mode)
            for (int ctas : {148, 296, 444}) {
                float t1 = 0, t2 = 0;
                for (int rep = 0; rep < 3; ++rep) {
                    ++epoch;
                    for (int k = 0; k < 16; ++k) hflag[k] = epoch;
                    cudaDeviceSynchronize();
                    cudaEventRecord(a, s);
                    cudaStreamWaitEvent(ci, a, 0);
                    cudaStreamWaitEvent(co, a, 0);
                    // kernel first: it spins until the copies land
                    pipe_kernel<<<ctas, 512, 0, s>>>(big, ck, dx, cx, mode == 2 ? ymap_d : dy, flags, done,
                                                     epoch);
                    for (int k = 0; k < 16; ++k) {
                        cudaMemcpyAsync(dx + k * cx, x + k * cx, cx * 8, cudaMemcpyHostToDevice, ci);
                        if (mode == 0)
                            cudaMemcpyAsync(flags + k, hflag + k, 4, cudaMemcpyHostToDevice, ci);
                        else
                            cuStreamWriteValue32((CUstream)ci, (CUdeviceptr)(flags + k), epoch, 0);
                    }
                    cudaEventRecord(b1, ci);
                    if (mode < 2)
                        for (int k = 0; k < 16; ++k) {
                            cuStreamWaitValue32((CUstream)co, (CUdeviceptr)(done + k), unsigned(ctas),
                                                CU_STREAM_WAIT_VALUE_GEQ);
                            cudaMemcpyAsync(y + k * cx, dy + k * cx, cx * 8, cudaMemcpyDeviceToHost, co);
                        }
                    cudaEventRecord(b2, mode < 2 ? co : s);
                    cudaDeviceSynchronize();
                    cudaEventElapsedTime(&t1, a, b1);
                    cudaEventElapsedTime(&t2, a, b2);
                    cudaMemset(done, 0, 64 * 4);
                    cudaDeviceSynchronize();
                }
                printf("persistent mode=%d ctas %4d: h2d done %.3f ms, all done %.3f ms  %s\n", mode, ctas, t1, t2,
                       cudaGetErrorString(cudaGetLastError()));
            }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
