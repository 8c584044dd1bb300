// Gather lab (not the product): how fast can one B200 fetch x[col[k]] for the
// 65 M column indices of config 3 (R-MAT 2^22, avg degree 16, sorted by row)?
// the LDG path tops out near one 128-byte line per SM-cycle
// (the L1TEX wavefront rate), 224 us for this matrix, which bounds every
// format on R-MAT.  This lab measures the alternatives:
//   ldg<M>     8 gathers per lane through LDG with cache qualifier M
//              (nc / cg / nc.L1::no_allocate / relaxed.gpu / ca / lu)
//   ldg+persist  the same with x in an L2 persisting access-policy window
//   tma        every gather through the TMA unit: cp.async.bulk.tensor
//              tile::gather4 on x viewed as [n/4][4] doubles (32-byte rows: the
//              shared-memory destination of a gather4 must be 128-byte aligned),
//              4 gathers per instruction, completion on an mbarrier
//   mix<f>     a fraction of each chunk via TMA, the rest via LDG, issued together
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o build/gather_lab scripts/gather_lab.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <random>
#include <type_traits>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ int ldcol(const int* p) {
    int v; asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p)); return v;
}
template <int M>
__device__ __forceinline__ double ldx(const double* p) {
    double v;
    if constexpr (M == 0) asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if constexpr (M == 1) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if constexpr (M == 2) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if constexpr (M == 3) asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if constexpr (M == 4) asm volatile("ld.global.ca.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if constexpr (M == 5) asm volatile("ld.global.lu.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else asm volatile("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

template <int M, int MINB>
__global__ void __launch_bounds__(256, MINB) ldg_probe(int64_t z, const int* __restrict__ col, const double* __restrict__ x,
                                                       double* __restrict__ sink) {
    double acc = 0.0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 8;
    for (int64_t base = (int64_t(blockIdx.x) * blockDim.x) * 8 + threadIdx.x; base < z; base += stride) {
        int c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t k = base + int64_t(u) * blockDim.x;
            c[u] = k < z ? ldcol(col + k) : -1;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += c[u] >= 0 ? ldx<M>(x + c[u]) : 0.0;
    }
    if (acc == 1.2345e300) *sink = acc;
}

// Hot-column form: entries on the K most frequent columns carry ~rank (< 0)
// and read a packed copy xh[rank]; the rest read x[col] -- a per-entry select
// between two bases, as a product kernel would do it.
template <int MINB>
__global__ void __launch_bounds__(256, MINB) hot_probe(int64_t z, const int* __restrict__ col, const double* __restrict__ x,
                                                       const double* __restrict__ xh, double* __restrict__ sink) {
    double acc = 0.0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 8;
    for (int64_t base = (int64_t(blockIdx.x) * blockDim.x) * 8 + threadIdx.x; base < z; base += stride) {
        int c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t k = base + int64_t(u) * blockDim.x;
            c[u] = k < z ? ldcol(col + k) : 0x7fffffff;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (c[u] == 0x7fffffff) continue;
            const double* p = c[u] < 0 ? xh + ~c[u] : x + c[u];
            acc += ldx<0>(p);
        }
    }
    if (acc == 1.2345e300) *sink = acc;
}

// ---------------------------------------------------------------- TMA gather4
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" :: "r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_g4(void* dst, const CUtensorMap* tm, uint64_t* bar, int r0, int r1, int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        :: "r"(smem_u32(dst)), "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar)) : "memory");
}

// Each warp walks chunks of 256 entries; TPL of every lane's 8 entries go via
// TMA (TPL multiple of 4), the rest via LDG.  Double-buffered per warp.
template <int TPL, int MINB>
__global__ void __launch_bounds__(256, MINB) tma_probe(int64_t z, const int* __restrict__ col, const double* __restrict__ x,
                                                       const __grid_constant__ CUtensorMap tm, double* __restrict__ sink) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kBuf = 32 * (TPL > 0 ? TPL : 4) * 32;  // bytes per chunk buffer (32-byte rows)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    unsigned char* buf = smem + 128 + size_t(warp) * 2 * kBuf;
    if (lane == 0) { mbar_init(&bars[warp * 2], 1); mbar_init(&bars[warp * 2 + 1], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t nch = z / 256;
    const int64_t wstride = int64_t(gridDim.x) * (blockDim.x >> 5);
    int64_t ch = int64_t(blockIdx.x) * (blockDim.x >> 5) + warp;
    double acc = 0.0;
    uint32_t phase[2] = {0, 0};
    int c[2][8];
    auto issue = [&](int64_t chk, auto bc) {
        constexpr int b = decltype(bc)::value;
        const int64_t k = chk * 256 + lane * 8;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            int4 v;
            asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(col + k + 4 * h));
            c[b][4 * h] = v.x; c[b][4 * h + 1] = v.y; c[b][4 * h + 2] = v.z; c[b][4 * h + 3] = v.w;
        }
        if constexpr (TPL > 0) {
            if (lane == 0) mbar_expect(&bars[warp * 2 + b], 32 * TPL * 32);
            __syncwarp();
            double* dst = reinterpret_cast<double*>(buf + b * kBuf) + lane * TPL * 4;
#pragma unroll
            for (int u = 0; u < TPL; u += 4)
                tma_g4(dst + u * 4, &tm, &bars[warp * 2 + b], c[b][u] >> 2, c[b][u + 1] >> 2, c[b][u + 2] >> 2, c[b][u + 3] >> 2);
        }
    };
    auto consume = [&](auto bc) {
        constexpr int b = decltype(bc)::value;
        double part = 0.0;
#pragma unroll
        for (int u = TPL; u < 8; ++u) part += __ldg(x + c[b][u]);
        if constexpr (TPL > 0) {
            mbar_wait(&bars[warp * 2 + b], phase[b]);
            phase[b] ^= 1;
            const double* src = reinterpret_cast<const double*>(buf + b * kBuf) + lane * TPL * 4;
#pragma unroll
            for (int u = 0; u < TPL; ++u) part += src[u * 4 + (c[b][u] & 3)];
        }
        acc += part;
        __syncwarp();
    };
    using B0 = std::integral_constant<int, 0>;
    using B1 = std::integral_constant<int, 1>;
    if (ch < nch) issue(ch, B0{});
    while (ch < nch) {
        if (ch + wstride < nch) issue(ch + wstride, B1{});
        consume(B0{});
        ch += wstride;
        if (ch >= nch) break;
        if (ch + wstride < nch) issue(ch + wstride, B0{});
        consume(B1{});
        ch += wstride;
    }
    if (acc == 1.2345e300) *sink = acc;
}

// ---------------------------------------------------------------- matrices
static std::vector<int> rmat_cols(int scale, int deg, uint64_t seed, int64_t& n) {
    n = int64_t(1) << scale;
    const int64_t draws = n * deg;
    std::mt19937_64 rng(seed);
    std::vector<uint64_t> keys(draws);
    for (int64_t e = 0; e < draws; ++e) {
        uint64_t r = 0, c = 0;
        for (int l = 0; l < scale; ++l) {
            double p = (rng() >> 11) * (1.0 / 9007199254740992.0);
            int q = p < 0.57 ? 0 : p < 0.76 ? 1 : p < 0.95 ? 2 : 3;
            r = 2 * r + (q >> 1); c = 2 * c + (q & 1);
        }
        keys[e] = (r << 32) | c;
    }
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    std::vector<int> col(keys.size());
    for (size_t k = 0; k < keys.size(); ++k) col[k] = int(keys[k] & 0xffffffffu);
    return col;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const char* which = argc > 1 ? argv[1] : "rmat,rmat-relabel,uniform,uniform8k,uniform64k";
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int clk_khz; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    EncodeTiled encode = reinterpret_cast<EncodeTiled>(fn);
    double* sink; CK(cudaMalloc(&sink, 8));
    double* flush; const size_t kFlush = size_t(512) << 20; CK(cudaMalloc(&flush, kFlush));
    // matrices: 0 rmat (sorted by row), 1 rmat with columns relabelled by
    // descending frequency (hot columns packed into the first lines of x),
    // 2 uniform random over all n columns, 3/4 uniform over the first 8K / 64K
    // columns (x lines all L1 hits / all L2 hits)
    const char* names[5] = {"rmat", "rmat-relabel", "uniform", "uniform8k", "uniform64k"};
    for (int mi = 0; mi < 5; ++mi) {
        const char* nm = names[mi];
        bool sel = false;
        for (const char* p = which; p && *p;) {
            const char* e = strchr(p, ',');
            const size_t len = e ? size_t(e - p) : strlen(p);
            if (len == strlen(nm) && strncmp(p, nm, len) == 0) sel = true;
            p = e ? e + 1 : nullptr;
        }
        if (!sel) continue;
        int64_t n = 0;
        std::vector<int> col;
        if (mi <= 1) {
            col = rmat_cols(22, 16, 42, n);
            if (mi == 1) {
                std::vector<int64_t> freq(n, 0);
                for (int c : col) freq[c]++;
                std::vector<int> order(n);
                for (int64_t i = 0; i < n; ++i) order[i] = int(i);
                std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return freq[a] > freq[b]; });
                std::vector<int> rank(n);
                for (int64_t i = 0; i < n; ++i) rank[order[i]] = int(i);
                int64_t cum = 0;
                for (int64_t i = 0; i < n; ++i) {
                    cum += freq[order[i]];
                    if (i == 1023 || i == 8191 || i == 65535 || i == 524287)
                        printf("  top %lld columns hold %.3f of the entries\n", (long long)(i + 1), double(cum) / col.size());
                }
                for (auto& c : col) c = rank[c];
            }
        } else {
            n = int64_t(1) << 22; col.resize(size_t(65245415));
            const uint64_t range = mi == 2 ? uint64_t(n) : mi == 3 ? 8192 : 65536;
            std::mt19937_64 rng(7);
            for (auto& c : col) c = int(rng() % range);
        }
        const int64_t z = int64_t(col.size());
        int* dcol; double* dx;
        CK(cudaMalloc(&dcol, (z + 256) * 4)); CK(cudaMalloc(&dx, n * 8));
        CK(cudaMemcpy(dcol, col.data(), z * 4, cudaMemcpyHostToDevice));
        std::vector<double> hx(n); for (int64_t i = 0; i < n; ++i) hx[i] = 1.0 + (i % 7);
        CK(cudaMemcpy(dx, hx.data(), n * 8, cudaMemcpyHostToDevice));
        printf("%s: n=%lld z=%lld (%d SMs @ %.3f GHz)\n", nm, (long long)n, (long long)z, sms, clk_khz / 1e6);
        CUtensorMap tm;
        cuuint64_t dims[2] = {4, cuuint64_t(n / 4)};
        cuuint64_t strides[1] = {32};
        cuuint32_t box[2] = {4, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dx, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) printf("tensor map encode failed: %d\n", int(r));
        cudaStream_t st; CK(cudaStreamCreate(&st));
        auto timeit = [&](const std::function<void()>& f, bool flush_l2) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            float tot = 0; const int reps = 20;
            for (int it = 0; it < reps + 3; ++it) {
                if (flush_l2) CK(cudaMemsetAsync(flush, it & 0xff, kFlush, st));
                cudaEventRecord(e0, st); f(); cudaEventRecord(e1, st); CK(cudaEventSynchronize(e1));
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (it >= 3) tot += ms;
            }
            CK(cudaGetLastError());
            return tot / reps;
        };
        auto rep = [&](const char* name, const std::function<void()>& f) {
            const float cold = timeit(f, true), warm = timeit(f, false);
            const double per_sm_cyc = double(z) / (double(sms) * (warm * 1e-3) * clk_khz * 1e3);
            printf("  %-34s cold %7.1f us  warm %7.1f us  %6.2f Ggath/s  %.3f gathers/SM-cycle\n", name, cold * 1e3, warm * 1e3,
                   z / (warm * 1e-3) / 1e9, per_sm_cyc);
            fflush(stdout);
        };
        const char* mn[7] = {"nc", "cg", "nc.L1::no_allocate", "relaxed.gpu", "ca", "lu", "nc.L1::evict_last"};
        auto ldg_all = [&](const char* tag) {
            auto run = [&](int m, auto kern, int minb) {
                char b[96]; snprintf(b, 96, "ldg %s B%d %s", mn[m], minb, tag);
                rep(b, [&] { kern<<<sms * minb, 256, 0, st>>>(z, dcol, dx, sink); });
            };
            run(0, ldg_probe<0, 8>, 8); run(1, ldg_probe<1, 8>, 8);
            if (getenv("GL_LDG_SHORT")) return;
            run(0, ldg_probe<0, 4>, 4); run(2, ldg_probe<2, 8>, 8); run(3, ldg_probe<3, 8>, 8);
            run(4, ldg_probe<4, 8>, 8); run(5, ldg_probe<5, 8>, 8); run(6, ldg_probe<6, 8>, 8);
        };
        if (!getenv("GL_NO_LDG")) ldg_all("");
        if (mi == 0 && getenv("GL_HOT")) {
            std::vector<int64_t> freq(n, 0);
            for (int c : col) freq[c]++;
            std::vector<int> order(n);
            for (int64_t i = 0; i < n; ++i) order[i] = int(i);
            std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return freq[a] > freq[b]; });
            double* dxh; CK(cudaMalloc(&dxh, size_t(1 << 20) * 8));
            int* dhc; CK(cudaMalloc(&dhc, (z + 256) * 4));
            for (int K : {1024, 4096, 8192, 16384, 32768, 65536, 262144}) {
                std::vector<int> rank(n, -1);
                for (int i = 0; i < K; ++i) rank[order[i]] = i;
                std::vector<int> hc(z);
                for (int64_t k = 0; k < z; ++k) hc[k] = rank[col[k]] >= 0 ? ~rank[col[k]] : col[k];
                CK(cudaMemcpy(dhc, hc.data(), z * 4, cudaMemcpyHostToDevice));
                char b[96]; snprintf(b, 96, "hot K=%d (%zu KB) B8", K, size_t(K) * 8 / 1024);
                rep(b, [&] { hot_probe<8><<<sms * 8, 256, 0, st>>>(z, dhc, dx, dxh, sink); });
                snprintf(b, 96, "hot K=%d (%zu KB) B6", K, size_t(K) * 8 / 1024);
                rep(b, [&] { hot_probe<6><<<sms * 6, 256, 0, st>>>(z, dhc, dx, dxh, sink); });
            }
            cudaFree(dxh); cudaFree(dhc);
        }
        auto tma = [&](int tpl, auto kern, int minb) {
            const size_t sm = 128 + size_t(8) * 2 * 32 * (tpl > 0 ? tpl : 4) * 32;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
            char b[96]; snprintf(b, 96, "tma gather4 %d/8 B%d smem %zuK", tpl, minb, sm / 1024);
            rep(b, [&] { kern<<<sms * minb, 256, sm, st>>>(z, dcol, dx, tm, sink); });
        };
        if (!getenv("GL_NO_TMA")) {
        tma(0, tma_probe<0, 4>, 4);
        tma(0, tma_probe<0, 8>, 8);
        tma(8, tma_probe<8, 1>, 1);
        tma(4, tma_probe<4, 2>, 2);
        tma(4, tma_probe<4, 3>, 3);
        }
        // L2 persistence window on x
        int maxp = 0; CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0));
        const size_t want = std::min<size_t>(size_t(maxp), size_t(n) * 8);
        if (!getenv("GL_NO_PERSIST") && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) {
            cudaStreamAttrValue a = {};
            a.accessPolicyWindow.base_ptr = dx;
            a.accessPolicyWindow.num_bytes = std::min<size_t>(size_t(n) * 8, want);
            a.accessPolicyWindow.hitRatio = 1.0f;
            a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a));
            char tag[64]; snprintf(tag, 64, "persist %zuMB", want >> 20);
            ldg_all(tag);
            tma(4, tma_probe<4, 3>, 3);
            a.accessPolicyWindow.num_bytes = 0;
            CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a));
            cudaCtxResetPersistingL2Cache();
        } else printf("  persisting L2 limit not settable (max %d)\n", maxp);
        CK(cudaStreamDestroy(st));
        cudaFree(dcol); cudaFree(dx);
    }
    return 0;
}
