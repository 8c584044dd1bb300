// Microbenchmark: bit-exact (reference row order) CSR SpMV variants, fp64.
// Standalone, not the product.  Inputs: banded n=4M (27/row), 2-D Laplacian
// 1000^2 (5/row), power-law rows (avg ~16, max ~20K).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/csrv scripts/csr_variants.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ double lds(const double* p) {
    double v; asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v;
}
__device__ __forceinline__ int lds(const int* p) {
    int v; asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p)); return v;
}

// V1: warp-level stream.  Group g = rows [gr[g], gr[g+1]) with entries
// [gk[g], gk[g+1]) (<= 32 rows, <= 2*W entries).  Each lane holds up to IT
// entries (coalesced), products go to warp-private smem, lane i sums row
// gr+i sequentially.  Next group's loads are issued before the sums.
template <int IT, int MINB>
__global__ void __launch_bounds__(256, MINB) csr_warp(int64_t ngroups, const int* __restrict__ gr, const int64_t* __restrict__ gk,
                                                const int64_t* __restrict__ rp, const int* __restrict__ col,
                                                const double* __restrict__ val, const double* __restrict__ x,
                                                double* __restrict__ y) {
    __shared__ double sp[8][32 * IT];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* prod = sp[wid];
    int64_t g = int64_t(blockIdx.x) * 8 + wid;
    const int64_t stride = int64_t(gridDim.x) * 8;
    if (g >= ngroups) return;
    int r0 = gr[g], r1 = gr[g + 1];
    int64_t k0 = gk[g], k1 = gk[g + 1];
    int c[IT]; double v[IT];
#pragma unroll
    for (int u = 0; u < IT; ++u) {
        int64_t k = k0 + u * 32 + lane;
        if (k < k1) { c[u] = lds(col + k); v[u] = lds(val + k); }
    }
    int64_t pa = 0, pe = 0;
    if (r0 + lane < r1) { pa = rp[r0 + lane]; pe = rp[r0 + lane + 1]; }
    while (true) {
        const int64_t gn = g + stride;
        int nr0 = 0, nr1 = 0; int64_t nk0 = 0, nk1 = 0;
        if (gn < ngroups) { nr0 = gr[gn]; nr1 = gr[gn + 1]; nk0 = gk[gn]; nk1 = gk[gn + 1]; }
#pragma unroll
        for (int u = 0; u < IT; ++u) {
            int64_t k = k0 + u * 32 + lane;
            if (k < k1) prod[u * 32 + lane] = __dmul_rn(v[u], __ldg(x + c[u]));
        }
        __syncwarp();
        int64_t npa = 0, npe = 0;
        if (gn < ngroups) {
#pragma unroll
            for (int u = 0; u < IT; ++u) {
                int64_t k = nk0 + u * 32 + lane;
                if (k < nk1) { c[u] = lds(col + k); v[u] = lds(val + k); }
            }
            if (nr0 + lane < nr1) { npa = rp[nr0 + lane]; npe = rp[nr0 + lane + 1]; }
        }
        if (r0 + lane < r1) {
            double s = 0.0;
            for (int64_t j = pa - k0; j < pe - k0; ++j) s = __dadd_rn(s, prod[j]);
            y[r0 + lane] = s;
        }
        __syncwarp();
        if (gn >= ngroups) break;
        g = gn; r0 = nr0; r1 = nr1; k0 = nk0; k1 = nk1; pa = npa; pe = npe;
    }
}

// V2: G lanes per row, sequential shuffle reduction by the group's lane 0.
template <int G>
__global__ void __launch_bounds__(256) csr_vec(int64_t n, const int64_t* __restrict__ rp, const int* __restrict__ col,
                                               const double* __restrict__ val, const double* __restrict__ x,
                                               double* __restrict__ y) {
    const int lane = threadIdx.x & 31, sub = lane & (G - 1);
    const int64_t row = (int64_t(blockIdx.x) * 256 + threadIdx.x) / G;
    const bool active = row < n;
    int64_t a = 0, e = 0;
    if (active) { a = rp[row]; e = rp[row + 1]; }
    double s = 0.0;
    // all groups of the warp iterate the same number of chunks (max len)
    int64_t len = e - a;
    int64_t maxlen = len;
#pragma unroll
    for (int o = G; o < 32; o <<= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    for (int64_t c0 = 0; c0 < maxlen; c0 += G) {
        const int64_t k = a + c0 + sub;
        double p = 0.0;
        if (c0 + sub < len) p = __dmul_rn(lds(val + k), __ldg(x + lds(col + k)));
        const int cnt = int(len - c0 < G ? len - c0 : G);
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const double q = __shfl_sync(0xffffffffu, p, j, G);
            if (j < cnt) s = __dadd_rn(s, q);
        }
    }
    if (active && sub == 0) y[row] = s;
}

struct Csr { int64_t n; std::vector<int64_t> rp; std::vector<int> col; std::vector<double> val; };

Csr banded(int64_t n, int h) {
    Csr m; m.n = n; m.rp.resize(n + 1); m.rp[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        for (int o = -h; o <= h; ++o) { int64_t j = i + o; if (j >= 0 && j < n) { m.col.push_back(int(j)); m.val.push_back(1.0 + ((i * 7 + j) % 13) / 8.0); } }
        m.rp[i + 1] = int64_t(m.col.size());
    }
    return m;
}
Csr lap(int g) {
    Csr m; m.n = int64_t(g) * g; m.rp.resize(m.n + 1); m.rp[0] = 0;
    for (int64_t i = 0; i < m.n; ++i) {
        int64_t x = i % g;
        int64_t cs[5] = {i - g, i - 1, i, i + 1, i + g};
        bool ok[5] = {i >= g, x > 0, true, x < g - 1, i < m.n - g};
        for (int t = 0; t < 5; ++t) if (ok[t]) { m.col.push_back(int(cs[t])); m.val.push_back(t == 2 ? 4.0 : -1.0 - (i % 5) / 8.0); }
        m.rp[i + 1] = int64_t(m.col.size());
    }
    return m;
}
Csr powerlaw(int64_t n, uint64_t seed) {
    std::mt19937_64 rng(seed);
    Csr m; m.n = n; m.rp.resize(n + 1); m.rp[0] = 0;
    std::uniform_real_distribution<double> u(0, 1);
    for (int64_t i = 0; i < n; ++i) {
        double p = u(rng);
        int64_t len = p < 0.5 ? 0 : int64_t(4.0 / std::pow(1.0 - (p - 0.5) * 2 + 1e-9, 0.85));
        len = std::min<int64_t>(len, 250);
        std::vector<int> cs(len);
        for (auto& c : cs) c = int(rng() % uint64_t(n));
        std::sort(cs.begin(), cs.end()); cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
        for (int c : cs) { m.col.push_back(c); m.val.push_back(1.0 + double(rng() % 8) / 8.0); }
        m.rp[i + 1] = int64_t(m.col.size());
    }
    return m;
}

void groups(const Csr& m, int W, std::vector<int>& gr, std::vector<int64_t>& gk) {
    // rows whose first entry falls in the same W-window, <= 32 rows; long rows alone
    gr.clear(); gk.clear();
    for (int64_t i = 0; i < m.n; ++i) {
        int64_t len = m.rp[i + 1] - m.rp[i];
        bool start = gr.empty() || (i - gr.back()) >= 32 || len > W ||
                     (i > 0 && ((m.rp[i] / W) != (m.rp[i - 1] / W) || (m.rp[i] - m.rp[i - 1]) > W));
        if (start) { gr.push_back(int(i)); gk.push_back(m.rp[i]); }
    }
    gr.push_back(int(m.n)); gk.push_back(m.rp[m.n]);
}

int main() {
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    char* flush; size_t fl = size_t(512) << 20; CK(cudaMalloc(&flush, fl));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    struct Case { const char* name; Csr m; };
    std::vector<Case> cases;
    cases.push_back({"banded 4M x27", banded(4000000, 13)});
    cases.push_back({"laplacian 1000^2", lap(1000)});
    cases.push_back({"powerlaw 4M", powerlaw(4000000, 7)});
    for (auto& cs : cases) {
        Csr& m = cs.m;
        int64_t z = m.rp[m.n];
        std::vector<double> hx(m.n);
        for (int64_t i = 0; i < m.n; ++i) hx[i] = 0.25 + (i % 97) / 128.0;
        std::vector<double> yr(m.n);
        for (int64_t i = 0; i < m.n; ++i) { double s = 0; for (int64_t k = m.rp[i]; k < m.rp[i + 1]; ++k) s += m.val[k] * hx[m.col[k]]; yr[i] = s; }
        int64_t *drp, *dgk; int *dcol, *dgr; double *dval, *dx, *dy;
        CK(cudaMalloc(&drp, (m.n + 1) * 8)); CK(cudaMalloc(&dcol, z * 4)); CK(cudaMalloc(&dval, z * 8));
        CK(cudaMalloc(&dx, m.n * 8)); CK(cudaMalloc(&dy, m.n * 8));
        CK(cudaMemcpy(drp, m.rp.data(), (m.n + 1) * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dcol, m.col.data(), z * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dval, m.val.data(), z * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dx, hx.data(), m.n * 8, cudaMemcpyHostToDevice));
        double bytes = z * 12.0 + (m.n + 1) * 8.0 + 16.0 * m.n;
        auto run = [&](const char* name, auto launch, bool exact_expected) {
            float tot = 0; int reps = 20;
            for (int r = 0; r < reps + 3; ++r) {
                CK(cudaMemsetAsync(flush, r, fl));
                cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
                float ms; cudaEventElapsedTime(&ms, e0, e1); if (r >= 3) tot += ms;
            }
            CK(cudaGetLastError());
            std::vector<double> yy(m.n); CK(cudaMemcpy(yy.data(), dy, m.n * 8, cudaMemcpyDeviceToHost));
            int64_t bad = 0; for (int64_t i = 0; i < m.n; ++i) bad += yy[i] != yr[i];
            printf("  %-26s avg %8.1f us  %7.0f GB/s  mismatches %lld%s\n", name, tot / reps * 1e3,
                   bytes / (tot / reps * 1e-3) / 1e9, (long long)bad, exact_expected ? "" : " (tree rows)");
        };
        printf("%s: n=%lld z=%lld\n", cs.name, (long long)m.n, (long long)z);
        for (int W : {128, 256}) {
            std::vector<int> gr; std::vector<int64_t> gk; groups(m, W, gr, gk);
            int64_t ng = int64_t(gr.size()) - 1;
            CK(cudaMalloc(&dgr, gr.size() * 4)); CK(cudaMalloc(&dgk, gk.size() * 8));
            CK(cudaMemcpy(dgr, gr.data(), gr.size() * 4, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dgk, gk.data(), gk.size() * 8, cudaMemcpyHostToDevice));
            char nm[64];
            if (W == 128) {
                snprintf(nm, 64, "warp W=128 IT8 minB4"); run(nm, [&] { csr_warp<8, 4><<<sms * 4, 256>>>(ng, dgr, dgk, drp, dcol, dval, dx, dy); }, true);
                snprintf(nm, 64, "warp W=128 IT8 minB6"); run(nm, [&] { csr_warp<8, 6><<<sms * 6, 256>>>(ng, dgr, dgk, drp, dcol, dval, dx, dy); }, true);
                snprintf(nm, 64, "warp W=128 IT8 minB8"); run(nm, [&] { csr_warp<8, 8><<<sms * 8, 256>>>(ng, dgr, dgk, drp, dcol, dval, dx, dy); }, true);
            } else {
                snprintf(nm, 64, "warp W=256 IT16 minB3"); run(nm, [&] { csr_warp<16, 3><<<sms * 3, 256>>>(ng, dgr, dgk, drp, dcol, dval, dx, dy); }, true);
                snprintf(nm, 64, "warp W=256 IT16 minB4"); run(nm, [&] { csr_warp<16, 4><<<sms * 4, 256>>>(ng, dgr, dgk, drp, dcol, dval, dx, dy); }, true);
                snprintf(nm, 64, "warp W=256 IT16 minB5"); run(nm, [&] { csr_warp<16, 5><<<sms * 5, 256>>>(ng, dgr, dgk, drp, dcol, dval, dx, dy); }, true);
            }
            cudaFree(dgr); cudaFree(dgk);
        }
        int64_t blocks8 = (m.n * 8 + 255) / 256, blocks16 = (m.n * 16 + 255) / 256, blocks32 = (m.n * 32 + 255) / 256;
        run("vec G=8", [&] { csr_vec<8><<<blocks8, 256>>>(m.n, drp, dcol, dval, dx, dy); }, true);
        run("vec G=16", [&] { csr_vec<16><<<blocks16, 256>>>(m.n, drp, dcol, dval, dx, dy); }, true);
        run("vec G=32", [&] { csr_vec<32><<<blocks32, 256>>>(m.n, drp, dcol, dval, dx, dy); }, true);
        cudaFree(drp); cudaFree(dcol); cudaFree(dval); cudaFree(dx); cudaFree(dy);
    }
    return 0;
}
