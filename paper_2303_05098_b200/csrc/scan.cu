// Hand-written device-wide exclusive scan (3-phase reduce-then-scan).
// Used by the conversions for row pointers, compaction positions and the
// row-block partition.  Tiles are staged through shared memory so every global
// access is coalesced.
#include "common.cuh"

namespace sob {

namespace {

constexpr int kScanBlock = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanBlock * kScanItems;

// Block-wide exclusive scan of one int64 per thread; returns the block total.
__device__ int64_t block_exclusive_scan(int64_t v, int64_t* warp_tot, int64_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t inc = warp_inclusive_sum(v);
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int64_t w = lane < kScanBlock / 32 ? warp_tot[lane] : 0;
        int64_t wi = warp_inclusive_sum(w);
        if (lane < kScanBlock / 32) warp_tot[lane] = wi - w;
        if (lane == kScanBlock / 32 - 1) warp_tot[kScanBlock / 32] = wi;
    }
    __syncthreads();
    int64_t excl = warp_tot[warp] + inc - v;
    total = warp_tot[kScanBlock / 32];
    __syncthreads();
    return excl;
}

template <typename TIn>
__global__ void __launch_bounds__(kScanBlock) tile_reduce(const TIn* __restrict__ in, int64_t n,
                                                           int64_t* __restrict__ tile_sums) {
    const int64_t base = int64_t(blockIdx.x) * kScanTile;
    int64_t s = 0;
#pragma unroll 4
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = base + j * kScanBlock + threadIdx.x;
        if (i < n) s += int64_t(in[i]);
    }
    s = warp_sum(s);
    __shared__ int64_t ws[kScanBlock / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        int64_t v = threadIdx.x < kScanBlock / 32 ? ws[threadIdx.x] : 0;
        v = warp_sum(v);
        if (threadIdx.x == 0) tile_sums[blockIdx.x] = v;
    }
}

// Single CTA: exclusive scan of the tile sums in place; writes the grand total
// to *total_out.  Each of the 1024 threads owns a contiguous run of sums
// (one block scan in total, not one per 256 sums).
constexpr int kSumsBlock = 1024;
__device__ int64_t block_exclusive_scan_1024(int64_t v, int64_t* warp_tot, int64_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t inc = warp_inclusive_sum(v);
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const int64_t w = warp_tot[lane];  // 32 warps
        const int64_t wi = warp_inclusive_sum(w);
        warp_tot[lane] = wi - w;
        if (lane == 31) warp_tot[32] = wi;
    }
    __syncthreads();
    total = warp_tot[32];
    return warp_tot[warp] + inc - v;
}

__global__ void __launch_bounds__(kSumsBlock) scan_tile_sums(int64_t* __restrict__ sums, int64_t m,
                                                              int64_t* __restrict__ total_out) {
    __shared__ int64_t warp_tot[33];
    const int64_t per = (m + kSumsBlock - 1) / kSumsBlock;
    const int64_t a = int64_t(threadIdx.x) * per, b = a + per < m ? a + per : m;
    int64_t loc = 0;
    for (int64_t i = a; i < b; ++i) loc += sums[i];
    int64_t tot;
    int64_t run = block_exclusive_scan_1024(loc, warp_tot, tot);
    for (int64_t i = a; i < b; ++i) {
        const int64_t v = sums[i];
        sums[i] = run;
        run += v;
    }
    if (threadIdx.x == 0) *total_out = tot;
}

// Tile staged through shared memory with one pad word per 16 (the blocked
// per-thread pass reads 16 consecutive int64 per thread: unpadded, a
// half-warp's 8-byte accesses all hit one bank pair).
__device__ __forceinline__ int tile_pad(int e) { return e + (e >> 4); }

template <typename TIn>
__global__ void __launch_bounds__(kScanBlock) tile_scan(const TIn* __restrict__ in, int64_t n,
                                                         const int64_t* __restrict__ tile_off,
                                                         int64_t* __restrict__ out) {
    __shared__ int64_t tile[kScanTile + kScanTile / 16];
    __shared__ int64_t warp_tot[kScanBlock / 32 + 1];
    const int64_t base = int64_t(blockIdx.x) * kScanTile;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int e = j * kScanBlock + threadIdx.x;
        const int64_t i = base + e;
        tile[tile_pad(e)] = i < n ? int64_t(in[i]) : 0;
    }
    __syncthreads();
    int64_t local[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        local[j] = s;
        s += tile[tile_pad(threadIdx.x * kScanItems + j)];
    }
    int64_t tot;
    const int64_t ex = block_exclusive_scan(s, warp_tot, tot) + tile_off[blockIdx.x];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) tile[tile_pad(threadIdx.x * kScanItems + j)] = ex + local[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int e = j * kScanBlock + threadIdx.x;
        const int64_t i = base + e;
        if (i < n) out[i] = tile[tile_pad(e)];
    }
}

template <typename TIn>
void exclusive_scan_impl(const TIn* in, int64_t* out, int64_t n, cudaStream_t s) {
    if (n <= 0) {
        SOB_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
        return;
    }
    int64_t tiles = ceil_div(n, kScanTile);
    DBuf<int64_t> sums(tiles, s);
    tile_reduce<TIn><<<unsigned(tiles), kScanBlock, 0, s>>>(in, n, sums.get());
    SOB_LAUNCH("tile_reduce");
    scan_tile_sums<<<1, kSumsBlock, 0, s>>>(sums.get(), tiles, out + n);
    SOB_LAUNCH("scan_tile_sums");
    tile_scan<TIn><<<unsigned(tiles), kScanBlock, 0, s>>>(in, n, sums.get(), out);
    SOB_LAUNCH("tile_scan");
}

}  // namespace

void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
    exclusive_scan_impl<int64_t>(in, out, n, s);
}

void exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, cudaStream_t s) {
    exclusive_scan_impl<int32_t>(in, out, n, s);
}

}  // namespace sob
