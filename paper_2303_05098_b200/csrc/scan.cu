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
// to *total_out.
__global__ void __launch_bounds__(kScanBlock) scan_tile_sums(int64_t* __restrict__ sums, int64_t m,
                                                              int64_t* __restrict__ total_out) {
    __shared__ int64_t warp_tot[kScanBlock / 32 + 1];
    int64_t carry = 0;
    for (int64_t base = 0; base < m; base += kScanBlock) {
        int64_t i = base + threadIdx.x;
        int64_t v = i < m ? sums[i] : 0;
        int64_t tot;
        int64_t ex = block_exclusive_scan(v, warp_tot, tot);
        if (i < m) sums[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) *total_out = carry;
}

template <typename TIn>
__global__ void __launch_bounds__(kScanBlock) tile_scan(const TIn* __restrict__ in, int64_t n,
                                                         const int64_t* __restrict__ tile_off,
                                                         int64_t* __restrict__ out) {
    __shared__ int64_t tile[kScanTile];
    __shared__ int64_t warp_tot[kScanBlock / 32 + 1];
    const int64_t base = int64_t(blockIdx.x) * kScanTile;
    for (int j = 0; j < kScanItems; ++j) {
        int e = j * kScanBlock + threadIdx.x;
        int64_t i = base + e;
        tile[e] = i < n ? int64_t(in[i]) : 0;
    }
    __syncthreads();
    int64_t local[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        local[j] = s;
        s += tile[threadIdx.x * kScanItems + j];
    }
    int64_t tot;
    int64_t ex = block_exclusive_scan(s, warp_tot, tot) + tile_off[blockIdx.x];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) tile[threadIdx.x * kScanItems + j] = ex + local[j];
    __syncthreads();
    for (int j = 0; j < kScanItems; ++j) {
        int e = j * kScanBlock + threadIdx.x;
        int64_t i = base + e;
        if (i < n) out[i] = tile[e];
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
    scan_tile_sums<<<1, kScanBlock, 0, s>>>(sums.get(), tiles, out + n);
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
