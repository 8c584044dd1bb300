// Device canonicalization: CooMatrix::from_triplets (formats.cpp:293-322)
// on the B200 -- range check (IndexOutOfRange), stable LSD radix sort of the
// (row, col) key with the value as payload, duplicate coordinates summed in
// input order.  Hand-written: 8-bit digits, 4096-key tiles, per-tile digit
// histograms -> one device-wide exclusive scan (digit-major, so equal digits
// keep tile order) -> stable scatter ranked with __match_any_sync per warp.
#include "matrix.cuh"

namespace sob {

namespace {

constexpr int kRB = 256;          // threads per tile
constexpr int kRItems = 16;       // keys per thread
constexpr int kRTile = kRB * kRItems;
constexpr int kDigits = 256;

__global__ void make_keys(const int64_t* __restrict__ row, const int64_t* __restrict__ col, int64_t n,
                          int64_t nrows, int64_t ncols, uint64_t* __restrict__ key, int* __restrict__ bad) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t r = row[i], c = col[i];
    if (r < 0 || r >= nrows || c < 0 || c >= ncols) {
        atomicExch(bad, 1);
        key[i] = 0;
        return;
    }
    key[i] = uint64_t(r) * uint64_t(ncols) + uint64_t(c);
}

__global__ void __launch_bounds__(kRB) radix_hist(const uint64_t* __restrict__ key, int64_t n, int shift,
                                                   int64_t ntiles, int32_t* __restrict__ hist) {
    __shared__ int32_t cnt[kDigits];
    cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = int64_t(blockIdx.x) * kRTile;
    for (int j = 0; j < kRItems; ++j) {
        const int64_t i = base + j * kRB + threadIdx.x;
        if (i < n) atomicAdd(&cnt[int((key[i] >> shift) & 0xFF)], 1);
    }
    __syncthreads();
    hist[int64_t(threadIdx.x) * ntiles + blockIdx.x] = cnt[threadIdx.x];  // digit-major
}

__global__ void __launch_bounds__(kRB)
    radix_scatter(const uint64_t* __restrict__ kin, const double* __restrict__ vin, int64_t n, int shift,
                  int64_t ntiles, const int64_t* __restrict__ offs, uint64_t* __restrict__ kout,
                  double* __restrict__ vout) {
    __shared__ int64_t base_d[kDigits];
    __shared__ int32_t wcnt[kRB / 32][kDigits];
    __shared__ int32_t wpre[kRB / 32][kDigits];
    __shared__ int32_t total[kDigits];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    base_d[threadIdx.x] = offs[int64_t(threadIdx.x) * ntiles + blockIdx.x];
    const int64_t tbase = int64_t(blockIdx.x) * kRTile;
    for (int j = 0; j < kRItems; ++j) {
        for (int w = 0; w < kRB / 32; ++w) wcnt[w][threadIdx.x] = 0;
        __syncthreads();
        const int64_t i = tbase + j * kRB + threadIdx.x;
        const bool valid = i < n;
        const uint64_t k = valid ? kin[i] : 0;
        const int d = valid ? int((k >> shift) & 0xFF) : -1 - lane;  // idle lanes never merge
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        if (valid && rank == 0) wcnt[warp][d] = __popc(peers);
        __syncthreads();
        {  // thread = digit: exclusive prefix over the warps of this round
            int run = 0;
            for (int w = 0; w < kRB / 32; ++w) {
                wpre[w][threadIdx.x] = run;
                run += wcnt[w][threadIdx.x];
            }
            total[threadIdx.x] = run;
        }
        __syncthreads();
        if (valid) {
            const int64_t p = base_d[d] + wpre[warp][d] + rank;
            kout[p] = k;
            vout[p] = vin[i];
        }
        __syncthreads();
        base_d[threadIdx.x] += total[threadIdx.x];
    }
}

__global__ void run_heads(const uint64_t* __restrict__ key, int64_t n, int32_t* __restrict__ head) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// duplicate coordinates summed in sorted (= input, the sort is stable) order
__global__ void run_reduce(const uint64_t* __restrict__ key, const double* __restrict__ val, int64_t n,
                           const int32_t* __restrict__ head, const int64_t* __restrict__ pos, int64_t ncols,
                           int32_t* __restrict__ orow, int32_t* __restrict__ ocol, double* __restrict__ oval) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n || !head[i]) return;
    double s = val[i];
    for (int64_t j = i + 1; j < n && key[j] == key[i]; ++j) s += val[j];
    const int64_t p = pos[i];
    orow[p] = int32_t(key[i] / uint64_t(ncols));
    ocol[p] = int32_t(key[i] % uint64_t(ncols));
    oval[p] = s;
}

}  // namespace

so_matrix* coo_from_triplets_device(int64_t nrows, int64_t ncols, int64_t n, const int64_t* row_h,
                                    const int64_t* col_h, const double* val_h, cudaStream_t s) {
    const TripletSegment seg{row_h, col_h, val_h, n};
    return coo_from_triplet_segments(nrows, ncols, &seg, n > 0 ? 1 : 0, s);
}

so_matrix* coo_from_triplet_segments(int64_t nrows, int64_t ncols, const TripletSegment* segs, int nseg,
                                     cudaStream_t s) {
    auto* m = new so_matrix();
    std::unique_ptr<so_matrix> guard(m);
    SOB_CUDA(cudaGetDevice(&m->device));
    m->format = SO_COO;
    m->nrows = nrows;
    m->ncols = ncols;
    int64_t n = 0;
    for (int i = 0; i < nseg; ++i) n += segs[i].n;
    if (n == 0) return guard.release();
    DBuf<int64_t> r(n, s), c(n, s);
    DBuf<double> v(n, s), v2(n, s);
    // the segments in order, straight into the device arrays (no host concatenation)
    int64_t at = 0;
    for (int i = 0; i < nseg; ++i) {
        const TripletSegment& g = segs[i];
        if (g.n == 0) continue;
        SOB_CUDA(cudaMemcpyAsync(r.get() + at, g.row, sizeof(int64_t) * size_t(g.n), cudaMemcpyHostToDevice, s));
        SOB_CUDA(cudaMemcpyAsync(c.get() + at, g.col, sizeof(int64_t) * size_t(g.n), cudaMemcpyHostToDevice, s));
        SOB_CUDA(cudaMemcpyAsync(v.get() + at, g.val, sizeof(double) * size_t(g.n), cudaMemcpyHostToDevice, s));
        at += g.n;
    }
    DBuf<uint64_t> k(n, s), k2(n, s);
    DBuf<int> bad(1, s);
    SOB_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    make_keys<<<unsigned(ceil_div(n, 256)), 256, 0, s>>>(r.get(), c.get(), n, nrows, ncols, k.get(), bad.get());
    SOB_LAUNCH("make_keys");
    if (d2h_scalar(bad.get(), s)) fail(SO_INDEX_OUT_OF_RANGE, "triplet outside " + std::to_string(nrows) + "x" +
                                                                   std::to_string(ncols));
    r.release();
    c.release();
    const uint64_t kmax = uint64_t(nrows) * uint64_t(ncols);
    int bits = 0;
    while (bits < 64 && (uint64_t(1) << bits) < kmax) ++bits;
    const int64_t ntiles = ceil_div(n, kRTile);
    DBuf<int32_t> hist(int64_t(kDigits) * ntiles, s);
    DBuf<int64_t> offs(int64_t(kDigits) * ntiles + 1, s);
    uint64_t *kin = k.get(), *kout = k2.get();
    double *vin = v.get(), *vout = v2.get();
    for (int shift = 0; shift < bits; shift += 8) {
        radix_hist<<<unsigned(ntiles), kRB, 0, s>>>(kin, n, shift, ntiles, hist.get());
        SOB_LAUNCH("radix_hist");
        exclusive_scan_i32_to_i64(hist.get(), offs.get(), int64_t(kDigits) * ntiles, s);
        radix_scatter<<<unsigned(ntiles), kRB, 0, s>>>(kin, vin, n, shift, ntiles, offs.get(), kout, vout);
        SOB_LAUNCH("radix_scatter");
        std::swap(kin, kout);
        std::swap(vin, vout);
    }
    DBuf<int32_t> head(n, s);
    DBuf<int64_t> pos(n + 1, s);
    run_heads<<<unsigned(ceil_div(n, 256)), 256, 0, s>>>(kin, n, head.get());
    SOB_LAUNCH("run_heads");
    exclusive_scan_i32_to_i64(head.get(), pos.get(), n, s);
    const int64_t z = d2h_scalar(pos.get() + n, s);
    CooPart& cp = m->coo;
    cp.nnz = z;
    cp.row.alloc(z, s);
    cp.col.alloc(z, s);
    cp.val.alloc(z, s);
    run_reduce<<<unsigned(ceil_div(n, 256)), 256, 0, s>>>(kin, vin, n, head.get(), pos.get(), ncols, cp.row.get(),
                                                          cp.col.get(), cp.val.get());
    SOB_LAUNCH("run_reduce");
    SOB_CUDA(cudaStreamSynchronize(s));
    return guard.release();
}

}  // namespace sob
