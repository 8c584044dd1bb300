// fp64 SpMV in the six formats, sm_100a.  Memory-bound (≈0.1 flop/B): no
// tensor cores; the design goal is full-width coalesced HBM streams of the
// matrix arrays with x served from L1/L2.
//
// Parity: every kernel that owns a whole row reproduces the reference's
// per-row summation order (spmv.cpp:21-108) with separately rounded multiply
// and add (__dmul_rn/__dadd_rn -- the reference is built without FMA), so
// CSR, DIA, ELL and HDC rows are BIT-EXACT versus the CPU reference.  Only
// rows split across threads (CSR rows longer than kWindow, COO/HYB-COO
// segments spanning thread or chunk boundaries) are combined in a fixed
// tree order: deterministic, within the 1e-12 relative contract.
#include "matrix.cuh"

namespace sob {

namespace {

__device__ __forceinline__ double fmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fadd(double a, double b) { return __dadd_rn(a, b); }

// Deterministic block-wide sum (fixed butterfly + fixed warp order).
template <int BLOCK>
__device__ double block_sum_det(double v, double* scratch) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < BLOCK / 32 ? scratch[threadIdx.x] : 0.0;
        t = warp_sum(t);
    }
    return t;  // valid in thread 0
}

// DIA contribution of one row, diagonals ascending (spmv.cpp:45-56 restated
// per row: y[i] += diag[i] * x[i + off] for every in-range diagonal).
__device__ __forceinline__ double dia_row(int64_t i, int64_t nrows, int64_t ncols, int ndiags,
                                          const int64_t* __restrict__ offsets,
                                          const double* __restrict__ vals,
                                          const double* __restrict__ x) {
    double acc = 0.0;
#pragma unroll 4
    for (int d = 0; d < ndiags; ++d) {
        const int64_t c = i + __ldg(offsets + d);
        if (c >= 0 && c < ncols) acc = fadd(acc, fmul(ld_stream(vals + int64_t(d) * nrows + i), __ldg(x + c)));
    }
    return acc;
}

// ---------------------------------------------------------------- CSR -------
// Streaming CSR ("CSR-stream"): CTA b owns rows [blk[b], blk[b+1]).  Phase 1
// streams the block's contiguous val/col range with coalesced loads, gathers
// x and stages the rounded products in shared memory; phase 2 gives each row
// to one thread which sums its products in the reference order.  WITH_DIA
// fuses the HDC DIA part in front of the CSR part (spmv.cpp:101-106).
template <bool WITH_DIA>
__global__ void __launch_bounds__(kStreamBlock)
    csr_stream_kernel(const int32_t* __restrict__ blk, const int64_t* __restrict__ rp,
                      const int32_t* __restrict__ col, const double* __restrict__ val,
                      const double* __restrict__ x, double* __restrict__ y, int64_t nrows,
                      int64_t ncols, int ndiags, const int64_t* __restrict__ offsets,
                      const double* __restrict__ dvals) {
    extern __shared__ double prod[];  // 2 * kWindow
    const int r0 = blk[blockIdx.x], r1 = blk[blockIdx.x + 1];
    const int64_t k0 = rp[r0], k1 = rp[r1];
    const int64_t nk = k1 - k0;
    if (nk <= 2 * kWindow) {
        constexpr int U = 4;
        const int n = int(nk);
        for (int j0 = 0; j0 < n; j0 += kStreamBlock * U) {
            int c[U];
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u * kStreamBlock + int(threadIdx.x);
                if (j < n) {
                    c[u] = ld_stream(col + k0 + j);
                    v[u] = ld_stream(val + k0 + j);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u * kStreamBlock + int(threadIdx.x);
                if (j < n) prod[j] = fmul(v[u], __ldg(x + c[u]));
            }
        }
        __syncthreads();
        for (int r = r0 + int(threadIdx.x); r < r1; r += kStreamBlock) {
            const int a = int(rp[r] - k0), e = int(rp[r + 1] - k0);
            double s = 0.0;
            for (int j = a; j < e; ++j) s = fadd(s, prod[j]);
            if (WITH_DIA) s = fadd(dia_row(r, nrows, ncols, ndiags, offsets, dvals, x), s);
            y[r] = s;
        }
    } else {
        // one row longer than kWindow: strided partial sums + fixed tree
        double s = 0.0;
        for (int64_t k = k0 + threadIdx.x; k < k1; k += kStreamBlock)
            s = fadd(s, fmul(ld_stream(val + k), __ldg(x + ld_stream(col + k))));
        double t = block_sum_det<kStreamBlock>(s, prod);
        if (threadIdx.x == 0) {
            if (WITH_DIA) t = fadd(dia_row(r0, nrows, ncols, ndiags, offsets, dvals, x), t);
            y[r0] = t;
        }
    }
}

// ---------------------------------------------------------------- DIA -------
// One thread per row, diagonals ascending: consecutive threads read
// consecutive cells of each diagonal (diagonal-major layout => coalesced).
__global__ void __launch_bounds__(256)
    dia_kernel(int64_t nrows, int64_t ncols, int ndiags, const int64_t* __restrict__ offsets,
               const double* __restrict__ vals, const double* __restrict__ x,
               double* __restrict__ y) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    y[i] = dia_row(i, nrows, ncols, ndiags, offsets, vals, x);
}

// ---------------------------------------------------------------- ELL -------
// Column-major ELL, one thread per row; slots are consumed in order and the
// row stops at the first sentinel (spmv.cpp:59-71).  Column indices for
// kU slots are fetched together; values/x only for live slots.
template <bool ACCUM>
__global__ void __launch_bounds__(256)
    ell_kernel(int64_t nrows, int width, const int32_t* __restrict__ col,
               const double* __restrict__ val, const double* __restrict__ x,
               double* __restrict__ y) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    constexpr int kU = 4;
    double s = 0.0;
    for (int k0 = 0; k0 < width; k0 += kU) {
        int c[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u)
            c[u] = (k0 + u < width) ? ld_stream(col + int64_t(k0 + u) * nrows + i) : -1;
        bool live[kU];
        bool alive = true;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            alive = alive && c[u] != -1;
            live[u] = alive;
        }
        double p[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u)
            p[u] = live[u] ? fmul(ld_stream(val + int64_t(k0 + u) * nrows + i), __ldg(x + c[u])) : 0.0;
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (live[u]) s = fadd(s, p[u]);
        if (!alive) break;
    }
    y[i] = ACCUM ? fadd(y[i], s) : s;
}

// ---------------------------------------------------------------- COO -------
// Segmented reduction over the row-sorted canonical COO.  CTA c owns the
// fixed chunk [c*kCooChunk, (c+1)*kCooChunk) (perfect load balance whatever
// the row lengths).  Products are staged in shared memory; each thread walks
// kCooItems consecutive entries sequentially (reference order inside a
// thread), pieces of a row that span threads are joined by a block-wide
// segmented scan, and rows that span chunks are finished by coo_fixup in
// chunk order.  Every pass has a fixed order => deterministic.
// ACCUM (HYB coo part): a row's sum starts from the ELL result already in y,
// exactly as the reference's coo_kernel adds into y (spmv.cpp:95-100).
constexpr int kCooBlock = 256;
constexpr int kCooItems = 8;
constexpr int kCooChunk = kCooBlock * kCooItems;

struct CooChunkRec {
    double first_sum;  // in-chunk piece of a segment that began in an earlier chunk
    double last_sum;   // in-chunk piece of the segment that continues past the chunk
    int32_t last_row;
    int32_t flags;
};
enum : int32_t { kFirstCont = 1, kLastOpen = 2, kSingle = 4 };

struct SegPair {
    bool f;
    double v;
};

__device__ __forceinline__ SegPair seg_combine(SegPair a, SegPair b) {
    // a precedes b
    return SegPair{a.f || b.f, b.f ? b.v : fadd(a.v, b.v)};
}

// Exclusive segmented scan over the CTA's threads (identity: {false, 0}).
__device__ SegPair block_excl_seg_scan(SegPair in, SegPair* wsc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    SegPair inc = in;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        SegPair up{bool(__shfl_up_sync(0xffffffffu, int(inc.f), o)),
                   __shfl_up_sync(0xffffffffu, inc.v, o)};
        if (lane >= o) inc = seg_combine(up, inc);
    }
    if (lane == 31) wsc[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        SegPair w = lane < kCooBlock / 32 ? wsc[lane] : SegPair{false, 0.0};
        SegPair wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            SegPair up{bool(__shfl_up_sync(0xffffffffu, int(wi.f), o)),
                       __shfl_up_sync(0xffffffffu, wi.v, o)};
            if (lane >= o) wi = seg_combine(up, wi);
        }
        // exclusive per warp
        SegPair ex{bool(__shfl_up_sync(0xffffffffu, int(wi.f), 1)), __shfl_up_sync(0xffffffffu, wi.v, 1)};
        if (lane == 0) ex = SegPair{false, 0.0};
        if (lane < kCooBlock / 32) wsc[lane] = ex;
    }
    __syncthreads();
    SegPair wex = wsc[warp];
    SegPair lex{bool(__shfl_up_sync(0xffffffffu, int(inc.f), 1)), __shfl_up_sync(0xffffffffu, inc.v, 1)};
    SegPair res;
    if (lane == 0)
        res = wex;
    else
        res = seg_combine(wex, lex);
    return res;
}

template <bool ACCUM>
__global__ void __launch_bounds__(kCooBlock)
    coo_chunk_kernel(int64_t z, int64_t nrows, const int32_t* __restrict__ row,
                     const int32_t* __restrict__ col, const double* __restrict__ val,
                     const double* __restrict__ x, double* __restrict__ y,
                     CooChunkRec* __restrict__ rec) {
    __shared__ double sp[kCooChunk];
    __shared__ int32_t sr[kCooChunk];
    __shared__ SegPair wsc[kCooBlock / 32 + 1];
    const int64_t base = int64_t(blockIdx.x) * kCooChunk;
    const int cnt = int(z - base < kCooChunk ? z - base : int64_t(kCooChunk));
#pragma unroll
    for (int j = 0; j < kCooItems; ++j) {
        const int e = j * kCooBlock + int(threadIdx.x);
        if (e < cnt) {
            const int64_t k = base + e;
            sr[e] = ld_stream(row + k);
            sp[e] = fmul(ld_stream(val + k), __ldg(x + ld_stream(col + k)));
        }
    }
    const int prev_row = base > 0 ? row[base - 1] : -1;
    const int next_row = base + cnt < z ? row[base + cnt] : -1;
    __syncthreads();

    auto is_head = [&](int e) -> bool { return e == 0 ? sr[0] != prev_row : sr[e] != sr[e - 1]; };
    const int first = int(threadIdx.x) * kCooItems;
    const int last = min(first + kCooItems, cnt) - 1;
    const bool has_items = first < cnt;

    // pass 1: this thread's tail piece
    SegPair mine{false, 0.0};
    if (has_items) {
        for (int e = first; e <= last; ++e) {
            if (is_head(e)) {
                mine.f = true;
                mine.v = ACCUM ? y[sr[e]] : 0.0;
            }
            mine.v = fadd(mine.v, sp[e]);
        }
    }
    const SegPair carry = block_excl_seg_scan(mine, wsc);
    if (!has_items) return;

    // pass 2: finish segments
    const bool first_cont = sr[0] == prev_row;
    bool orphan = !carry.f && !is_head(first);  // piece of a segment begun before this chunk
    double s = is_head(first) ? (ACCUM ? y[sr[first]] : 0.0) : carry.v;
    for (int e = first; e <= last; ++e) {
        const bool head = is_head(e);
        if (e > first && head) {
            s = ACCUM ? y[sr[e]] : 0.0;
            orphan = false;
        }
        if (!ACCUM && head) {  // rows strictly between consecutive entries are empty
            const int p = e == 0 ? prev_row : sr[e - 1];
            for (int r = p + 1; r < sr[e]; ++r) y[r] = 0.0;
        }
        s = fadd(s, sp[e]);
        const bool ends = (e + 1 < cnt) ? sr[e + 1] != sr[e] : next_row != sr[e];
        if (ends) {
            if (orphan)
                rec[blockIdx.x].first_sum = s;
            else
                y[sr[e]] = s;
        } else if (e == cnt - 1) {  // continues into the next chunk
            if (orphan) rec[blockIdx.x].first_sum = s;
        }
        if (e == cnt - 1) {
            const bool open = !ends;
            int32_t f = (first_cont ? kFirstCont : 0) | (open ? kLastOpen : 0) |
                        ((open && orphan) ? kSingle : 0);
            rec[blockIdx.x].flags = f;
            rec[blockIdx.x].last_row = sr[e];
            rec[blockIdx.x].last_sum = s;
            if (!ACCUM && base + cnt == z)  // trailing empty rows
                for (int64_t r = int64_t(sr[e]) + 1; r < nrows; ++r) y[r] = 0.0;
        }
    }
}

// Rows spanning chunks: the chunk holding the row's first entry walks forward
// in chunk order (deterministic) and writes the final value.
__global__ void coo_fixup(int64_t nchunks, const CooChunkRec* __restrict__ rec, double* __restrict__ y) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    const int32_t f = rec[c].flags;
    if (!(f & kLastOpen) || (f & kSingle)) return;
    double t = rec[c].last_sum;
    for (int64_t j = c + 1; j < nchunks; ++j) {
        t = fadd(t, rec[j].first_sum);
        if (!(rec[j].flags & kSingle)) break;
    }
    y[rec[c].last_row] = t;
}

template <bool ACCUM>
void launch_coo(const CooPart& coo, int64_t nrows, const double* x, double* y, cudaStream_t s) {
    const int64_t nchunks = ceil_div(coo.nnz, kCooChunk);
    DBuf<CooChunkRec> rec(nchunks, s);
    coo_chunk_kernel<ACCUM><<<unsigned(nchunks), kCooBlock, 0, s>>>(
        coo.nnz, nrows, coo.row.get(), coo.col.get(), coo.val.get(), x, y, rec.get());
    SOB_LAUNCH("coo_chunk_kernel");
    coo_fixup<<<unsigned(ceil_div(nchunks, 256)), 256, 0, s>>>(nchunks, rec.get(), y);
    SOB_LAUNCH("coo_fixup");
}

void launch_csr_stream(const so_matrix& m, bool with_dia, const double* x, double* y, cudaStream_t s) {
    const CsrPart& c = m.csr;
    const size_t smem = sizeof(double) * 2 * kWindow;
    if (with_dia) {
        csr_stream_kernel<true><<<unsigned(c.nblk), kStreamBlock, smem, s>>>(
            c.blk.get(), c.row_ptr.get(), c.col.get(), c.val.get(), x, y, m.nrows, m.ncols,
            int(m.dia.ndiags), m.dia.offsets.get(), m.dia.values.get());
    } else {
        csr_stream_kernel<false><<<unsigned(c.nblk), kStreamBlock, smem, s>>>(
            c.blk.get(), c.row_ptr.get(), c.col.get(), c.val.get(), x, y, m.nrows, m.ncols, 0,
            nullptr, nullptr);
    }
    SOB_LAUNCH("csr_stream_kernel");
}

void launch_dia(const so_matrix& m, const double* x, double* y, cudaStream_t s) {
    dia_kernel<<<unsigned(ceil_div(m.nrows, 256)), 256, 0, s>>>(
        m.nrows, m.ncols, int(m.dia.ndiags), m.dia.offsets.get(), m.dia.values.get(), x, y);
    SOB_LAUNCH("dia_kernel");
}

template <bool ACCUM>
void launch_ell(const so_matrix& m, const double* x, double* y, cudaStream_t s) {
    ell_kernel<ACCUM><<<unsigned(ceil_div(m.nrows, 256)), 256, 0, s>>>(
        m.nrows, int(m.ell.width), m.ell.col.get(), m.ell.val.get(), x, y);
    SOB_LAUNCH("ell_kernel");
}

}  // namespace

void spmv_device(const so_matrix& m, const double* x, double* y, cudaStream_t s) {
    if (m.nrows <= 0) return;
    switch (m.format) {
        case SO_COO:
            if (m.coo.nnz == 0) {
                SOB_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * size_t(m.nrows), s));
            } else {
                launch_coo<false>(m.coo, m.nrows, x, y, s);
            }
            break;
        case SO_CSR:
            launch_csr_stream(m, false, x, y, s);
            break;
        case SO_DIA:
            launch_dia(m, x, y, s);
            break;
        case SO_ELL:
            launch_ell<false>(m, x, y, s);
            break;
        case SO_HYB:
            launch_ell<false>(m, x, y, s);
            if (m.coo.nnz > 0) launch_coo<true>(m.coo, m.nrows, x, y, s);
            break;
        case SO_HDC:
            launch_csr_stream(m, true, x, y, s);
            break;
        default:
            fail(SO_INVALID_INPUT, "unknown format");
    }
}

}  // namespace sob
