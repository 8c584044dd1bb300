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
#include <algorithm>

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
// per row: y[i] += diag[i] * x[i + off] for every in-range diagonal).  Eight
// diagonals are fetched before any is accumulated so each thread keeps eight
// coalesced HBM loads in flight; in-range holes multiply as 0 * x exactly as
// the reference does.
constexpr int kDiaSmem = 512;

// offsets come from shared memory (staged per CTA) when ndiags <= kDiaSmem,
// else straight from global memory (GLOBAL_OFF)
template <bool GLOBAL_OFF>
__device__ __forceinline__ double dia_row(int64_t i, int64_t nrows, int64_t ncols, int ndiags,
                                          const int64_t* __restrict__ soff,
                                          const int64_t* __restrict__ offsets,
                                          const double* __restrict__ vals,
                                          const double* __restrict__ x) {
    constexpr int U = 8;
    const int64_t* off = GLOBAL_OFF ? offsets : soff;
    double acc = 0.0;
    int d0 = 0;
    for (; d0 + U <= ndiags; d0 += U) {
        double v[U], xv[U];
        bool ok[U];
        // unpredicated loads (cells outside the column range exist in the
        // diagonal-major array, x index is clamped) so all 2U loads issue
        // back to back; only in-range diagonals are accumulated
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int d = d0 + u;
            const int64_t c = i + off[d];
            ok[u] = c >= 0 && c < ncols;
            const int64_t cc = c < 0 ? 0 : (c >= ncols ? ncols - 1 : c);
            v[u] = ld_stream(vals + int64_t(d) * nrows + i);
            xv[u] = __ldg(x + cc);
        }
        // x + (-0.0) == x exactly for every x (round-to-nearest), so skipped
        // diagonals add -0.0: an unconditional chain keeps the loads hoisted
#pragma unroll
        for (int u = 0; u < U; ++u) acc = fadd(acc, ok[u] ? fmul(v[u], xv[u]) : -0.0);
    }
    for (; d0 < ndiags; ++d0) {
        const int64_t c = i + off[d0];
        if (c >= 0 && c < ncols) acc = fadd(acc, fmul(ld_stream(vals + int64_t(d0) * nrows + i), __ldg(x + c)));
    }
    return acc;
}

__device__ __forceinline__ void stage_offsets(int64_t* soff, const int64_t* __restrict__ offsets, int ndiags) {
    const int m = ndiags < kDiaSmem ? ndiags : kDiaSmem;
    for (int d = threadIdx.x; d < m; d += blockDim.x) soff[d] = offsets[d];
    __syncthreads();
}

// ---------------------------------------------------------------- CSR -------
// Streaming CSR ("CSR-stream"), persistent and software-pipelined.  Window w
// owns rows [blk[w], blk[w+1]) whose entries [blk_k[w], blk_k[w+1]) (at most
// 2*kWindow) are contiguous.  Phase 1 gathers x for the window's col/val
// (already in registers) and stages the rounded products in shared memory;
// then the col/val (and row_ptr) loads of the CTA's NEXT window are issued so
// they are in flight while phase 2 gives each row to one thread that sums its
// products in the reference order (bit-exact).  WITH_DIA fuses the HDC DIA
// part in front of the CSR part (spmv.cpp:101-106).  Windows holding a single
// row longer than 2*kWindow are skipped here: csr_long_pieces + csr_long_fixup
// split them over many CTAs.
// Warp-level CSR stream.  Group g = rows [grp[g], grp[g+1]) (<= 32 rows,
// entries [grp_k[g], grp_k[g+1]) <= 32*IT) is owned by one warp: coalesced
// col/val loads (IT per lane), x gather, rounded products into warp-private
// shared memory, then lane i sums row grp[g]+i sequentially (reference order,
// bit-exact).  The next group's loads are issued before the sums, so each
// warp keeps 2*IT loads in flight with no CTA-wide barrier anywhere.
template <int IT, bool WITH_DIA>
__global__ void __launch_bounds__(256, (IT > 8 ? 3 : 4))
    csr_warp_kernel(const int32_t* __restrict__ grp, const int64_t* __restrict__ grp_k, int64_t ngrp,
                    const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                    const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
                    int64_t nrows, int64_t ncols, int ndiags, const int64_t* __restrict__ offsets,
                    const double* __restrict__ dvals) {
    __shared__ double sp[8][32 * IT];
    __shared__ int64_t soff[WITH_DIA ? kDiaSmem : 1];
    if (WITH_DIA) stage_offsets(soff, offsets, ndiags);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* prod = sp[wid];
    int64_t g = int64_t(blockIdx.x) * 8 + wid;
    const int64_t stride = int64_t(gridDim.x) * 8;
    if (g >= ngrp) return;
    int r0 = grp[g], r1 = grp[g + 1];
    int64_t k0 = grp_k[g], k1 = grp_k[g + 1];
    int c[IT];
    double v[IT];
    bool longrow = k1 - k0 > 32 * IT;
#pragma unroll
    for (int u = 0; u < IT; ++u) {
        const int64_t k = k0 + u * 32 + lane;
        if (!longrow && k < k1) {
            c[u] = ld_stream(col + k);
            v[u] = ld_stream(val + k);
        }
    }
    int64_t pa = 0, pe = 0;
    if (r0 + lane < r1) {
        pa = rp[r0 + lane];
        pe = rp[r0 + lane + 1];
    }
    while (true) {
        const int64_t gn = g + stride;
        int nr0 = 0, nr1 = 0;
        int64_t nk0 = 0, nk1 = 0;
        if (gn < ngrp) {
            nr0 = grp[gn];
            nr1 = grp[gn + 1];
            nk0 = grp_k[gn];
            nk1 = grp_k[gn + 1];
        }
        if (!longrow) {
#pragma unroll
            for (int u = 0; u < IT; ++u) {
                const int64_t k = k0 + u * 32 + lane;
                if (k < k1) prod[u * 32 + lane] = fmul(v[u], __ldg(x + c[u]));
            }
        }
        __syncwarp();
        const bool nlong = nk1 - nk0 > 32 * IT;
        int64_t npa = 0, npe = 0;
        if (gn < ngrp) {
#pragma unroll
            for (int u = 0; u < IT; ++u) {
                const int64_t k = nk0 + u * 32 + lane;
                if (!nlong && k < nk1) {
                    c[u] = ld_stream(col + k);
                    v[u] = ld_stream(val + k);
                }
            }
            if (nr0 + lane < nr1) {
                npa = rp[nr0 + lane];
                npe = rp[nr0 + lane + 1];
            }
        }
        if (!longrow && r0 + lane < r1) {
            const int r = r0 + lane;
            double s = 0.0;
            for (int64_t j = pa - k0; j < pe - k0; ++j) s = fadd(s, prod[j]);
            if (WITH_DIA)
                s = fadd(ndiags <= kDiaSmem ? dia_row<false>(r, nrows, ncols, ndiags, soff, offsets, dvals, x)
                                            : dia_row<true>(r, nrows, ncols, ndiags, soff, offsets, dvals, x),
                         s);
            y[r] = s;
        }
        __syncwarp();
        if (gn >= ngrp) break;
        g = gn;
        r0 = nr0;
        r1 = nr1;
        k0 = nk0;
        k1 = nk1;
        pa = npa;
        pe = npe;
        longrow = nlong;
    }
}

// Rows longer than 2*grp_window: piece p covers entries [pk[2p], pk[2p+1]) of row
// prow[p] (<= kPiece entries, 8 independent loads per thread), reduced with a
// fixed tree into part[p]; csr_long_fixup then adds the pieces of each row in
// piece order (deterministic, within the 1e-12 contract).
__global__ void __launch_bounds__(kStreamBlock)
    csr_long_pieces(const int64_t* __restrict__ pk, const int32_t* __restrict__ col,
                    const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ part) {
    __shared__ double scratch[kStreamBlock / 32];
    const int64_t k0 = pk[2 * blockIdx.x], k1 = pk[2 * blockIdx.x + 1];
    constexpr int U = kPiece / kStreamBlock;
    int c[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t k = k0 + u * kStreamBlock + threadIdx.x;
        c[u] = k < k1 ? ld_stream(col + k) : 0;
        v[u] = k < k1 ? ld_stream(val + k) : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t k = k0 + u * kStreamBlock + threadIdx.x;
        if (k < k1) s = fadd(s, fmul(v[u], __ldg(x + c[u])));
    }
    const double t = block_sum_det<kStreamBlock>(s, scratch);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

template <bool WITH_DIA>
__global__ void csr_long_fixup(int64_t nlong, const int32_t* __restrict__ lrow, const int64_t* __restrict__ lpiece,
                               const double* __restrict__ part, double* __restrict__ y, int64_t nrows, int64_t ncols,
                               int ndiags, const int64_t* __restrict__ offsets, const double* __restrict__ dvals,
                               const double* __restrict__ x) {
    const int64_t l = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (l >= nlong) return;
    double t = 0.0;
    for (int64_t p = lpiece[l]; p < lpiece[l + 1]; ++p) t = fadd(t, part[p]);
    const int r = lrow[l];
    if (WITH_DIA) t = fadd(dia_row<true>(r, nrows, ncols, ndiags, nullptr, offsets, dvals, x), t);
    y[r] = t;
}

// ---------------------------------------------------------------- DIA -------
// One thread per row, diagonals ascending: consecutive threads read
// consecutive cells of each diagonal (diagonal-major layout => coalesced).
template <bool GLOBAL_OFF>
__global__ void __launch_bounds__(256, 8)
    dia_kernel(int64_t nrows, int64_t ncols, int ndiags, const int64_t* __restrict__ offsets,
               const double* __restrict__ vals, const double* __restrict__ x,
               double* __restrict__ y, int64_t row_lo, int64_t row_hi) {
    __shared__ int64_t soff[GLOBAL_OFF ? 1 : kDiaSmem];
    if (!GLOBAL_OFF) stage_offsets(soff, offsets, ndiags);
    const int64_t i = row_lo + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= row_hi) return;
    y[i] = dia_row<GLOBAL_OFF>(i, nrows, ncols, ndiags, soff, offsets, vals, x);
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

// shared-memory slot of chunk item e: one pad slot per kCooItems keeps the
// per-thread sequential reads (items t*8 .. t*8+7) bank-conflict free
__device__ __forceinline__ int coo_slot(int e) { return e + (e >> 3); }

template <bool ACCUM>
__global__ void __launch_bounds__(kCooBlock, 6)
    coo_chunk_kernel(int64_t z, int64_t nrows, const int32_t* __restrict__ row,
                     const int32_t* __restrict__ col, const double* __restrict__ val,
                     const double* __restrict__ x, double* __restrict__ y,
                     CooChunkRec* __restrict__ rec) {
    __shared__ double sp[kCooChunk + kCooChunk / kCooItems];
    __shared__ int32_t sr[kCooChunk + kCooChunk / kCooItems];
    __shared__ SegPair wsc[kCooBlock / 32 + 1];
    const int64_t base = int64_t(blockIdx.x) * kCooChunk;
    const int cnt = int(z - base < kCooChunk ? z - base : int64_t(kCooChunk));
    const int prev_row = base > 0 ? row[base - 1] : -1;
    const int next_row = base + cnt < z ? row[base + cnt] : -1;
#pragma unroll
    for (int j = 0; j < kCooItems; ++j) {
        const int e = j * kCooBlock + int(threadIdx.x);
        if (e < cnt) {
            const int64_t k = base + e;
            sr[coo_slot(e)] = ld_stream(row + k);
            sp[coo_slot(e)] = fmul(ld_stream(val + k), __ldg(x + ld_stream(col + k)));
        }
    }
    __syncthreads();

    // this thread's kCooItems consecutive entries, in registers
    const int first = int(threadIdx.x) * kCooItems;
    const int nmine = cnt - first < 0 ? 0 : (cnt - first > kCooItems ? kCooItems : cnt - first);
    int rr[kCooItems];
    double pp[kCooItems];
#pragma unroll
    for (int j = 0; j < kCooItems; ++j) {
        rr[j] = j < nmine ? sr[coo_slot(first + j)] : -1;
        pp[j] = j < nmine ? sp[coo_slot(first + j)] : 0.0;
    }
    const int r_before = nmine == 0 ? -1 : (first == 0 ? prev_row : sr[coo_slot(first - 1)]);
    const int r_after = nmine == 0 ? -1 : (first + nmine < cnt ? sr[coo_slot(first + nmine)] : next_row);
    const int chunk_first_row = sr[0];

    // pass 1: this thread's tail piece (sum of its last segment)
    SegPair mine{false, 0.0};
#pragma unroll
    for (int j = 0; j < kCooItems; ++j) {
        if (j < nmine) {
            const bool head = rr[j] != (j == 0 ? r_before : rr[j - 1]);
            if (head) {
                mine.f = true;
                mine.v = ACCUM ? y[rr[j]] : 0.0;
            }
            mine.v = fadd(mine.v, pp[j]);
        }
    }
    const SegPair carry = block_excl_seg_scan(mine, wsc);
    if (nmine == 0) return;

    // pass 2: finish segments
    const bool first_cont = chunk_first_row == prev_row;
    const bool head0 = rr[0] != r_before;
    bool orphan = !carry.f && !head0;  // piece of a segment begun before this chunk
    double s = head0 ? (ACCUM ? y[rr[0]] : 0.0) : carry.v;
#pragma unroll
    for (int j = 0; j < kCooItems; ++j) {
        if (j < nmine) {
            const int prv = j == 0 ? r_before : rr[j - 1];
            const bool head = rr[j] != prv;
            if (j > 0 && head) {
                s = ACCUM ? y[rr[j]] : 0.0;
                orphan = false;
            }
            if (!ACCUM && head)  // rows strictly between consecutive entries are empty
                for (int r = prv + 1; r < rr[j]; ++r) y[r] = 0.0;
            s = fadd(s, pp[j]);
            const int nxt = j + 1 < nmine ? rr[j + 1] : r_after;
            const bool ends = nxt != rr[j];
            const bool chunk_last = first + j == cnt - 1;
            if (ends) {
                if (orphan)
                    rec[blockIdx.x].first_sum = s;
                else
                    y[rr[j]] = s;
            } else if (chunk_last && orphan) {  // continues into the next chunk
                rec[blockIdx.x].first_sum = s;
            }
            if (chunk_last) {
                const bool open = !ends;
                rec[blockIdx.x].flags = (first_cont ? kFirstCont : 0) | (open ? kLastOpen : 0) |
                                        ((open && orphan) ? kSingle : 0);
                rec[blockIdx.x].last_row = rr[j];
                rec[blockIdx.x].last_sum = s;
                if (!ACCUM && base + cnt == z)  // trailing empty rows
                    for (int64_t r = int64_t(rr[j]) + 1; r < nrows; ++r) y[r] = 0.0;
            }
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

template <int IT>
void launch_csr_warp(const so_matrix& m, bool with_dia, const double* x, double* y, cudaStream_t s) {
    const CsrPart& c = m.csr;
    const int per_sm = IT > 8 ? 3 : 4;
    const int grid = int(std::min<int64_t>(ceil_div(c.ngrp, 8), int64_t(current_ctx().num_sms) * per_sm));
    if (with_dia)
        csr_warp_kernel<IT, true><<<grid, 256, 0, s>>>(c.grp.get(), c.grp_k.get(), c.ngrp, c.row_ptr.get(),
                                                       c.col.get(), c.val.get(), x, y, m.nrows, m.ncols,
                                                       int(m.dia.ndiags), m.dia.offsets.get(), m.dia.values.get());
    else
        csr_warp_kernel<IT, false><<<grid, 256, 0, s>>>(c.grp.get(), c.grp_k.get(), c.ngrp, c.row_ptr.get(),
                                                        c.col.get(), c.val.get(), x, y, m.nrows, m.ncols, 0,
                                                        nullptr, nullptr);
    SOB_LAUNCH("csr_warp_kernel");
}

void launch_csr_stream(const so_matrix& m, bool with_dia, const double* x, double* y, cudaStream_t s) {
    const CsrPart& c = m.csr;
    if (c.ngrp == 0) return;
    if (c.grp_window == kGroupWindowShort)
        launch_csr_warp<2 * kGroupWindowShort / 32>(m, with_dia, x, y, s);
    else
        launch_csr_warp<2 * kGroupWindowLong / 32>(m, with_dia, x, y, s);
    if (c.nlong > 0) {
        const int nd = with_dia ? int(m.dia.ndiags) : 0;
        DBuf<double> part(c.npieces, s);
        csr_long_pieces<<<unsigned(c.npieces), kStreamBlock, 0, s>>>(c.piece_k.get(), c.col.get(), c.val.get(), x,
                                                                     part.get());
        SOB_LAUNCH("csr_long_pieces");
        const unsigned g = unsigned(ceil_div(c.nlong, 128));
        if (with_dia)
            csr_long_fixup<true><<<g, 128, 0, s>>>(c.nlong, c.long_row.get(), c.long_piece.get(), part.get(), y,
                                                  m.nrows, m.ncols, nd, m.dia.offsets.get(), m.dia.values.get(), x);
        else
            csr_long_fixup<false><<<g, 128, 0, s>>>(c.nlong, c.long_row.get(), c.long_piece.get(), part.get(), y,
                                                   m.nrows, m.ncols, 0, nullptr, nullptr, x);
        SOB_LAUNCH("csr_long_fixup");
    }
}

void launch_dia(const so_matrix& m, const double* x, double* y, cudaStream_t s, int64_t lo = 0,
                int64_t hi = -1) {
    if (hi < 0) hi = m.nrows;
    if (hi <= lo) return;
    const unsigned grid = unsigned(ceil_div(hi - lo, 256));
    if (m.dia.ndiags <= kDiaSmem)
        dia_kernel<false><<<grid, 256, 0, s>>>(m.nrows, m.ncols, int(m.dia.ndiags), m.dia.offsets.get(),
                                               m.dia.values.get(), x, y, lo, hi);
    else
        dia_kernel<true><<<grid, 256, 0, s>>>(m.nrows, m.ncols, int(m.dia.ndiags), m.dia.offsets.get(),
                                              m.dia.values.get(), x, y, lo, hi);
    SOB_LAUNCH("dia_kernel");
}

template <bool ACCUM>
void launch_ell(const so_matrix& m, const double* x, double* y, cudaStream_t s) {
    ell_kernel<ACCUM><<<unsigned(ceil_div(m.nrows, 256)), 256, 0, s>>>(
        m.nrows, int(m.ell.width), m.ell.col.get(), m.ell.val.get(), x, y);
    SOB_LAUNCH("ell_kernel");
}

}  // namespace

void spmv_device_rows(const so_matrix& m, const double* x, double* y, int64_t lo, int64_t hi, cudaStream_t s) {
    if (m.format != SO_DIA) fail(SO_INVALID_INPUT, "row-range SpMV is implemented for DIA matrices");
    if (lo < 0 || hi > m.nrows || lo > hi) fail(SO_INVALID_INPUT, "row range outside the matrix");
    launch_dia(m, x, y, s, lo, hi);
}

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
            // one kernel per non-empty part; both parts -> fused per-row kernel
            if (m.csr.nnz == 0)
                launch_dia(m, x, y, s);
            else
                launch_csr_stream(m, m.dia.ndiags > 0, x, y, s);
            break;
        default:
            fail(SO_INVALID_INPUT, "unknown format");
    }
}

}  // namespace sob
