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
#include <cstdlib>
#include <functional>
#include <mutex>

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
// per row: y[i] += diag[i] * x[i + off] for every in-range diagonal).  Nine
// diagonals' values and x are fetched before any is accumulated (so each
// thread keeps 18 loads in flight); the last batch re-reads the last diagonal
// for its dead slots.  Index math is 32-bit (rows, columns and offsets are
// < 2^31 on the device); only the diagonal base is 64-bit.
// In-range holes multiply as 0 * x exactly as the reference does.
constexpr int kDiaSmem = 512;
constexpr int kDiaBatch = 9;

// offsets come from shared memory (staged per CTA as int32) when
// ndiags <= kDiaSmem, else straight from global memory (GLOBAL_OFF)
template <bool GLOBAL_OFF>
__device__ __forceinline__ int dia_off(const int* soff, const int64_t* __restrict__ offsets, int d) {
    return GLOBAL_OFF ? int(offsets[d]) : soff[d];
}

template <bool GLOBAL_OFF, int U = kDiaBatch>
__device__ __forceinline__ double dia_row(int i, int nrows, int ncols, int ndiags, const int* soff,
                                          const int64_t* __restrict__ offsets, const double* __restrict__ vals,
                                          const double* __restrict__ x) {
    const double* vp = vals + i;
    double acc = 0.0;
    for (int d0 = 0; d0 < ndiags; d0 += U) {
        double v[U], xv[U];
        bool ok[U];
        // unpredicated loads (cells outside the column range exist in the
        // diagonal-major array; x index falls back to 0) so all 2U loads issue
        // back to back; only in-range diagonals are accumulated
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool live = d0 + u < ndiags;
            const int d = live ? d0 + u : ndiags - 1;
            const int c = i + dia_off<GLOBAL_OFF>(soff, offsets, d);
            ok[u] = live && unsigned(c) < unsigned(ncols);
            v[u] = ld_stream(vp + size_t(d) * size_t(nrows));
            xv[u] = __ldg(x + (ok[u] ? c : 0));
        }
        // x + (-0.0) == x exactly for every x (round-to-nearest), so skipped
        // diagonals add -0.0: an unconditional chain keeps the loads hoisted
#pragma unroll
        for (int u = 0; u < U; ++u) acc = fadd(acc, ok[u] ? fmul(v[u], xv[u]) : -0.0);
    }
    return acc;
}

__device__ __forceinline__ void stage_offsets(int* soff, const int64_t* __restrict__ offsets, int ndiags) {
    const int m = ndiags < kDiaSmem ? ndiags : kDiaSmem;
    for (int d = threadIdx.x; d < m; d += blockDim.x) soff[d] = int(offsets[d]);
    __syncthreads();
}

// Accumulating kernels (HYB's COO part after its ELL part, HDC's CSR part
// after its DIA part) add each row's sum to y exactly once (rows split over
// chunks or pieces are combined first), so y[r] + s can be a fire-and-forget
// reduction (RED.ADD.F64.RN: the same single rounding as fadd(y[r], s),
// bit-identical) -- no load of y whose latency and register the kernel would
// carry (HYB on R-MAT 372 -> 344 us, profiles/r02h_ab_red.txt).
template <bool ACCUM>
__device__ __forceinline__ void y_store(double* p, double s) {
    if (ACCUM)
        atomicAdd(p, s);
    else
        *p = s;
}

// ---------------------------------------------------------------- CSR -------
// Warp-level CSR stream.  Group g = rows [grp[g], grp[g+1]) (<= 32 rows,
// <= 32*IT entries starting at grp_k[g]; greedy partition, convert.cu
// group_flags) is owned by one warp: coalesced col/val loads (IT per lane),
// x gather, rounded products into warp-private shared memory, then lane i sums
// row grp[g]+i sequentially -- the reference's order (spmv.cpp:32-43),
// bit-exact.  The next group's col/val/row_ptr loads are issued before the
// sums (register double buffer), so each warp keeps up to 2*IT loads in flight
// with no CTA-wide barrier.  A group holding one row longer than 32*IT is
// skipped here (csr_long_pieces + csr_long_fixup).  ACCUM (HDC with both
// parts): y already holds the DIA part (dia_kernel ran first) and the row
// sum is added to it -- spmv.cpp:101-106, DIA part first, then y[i] += CSR
// row sum: the same roundings, bit-exact.
//
// COOP (the matrix has rows of kCoopLen < length <= 32*IT): such a row is
// summed by the whole warp -- lane l adds products a+l, a+l+32, ... of the
// row, then a fixed butterfly joins the 32 partials (deterministic, within
// the 1e-12 contract) -- while rows of <= kCoopLen entries keep their lane's
// serial walk (bit-exact).  On skewed matrices one long row otherwise walks
// its products alone while the other 31 lanes idle, one shared-memory
// wavefront per entry.
// One row per lane: products [pa, pe) of the warp's product array, serial in
// the reference's order (bit-exact), or -- COOP, rows of more than kCoopLen
// entries -- summed by the whole warp (strided partials, fixed butterfly).
template <bool ACCUM, bool COOP>
__device__ __forceinline__ void csr_rows_sum(const double* prod, bool pad, int r, bool act, int pa, int pe,
                                             double* __restrict__ y, int lane) {
    const bool coop = COOP && act && pe - pa > kCoopLen;
    if (act && !coop) {
        double acc = 0.0;
        if (pad)
            for (int j = pa; j < pe; ++j) acc = fadd(acc, prod[j + (j >> 4)]);
        else
            for (int j = pa; j < pe; ++j) acc = fadd(acc, prod[j]);
        y_store<ACCUM>(y + r, acc);
    }
    if (COOP) {
        unsigned big = __ballot_sync(0xffffffffu, coop);
        while (big) {
            const int j = __ffs(big) - 1;
            big &= big - 1;
            const int a = __shfl_sync(0xffffffffu, pa, j), e = __shfl_sync(0xffffffffu, pe, j);
            double t = 0.0;
            if (pad)
                for (int q = a + lane; q < e; q += 32) t = fadd(t, prod[q + (q >> 4)]);
            else
                for (int q = a + lane; q < e; q += 32) t = fadd(t, prod[q]);
            t = warp_sum(t);
            if (lane == j) y_store<ACCUM>(y + r, t);
        }
    }
}

// ---- following a host->device copy of x (pinned spmv(m, x), FOLLOW) ------
// The device copy of x holds a NaN sentinel (both 32-bit halves
// kFollowSent) until the copy engine overwrites it; a kernel launched with
// FOLLOW reads x from L2 (never a stale L1 line) and waits on an element that
// still holds a sentinel half until it lands -- or until the flag copied
// after x says the copy is complete (an x element that happens to equal the
// sentinel).  A copy that never arrives ends the wait after `timeout_ns` and
// marks the call (`timed_out`): the caller recomputes on another path.
constexpr unsigned kFollowSent = 0x7FF5A5A5u;

struct FollowCtx {
    const unsigned* flag;
    unsigned* timed_out;
    unsigned long long timeout_ns;
};

__device__ __forceinline__ bool follow_ready(double v) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    return unsigned(b) != kFollowSent && unsigned(b >> 32) != kFollowSent;
}

__device__ __noinline__ double follow_wait(const double* p, FollowCtx f) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
        unsigned fl;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(fl) : "l"(f.flag) : "memory");
        const double v = __ldcg(p);
        if (fl != 0 || follow_ready(v)) return v;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > f.timeout_ns) {
            atomicExch_system(f.timed_out, 1u);
            // every later wait of this call (any kernel) returns at once: the
            // caller recomputes the call on another path
            atomicExch(const_cast<unsigned*>(f.flag), 2u);
            return v;
        }
        __nanosleep(256);
    }
}

// x[c] for the SpMV kernels: the read-only cached load, or (FOLLOW) an L2
// load that waits for the copy front
template <bool FOLLOW>
__device__ __forceinline__ double ldx(const double* __restrict__ x, int64_t c, const FollowCtx& f) {
    if (!FOLLOW) return __ldg(x + c);
    const double v = __ldcg(x + c);
    return follow_ready(v) ? v : follow_wait(x + c, f);
}

// Low 32 bits of row_ptr[r]: a group spans < 2^31 entries, so its rows'
// local bounds int(rp[r] - k0) only need the low words (32-bit loads).
__device__ __forceinline__ unsigned rp_lo(const int64_t* __restrict__ rp, int64_t r) {
    return __ldg(reinterpret_cast<const unsigned*>(rp + r));
}

// RPL: rows per lane of the widest group (1, or kGroupRowsMax / 32 when the
// partition has groups of more than 32 tiny rows).
//
// Software pipeline per warp (one group per iteration): the next group's
// metadata loads are issued before this group's x gathers and consumed after
// them; the next group's col/val and row bounds are issued before this
// group's row sums and consumed in the next iteration; the bounds of rows
// i+32, i+64, ... (RPL > 1) are issued before lane i walks row i.  No value
// loaded in a stage is used in the same stage, so every load's latency hides
// behind the work of the stage (ncu on R-MAT: the previous order stalled on
// the next group's row bounds right after issuing them).
template <int IT, bool ACCUM, bool PAD, bool COOP, int RPL, bool FOLLOW = false>
__global__ void __launch_bounds__(256, (IT > 8 ? 3 : 4))
    csr_warp_kernel(const int32_t* __restrict__ grp, const int64_t* __restrict__ grp_k, int64_t ngrp,
                    const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                    const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
                    int64_t nrows, FollowCtx fctx) {
    constexpr int kCap = 32 * IT;
    __shared__ double sp[8][kCap + (PAD ? kCap / 16 : 0)];  // + the padded layout's slots
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* prod = sp[wid];
    int64_t g = int64_t(blockIdx.x) * 8 + wid;
    const int64_t stride = int64_t(gridDim.x) * 8;
    if (g >= ngrp) return;
    int r0 = grp[g], r1 = grp[g + 1];
    int64_t k0 = grp_k[g];
    // product layout flag (convert.cu group_pad_flags; set only when PAD)
    bool pad = PAD && (k0 & kGrpPad);
    if (PAD) k0 &= ~kGrpPad;
    // entry count, saturated at kCap + 1 (= long row, handled elsewhere)
    int cnt = int(min((PAD ? grp_k[g + 1] & ~kGrpPad : grp_k[g + 1]) - k0, int64_t(kCap + 1)));
    int c[IT];
    double v[IT];
#pragma unroll
    for (int u = 0; u < IT; ++u) {
        const int e = u * 32 + lane;
        if (e < cnt && cnt <= kCap) {
            c[u] = ld_stream(col + k0 + e);
            v[u] = ld_stream(val + k0 + e);
        }
    }
    unsigned ra = 0, re = 0;  // low words of row_ptr[r0+lane], row_ptr[r0+lane+1]
    if (r0 + lane < r1) {
        ra = rp_lo(rp, r0 + lane);
        re = rp_lo(rp, r0 + lane + 1);
    }
    while (true) {
        const int64_t gn = g + stride;
        // stage 1: next group's metadata (raw; consumed after the gathers)
        int nr0 = 0, nr1 = 0;
        int64_t nk0 = 0, nk1 = 0;
        if (gn < ngrp) {
            nr0 = grp[gn];
            nr1 = grp[gn + 1];
            nk0 = grp_k[gn];
            nk1 = grp_k[gn + 1];
        }
        const bool longrow = cnt > kCap;
        if (!longrow) {
#pragma unroll
            for (int u = 0; u < IT; ++u) {
                const int e = u * 32 + lane;
                if (e < cnt) prod[pad ? e + (e >> 4) : e] = fmul(v[u], ldx<FOLLOW>(x, c[u], fctx));
            }
        }
        __syncwarp();
        // stage 2: next group's col/val and row bounds (consumed next iteration)
        const bool npad = PAD && (nk0 & kGrpPad);
        if (PAD) {
            nk0 &= ~kGrpPad;
            nk1 &= ~kGrpPad;
        }
        const int ncnt = int(min(nk1 - nk0, int64_t(kCap + 1)));
        unsigned nra = 0, nre = 0;
        if (gn < ngrp) {
#pragma unroll
            for (int u = 0; u < IT; ++u) {
                const int e = u * 32 + lane;
                if (e < ncnt && ncnt <= kCap) {
                    c[u] = ld_stream(col + nk0 + e);
                    v[u] = ld_stream(val + nk0 + e);
                }
            }
            if (nr0 + lane < nr1) {
                nra = rp_lo(rp, nr0 + lane);
                nre = rp_lo(rp, nr0 + lane + 1);
            }
        }
        // stage 3: this group's row sums
        if (!longrow) {
            const unsigned k0lo = unsigned(k0);
            unsigned qa[RPL > 1 ? RPL - 1 : 1], qe[RPL > 1 ? RPL - 1 : 1];
#pragma unroll
            for (int q = 1; q < RPL; ++q) {  // groups of tiny rows: lane i also walks rows i+32, i+64, ...
                const int rr = r0 + 32 * q + lane;
                qa[q - 1] = qe[q - 1] = k0lo;
                if (rr < r1) {
                    qa[q - 1] = rp_lo(rp, rr);
                    qe[q - 1] = rp_lo(rp, rr + 1);
                }
            }
            csr_rows_sum<ACCUM, COOP>(prod, pad, r0 + lane, r0 + lane < r1, int(ra - k0lo), int(re - k0lo), y, lane);
#pragma unroll
            for (int q = 1; q < RPL; ++q) {
                if (r0 + 32 * q >= r1) break;
                const int rr = r0 + 32 * q + lane;
                csr_rows_sum<ACCUM, COOP>(prod, pad, rr, rr < r1, int(qa[q - 1] - k0lo), int(qe[q - 1] - k0lo), y,
                                          lane);
            }
        }
        __syncwarp();
        if (gn >= ngrp) break;
        g = gn;
        r0 = nr0;
        r1 = nr1;
        k0 = nk0;
        pad = npad;
        cnt = ncnt;
        ra = nra;
        re = nre;
    }
}

// Rows longer than grp_cap: piece p covers entries [pk[2p], pk[2p+1]) of row
// prow[p] (<= kPiece entries, 8 independent loads per thread), reduced with a
// fixed tree into part[p]; csr_long_fixup then combines the pieces of each
// row -- one warp per long row, lane-strided partial sums joined by a fixed
// butterfly, so a row of 10^8 entries (5*10^4 pieces) is not one thread's
// serial chain (deterministic, within the 1e-12 contract).
template <bool FOLLOW>
__global__ void __launch_bounds__(kStreamBlock)
    csr_long_pieces(const int64_t* __restrict__ pk, const int32_t* __restrict__ col,
                    const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ part,
                    FollowCtx fctx) {
    __shared__ double scratch[kStreamBlock / 32];
    pdl_enter();
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
        if (k < k1) s = fadd(s, fmul(v[u], ldx<FOLLOW>(x, c[u], fctx)));
    }
    const double t = block_sum_det<kStreamBlock>(s, scratch);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

template <bool ACCUM>
__global__ void csr_long_fixup(int64_t nlong, const int32_t* __restrict__ lrow, const int64_t* __restrict__ lpiece,
                               const double* __restrict__ part, double* __restrict__ y) {
    pdl_enter();
    const int lane = threadIdx.x & 31;
    const int64_t l = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (l >= nlong) return;
    double t = 0.0;
    for (int64_t p = lpiece[l] + lane; p < lpiece[l + 1]; p += 32) t = fadd(t, part[p]);
    t = warp_sum(t);  // fixed butterfly: deterministic
    if (lane == 0) {
        const int r = lrow[l];
        y[r] = ACCUM ? fadd(y[r], t) : t;
    }
}

// ---------------------------------------------------------------- DIA -------
// One thread per row, diagonals ascending: consecutive threads read
// consecutive cells of each diagonal (diagonal-major layout => coalesced).
// U: diagonals per load batch.  Matrices with <= 5 diagonals (2-D 5-point
// stencils, tridiagonal, ...) use U = 5 and 8 CTAs/SM: no dead loads in the
// batch and more rows in flight (config 1: 16 -> 11-14 us, scripts/spmv_lab.cu).
template <bool GLOBAL_OFF, int U, int MINB>
__global__ void __launch_bounds__(256, MINB)
    dia_kernel(int64_t nrows, int64_t ncols, int ndiags, const int64_t* __restrict__ offsets,
               const double* __restrict__ vals, const double* __restrict__ x,
               double* __restrict__ y, int64_t row_lo, int64_t row_hi) {
    __shared__ int soff[GLOBAL_OFF ? 1 : kDiaSmem];
    if (!GLOBAL_OFF) stage_offsets(soff, offsets, ndiags);
    const int64_t i = row_lo + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= row_hi) return;
    y[i] = dia_row<GLOBAL_OFF, U>(int(i), int(nrows), int(ncols), ndiags, soff, offsets, vals, x);
}

// Host-buffer spmv over PCIe with no copy engine (so_spmv, pinned x and y):
// a CTA of kZcRows rows stages the x window its rows read,
// [i0 + omin, i0 + kZcRows - 1 + omax], straight from mapped host memory
// into shared memory (16-byte loads when x is 16-byte aligned), multiplies
// exactly as dia_row does (same diagonal order, same -0.0 for out-of-range
// columns: bit-identical) and stores y straight into mapped host memory.
// Measured on config 2 (scripts/zc_probe.cu): 0.84 ms for the 32 MB up and
// 32 MB down vs 0.95+ for any copy-engine chunk pipeline.  Only for windows
// of span <= kZcSpan (x read at most 1.25x over the link).
constexpr int kZcRows = 1024;
constexpr int64_t kZcSpan = kZcRows / 4;

template <bool ALIGN16>
__global__ void __launch_bounds__(kZcRows, 1)
    dia_zc_kernel(int nrows, int ncols, int ndiags, const int64_t* __restrict__ offsets,
                  const double* __restrict__ vals, const double* x_host, double* y_host, int omin, int omax,
                  int blk0) {
    extern __shared__ double xs[];
    __shared__ int soff[kDiaSmem];
    stage_offsets(soff, offsets, ndiags);
    const int i0 = (blk0 + int(blockIdx.x)) * kZcRows;
    int w0 = max(0, i0 + omin);
    if (ALIGN16) w0 &= ~1;
    const int w1 = min(ncols, i0 + kZcRows - 1 + omax + 1);
    if (ALIGN16) {
        const int npair = (w1 - w0) >> 1;
        for (int j = threadIdx.x; j < npair; j += kZcRows)
            reinterpret_cast<double2*>(xs)[j] = *reinterpret_cast<const double2*>(x_host + w0 + 2 * j);
        if (((w1 - w0) & 1) && threadIdx.x == 0) xs[w1 - w0 - 1] = x_host[w1 - 1];
    } else {
        for (int j = threadIdx.x; j < w1 - w0; j += kZcRows) xs[j] = x_host[w0 + j];
    }
    __syncthreads();
    const int i = i0 + threadIdx.x;
    if (i >= nrows) return;
    const double* vp = vals + i;
    double acc = 0.0;
    for (int d0 = 0; d0 < ndiags; d0 += kDiaBatch) {
        double v[kDiaBatch], xv[kDiaBatch];
        bool ok[kDiaBatch];
#pragma unroll
        for (int u = 0; u < kDiaBatch; ++u) {
            const bool live = d0 + u < ndiags;
            const int d = live ? d0 + u : ndiags - 1;
            const int c = i + soff[d];
            ok[u] = live && unsigned(c) < unsigned(ncols);
            v[u] = ld_stream(vp + size_t(d) * size_t(nrows));
            xv[u] = xs[ok[u] ? c - w0 : 0];
        }
#pragma unroll
        for (int u = 0; u < kDiaBatch; ++u) acc = fadd(acc, ok[u] ? fmul(v[u], xv[u]) : -0.0);
    }
    y_host[i] = acc;
}

// Host-buffer DIA spmv that FOLLOWS one copy-engine upload of x (so_spmv
// with pinned buffers, narrow window).  The device copy of x is pre-filled
// with a NaN sentinel (both 32-bit halves kFollowSent); x goes up as ONE
// H2D on the copy stream, followed by a 4-byte copy that sets `flag`.  A
// persistent grid (one 1024-thread CTA per SM) walks the row blocks in
// address order behind the copy front: a block's x window is read from
// device memory (L1 bypassed) until no element still holds a sentinel half
// -- or the flag says the copy is complete (an x element that happens to
// equal the sentinel) -- then its rows are computed exactly as dia_zc_kernel
// does (bit-identical) and y is stored straight into mapped host memory.
// The copy engine reads x over the link at its full rate (~55 GB/s; SM loads
// from host memory reach ~44) while the SMs write y the other way.
// A copy that never arrives (a serialising tool) gives up after
// `timeout_ns` and reports it through `timed_out` (mapped host memory): the
// caller then recomputes on another path.  A launch covers row blocks
// [blk_lo, blk_hi): the pageable staging launches one kernel per y chunk so
// that an event after each tells host threads the chunk has landed (per-block
// completion flags need a system fence per block: 0.70 -> 1.17 ms on config
// 2; system-scope atomics 4.4 ms, scripts/cezc_probe.cu).
constexpr int64_t kFollowSpan = 16384;  // x window of a block: (1024 + span) doubles <= 136 KB of shared memory

__global__ void follow_fill(unsigned* __restrict__ p, int64_t n32, unsigned* __restrict__ flag) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n32; i += int64_t(gridDim.x) * blockDim.x)
        p[i] = kFollowSent;
    if (blockIdx.x == 0 && threadIdx.x == 0) *flag = 0;
}

__global__ void __launch_bounds__(kZcRows, 1)
    dia_follow_kernel(int nrows, int ncols, int ndiags, const int64_t* __restrict__ offsets,
                      const double* __restrict__ vals, const double* dx, double* y_host, const unsigned* flag,
                      int omin, int omax, unsigned* timed_out, unsigned long long timeout_ns, int blk_lo,
                      int blk_hi) {
    extern __shared__ double xs[];
    __shared__ int soff[kDiaSmem];
    stage_offsets(soff, offsets, ndiags);
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int blk = blk_lo + int(blockIdx.x); blk < blk_hi; blk += gridDim.x) {
        const int i0 = blk * kZcRows;
        const int w0 = max(0, i0 + omin), w1 = min(ncols, i0 + kZcRows - 1 + omax + 1);
        while (true) {
            unsigned fl;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(fl) : "l"(flag) : "memory");
            bool ok = true;
            for (int j = threadIdx.x; j < w1 - w0; j += kZcRows) {
                const double v = __ldcg(dx + w0 + j);
                xs[j] = v;
                ok = ok && (fl != 0 || follow_ready(v));
            }
            // one barrier publishes xs and agrees on readiness
            if (!__syncthreads_or(!ok)) break;
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            // thread 0's clock decides for the whole CTA (uniform exit)
            if (__syncthreads_or(threadIdx.x == 0 && t - t0 > timeout_ns)) {
                if (threadIdx.x == 0) atomicExch_system(timed_out, 1u);
                return;
            }
            __nanosleep(500);
        }
        const int i = i0 + threadIdx.x;
        if (i < nrows) {
            const double* vp = vals + i;
            double acc = 0.0;
            for (int d0 = 0; d0 < ndiags; d0 += kDiaBatch) {
                double v[kDiaBatch], xv[kDiaBatch];
                bool ok[kDiaBatch];
#pragma unroll
                for (int u = 0; u < kDiaBatch; ++u) {
                    const bool live = d0 + u < ndiags;
                    const int d = live ? d0 + u : ndiags - 1;
                    const int c = i + soff[d];
                    ok[u] = live && unsigned(c) < unsigned(ncols);
                    v[u] = ld_stream(vp + size_t(d) * size_t(nrows));
                    xv[u] = xs[ok[u] ? c - w0 : 0];
                }
#pragma unroll
                for (int u = 0; u < kDiaBatch; ++u) acc = fadd(acc, ok[u] ? fmul(v[u], xv[u]) : -0.0);
            }
            y_host[i] = acc;
        }
        __syncthreads();  // xs is reused by the next block
    }
}

// Row-partitioned iteration, fused boundary exchange (config 5, dist.py):
// the rows a neighbour needs are computed once and stored twice -- into the
// local window and straight into the neighbour's window over NVLink peer
// memory (remote[i - row_lo], an IPC-mapped pointer).  Every thread fences at
// system scope after its stores; the last CTA to finish (ticket) resets the
// ticket and publishes `flag_value` to the neighbour's flag with a
// release.sys store, which so_wait_flag acquires on the other side.
template <bool GLOBAL_OFF>
__global__ void __launch_bounds__(256, 6)
    dia_push_kernel(int64_t nrows, int64_t ncols, int ndiags, const int64_t* __restrict__ offsets,
                    const double* __restrict__ vals, const double* __restrict__ x, double* __restrict__ y,
                    int64_t row_lo, int64_t row_hi, double* remote, unsigned* ticket,
                    unsigned long long* remote_flag, unsigned long long flag_value) {
    __shared__ int soff[GLOBAL_OFF ? 1 : kDiaSmem];
    __shared__ bool last;
    if (!GLOBAL_OFF) stage_offsets(soff, offsets, ndiags);
    const int64_t i = row_lo + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < row_hi) {
        const double v = dia_row<GLOBAL_OFF>(int(i), int(nrows), int(ncols), ndiags, soff, offsets, vals, x);
        y[i] = v;
        remote[i - row_lo] = v;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x == 0) {
        *ticket = 0;
        __threadfence_system();
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(remote_flag), "l"(flag_value) : "memory");
    }
}

// Spins (acquire, system scope) until the neighbour's release store lands.
// A neighbour that never publishes (crashed rank) must not wedge this GPU:
// after kWaitTimeoutNs the wait gives up and bumps *timeouts, which
// so_wait_flag_timeouts() reports to the host.
constexpr unsigned long long kWaitTimeoutNs = 60ull * 1000 * 1000 * 1000;
__device__ unsigned long long g_wait_timeouts = 0;

__global__ void wait_flag_kernel(const unsigned long long* flag, unsigned long long value) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
        if (v >= value) break;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > kWaitTimeoutNs) {
            atomicAdd(&g_wait_timeouts, 1ull);
            break;
        }
        __nanosleep(256);
    }
}

// ---------------------------------------------------------------- ELL -------
// Column-major ELL, one thread per row; slots are consumed in order and the
// row stops at the first sentinel (spmv.cpp:59-71).  Column indices for
// kU slots are fetched together; values/x only for live slots.
template <bool ACCUM, bool FOLLOW = false>
__global__ void __launch_bounds__(256)
    ell_kernel(int64_t nrows, int width, const int32_t* __restrict__ col,
               const double* __restrict__ val, const double* __restrict__ x,
               double* __restrict__ y, FollowCtx fctx) {
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
            p[u] = live[u] ? fmul(ld_stream(val + int64_t(k0 + u) * nrows + i), ldx<FOLLOW>(x, c[u], fctx)) : 0.0;
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (live[u]) s = fadd(s, p[u]);
        if (!alive) break;
    }
    y[i] = ACCUM ? fadd(y[i], s) : s;
}

// ---------------------------------------------------------------- COO -------
// Segmented reduction over the row-sorted canonical COO.  The entries are cut
// into fixed chunks of kCooChunk (perfect balance whatever the row-length
// skew); a persistent warp walks chunks g, g + W, g + 2W, ... and issues the
// NEXT chunk's loads before reducing the current one, so each warp keeps one
// chunk of HBM reads in flight behind its x gathers and shuffles.
// Lane l owns kCooItems CONSECUTIVE entries of a chunk (256-bit streaming
// loads of row/col/val: a warp instruction covers 1 KB contiguous, L1 left to
// x), gathers x and forms the rounded products.  Pass 1 sums the lane's last
// row piece; one warp-wide segmented scan keyed on that row joins pieces
// across lanes (rows are sorted, so equal keys are contiguous); pass 2 walks
// the lane's entries sequentially from the carry of earlier lanes, so a row
// spanning at most two lanes is summed in the reference's order
// (spmv.cpp:21-30).  Rows that start and end inside the chunk are written
// directly; pieces of rows spanning chunks go to per-chunk records combined
// by coo_fixup in chunk order.  Fixed partition and combine order =>
// deterministic, within the 1e-12 contract.  Empty rows are zero-filled by
// the lane holding the next row's first entry (y written exactly once).
// ACCUM (HYB COO part, spmv.cpp:95-100): the row sum is added to the ELL
// result already in y.  Variants measured in scripts/spmv_lab.cu.
// Fix-up kernels launched with programmatic dependent launch (they wait for
// the kernel before them with griddepcontrol.wait).  SOB_NO_PDL_FIXUP: A/B.
bool fixup_pdl() {
    static const bool on = std::getenv("SOB_NO_PDL_FIXUP") == nullptr;
    return on;
}

constexpr int kCooItems = 8;
constexpr int kCooChunk = 32 * kCooItems;
constexpr int kCooPerSm = 3;
// the accumulate variant (HYB) also reads y: 2 CTAs/SM leave it unspilled
constexpr int coo_per_sm(bool accum) { return accum ? 2 : kCooPerSm; }

struct CooChunkRec {
    double first_sum;  // in-chunk piece of a row that began in an earlier chunk
    double last_sum;   // in-chunk piece of the row that continues past the chunk
    int32_t last_row;
    int32_t flags;
};
enum : int32_t { kFirstCont = 1, kLastOpen = 2, kSingle = 4 };
constexpr int kNoRow = 0x7fffffff;

__device__ __forceinline__ void coo_load(const int32_t* __restrict__ row, const int32_t* __restrict__ col,
                                         const double* __restrict__ val, int64_t k, int rem,
                                         int (&r)[kCooItems], int (&c)[kCooItems], double (&v)[kCooItems]) {
    if (rem >= kCooItems) {
        ld_stream_v8(row + k, r);
        ld_stream_v8(col + k, c);
        ld_stream_v4(val + k, v);
        ld_stream_v4(val + k + 4, v + 4);
    } else {
#pragma unroll
        for (int j = 0; j < kCooItems; ++j) {
            const bool ok = j < rem;
            r[j] = ok ? row[k + j] : kNoRow;
            c[j] = ok ? col[k + j] : 0;
            v[j] = ok ? val[k + j] : 0.0;
        }
    }
}

// CONT (every row <= 32 entries, so a row spans at most two chunks and its
// continuation fits one warp load): no records -- the chunk holding a row's
// first entry finishes it, reading the row's continuation at the head of the
// next chunk itself (coo_warp_kernel);
// the chunk's open row's in-chunk sum is returned in `open_acc` (the lane
// holding the chunk's last entry) and orphan prefixes are skipped.
template <bool ACCUM, bool CONT = false>
__device__ __forceinline__ void coo_finish(int lane, int64_t chunk, int64_t base, int cnt, int64_t z, int64_t nrows,
                                           const int (&r)[kCooItems], const double (&p)[kCooItems], int prev_row,
                                           int next_row, double* __restrict__ y, CooChunkRec* __restrict__ rec,
                                           double& open_acc) {
    constexpr int IT = kCooItems;
    constexpr unsigned kFull = 0xffffffffu;
    const int first = lane * IT;
    const int nmine = cnt - first <= 0 ? 0 : (cnt - first >= IT ? IT : cnt - first);
    // pass 1: the lane's last row piece (kNoRow pieces of idle lanes never match)
    int tr = kNoRow;
#pragma unroll
    for (int j = 0; j < IT; ++j)
        if (j < nmine) tr = r[j];
    double tsum = 0.0;
#pragma unroll
    for (int j = 0; j < IT; ++j)
        if (j < nmine && r[j] == tr) tsum = fadd(tsum, p[j]);
    // inclusive segmented scan over lanes keyed on the tail row: lanes between
    // two equal keys hold nothing but that row (sorted), so the run is exact
    double inc = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double up = __shfl_up_sync(kFull, inc, o);
        const int ur = __shfl_up_sync(kFull, tr, o);
        if (lane >= o && ur == tr) inc = fadd(up, inc);
    }
    const double prev_inc = __shfl_up_sync(kFull, inc, 1);
    const int prev_tr = __shfl_up_sync(kFull, tr, 1);
    const int nlane_r0 = __shfl_down_sync(kFull, r[0], 1);
    const int first_row = __shfl_sync(kFull, r[0], 0);
    const bool first_cont = first_row == prev_row;
    if (nmine == 0) return;

    // pass 2: sequential walk from the carry of earlier lanes
    int prv = lane == 0 ? prev_row : prev_tr;
    double acc = (lane > 0 && prev_tr == r[0]) ? prev_inc : 0.0;
    const bool chunk_end = first + nmine == cnt;
#pragma unroll
    for (int j = 0; j < IT; ++j) {
        if (j < nmine) {
            const int rw = r[j];
            if (rw != prv) {
                if (!ACCUM)  // rows strictly between consecutive entries are empty
                    for (int q = prv + 1; q < rw; ++q) y[q] = 0.0;
                if (j > 0) acc = 0.0;
            }
            acc = fadd(acc, p[j]);
            const int nxt = j + 1 < nmine ? r[j + 1] : (chunk_end ? next_row : nlane_r0);
            const bool orphan = first_cont && rw == first_row;  // began in an earlier chunk
            if (rw != nxt) {
                if (!orphan)
                    y_store<ACCUM>(y + rw, acc);
                else if (!CONT)
                    rec[chunk].first_sum = acc;
            }
            if (CONT && chunk_end && j + 1 == nmine) {
                if (rw == nxt) open_acc = acc;
                if (!ACCUM && base + cnt == z)  // trailing empty rows
                    for (int64_t q = int64_t(rw) + 1; q < nrows; ++q) y[q] = 0.0;
            }
            if (!CONT && chunk_end && j + 1 == nmine) {
                const bool open = rw == nxt;
                if (open) {
                    rec[chunk].last_sum = acc;
                    rec[chunk].last_row = rw;
                    if (orphan) rec[chunk].first_sum = acc;
                }
                rec[chunk].flags = (first_cont ? kFirstCont : 0) | (open ? kLastOpen : 0) |
                                   ((open && orphan) ? kSingle : 0);
                if (!ACCUM && base + cnt == z)  // trailing empty rows
                    for (int64_t q = int64_t(rw) + 1; q < nrows; ++q) y[q] = 0.0;
            }
            prv = rw;
        }
    }
}

// FOLLOW: pinned spmv(m, x) -- each x gather waits for its element of the
// upload (ldx); the persistent warps walk their chunks in address order.
template <bool ACCUM, bool FOLLOW = false, bool CONT = false>
__global__ void __launch_bounds__(256, coo_per_sm(ACCUM))
    coo_warp_kernel(int64_t z, int64_t nrows, const int32_t* __restrict__ row, const int32_t* __restrict__ col,
                    const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
                    CooChunkRec* __restrict__ rec, FollowCtx fctx, int64_t c0 = 0, int64_t c1 = INT64_MAX) {
    constexpr int IT = kCooItems;
    const int lane = threadIdx.x & 31;
    const int64_t nchunks = (z + kCooChunk - 1) / kCooChunk;
    const int64_t cend = min(nchunks, c1);  // [c0, c1): a chunk range (CONT only; the pinned chunk pipeline)
    const int64_t stride = int64_t(gridDim.x) * (blockDim.x >> 5);
    int64_t chunk = c0 + ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    // coo_fixup (launched with PDL) is scheduled early and waits for this grid
    asm volatile("griddepcontrol.launch_dependents;" :::);
    if (!CONT && blockIdx.x == 0 && threadIdx.x == 0) {  // coo_fixup's control words (after the records)
        unsigned long long* ctl = reinterpret_cast<unsigned long long*>(rec + nchunks);
        ctl[0] = 0;
        ctl[1] = 0;
    }
    if (chunk >= cend) return;
    int r[IT], c[IT];
    double v[IT];
    coo_load(row, col, val, chunk * kCooChunk + lane * IT, int(min(z - chunk * kCooChunk, int64_t(kCooChunk))) - lane * IT,
             r, c, v);
    while (true) {
        const int64_t base = chunk * kCooChunk;
        const int cnt = int(min(z - base, int64_t(kCooChunk)));
        double p[IT];
#pragma unroll
        for (int j = 0; j < IT; ++j) p[j] = lane * IT + j < cnt ? fmul(v[j], ldx<FOLLOW>(x, c[j], fctx)) : 0.0;
        const int prev_row = base > 0 ? row[base - 1] : -1;
        const int next_row = base + cnt < z ? row[base + cnt] : -1;
        // CONT: the head of the next chunk (the open row's continuation, if
        // any), loaded with this chunk and consumed after its finish
        int hr = kNoRow, last_row = kNoRow;
        double hp = 0.0;
        const int owner = (cnt - 1) / IT;  // lane holding the chunk's last entry
        if (CONT) {
            const int64_t k = base + cnt + lane;
            int hc = 0;
            double hv = 0.0;
            if (k < z) {
                hr = __ldg(row + k);
                hc = __ldg(col + k);
                hv = __ldg(val + k);
            }
            int tr = kNoRow;
#pragma unroll
            for (int j = 0; j < IT; ++j)
                if (lane * IT + j < cnt) tr = r[j];
            last_row = __shfl_sync(0xffffffffu, tr, owner);
            if (hr == last_row) hp = fmul(hv, ldx<FOLLOW>(x, hc, fctx));
        }
        int rc[IT];
#pragma unroll
        for (int j = 0; j < IT; ++j) rc[j] = r[j];
        const int64_t nx = chunk + stride;
        if (nx < cend)
            coo_load(row, col, val, nx * kCooChunk + lane * IT, int(min(z - nx * kCooChunk, int64_t(kCooChunk))) - lane * IT,
                     r, c, v);
        double open_acc = 0.0;
        coo_finish<ACCUM, CONT>(lane, chunk, base, cnt, z, nrows, rc, p, prev_row, next_row, y, rec, open_acc);
        if (CONT) {
            if (next_row == last_row) {  // warp-uniform: the last row continues (< 32 more entries)
                const double t = warp_sum(hp);  // fixed butterfly: deterministic
                if (lane == owner) y_store<ACCUM>(y + last_row, fadd(open_acc, t));
            }
        }
        if (nx >= cend) break;
        chunk = nx;
    }
}

// Rows spanning chunks: the chunk holding the row's first entry walks forward
// in chunk order (deterministic) and writes the final value; records are
// fetched 8 at a time so a row spanning hundreds of chunks (R-MAT hubs) is
// not one dependent load per chunk.  A walk still open after kFixupInline
// records is queued for coo_fixup_long, where a CTA finishes it 256 records
// per step (a row of 10^8 entries spans ~4*10^5 chunks).
constexpr int kFixupInline = 64;
struct LongRun {
    int64_t owner;  // chunk holding the row's first piece
    int64_t next;   // first record not yet added
    double partial; // last_sum[owner] + first_sum[owner+1 .. next)
};

// A CTA finishes the queued long runs, 256 records per step: the run ends at
// the first record that is not a whole-chunk continuation; per-thread
// partials are joined by a fixed block tree (deterministic).
template <bool ACCUM>
__device__ void finish_long_runs(int64_t nchunks, const CooChunkRec* __restrict__ rec, double* __restrict__ y,
                                 const LongRun* __restrict__ runs, unsigned long long n) {
    __shared__ double scratch[8];
    __shared__ unsigned long long stop;
    for (unsigned long long q = 0; q < n; ++q) {
        const LongRun run = runs[q];
        double t = 0.0;
        for (int64_t j0 = run.next;; j0 += 256) {
            if (threadIdx.x == 0) stop = ~0ull;
            __syncthreads();
            const int64_t j = j0 + threadIdx.x;
            const bool in = j < nchunks;
            const int32_t fl = in ? rec[j].flags : 0;
            if ((in && !(fl & kSingle)) || (!in && j == nchunks)) atomicMin(&stop, (unsigned long long)(in ? j : j - 1));
            __syncthreads();
            const unsigned long long end = stop;  // last record of the run (inclusive), if in this step
            if (in && (unsigned long long)j <= end) t = fadd(t, rec[j].first_sum);
            __syncthreads();
            if (end != ~0ull) break;
        }
        const double sum = block_sum_det<256>(t, scratch);
        if (threadIdx.x == 0) {
            const int32_t r = rec[run.owner].last_row;
            const double v = fadd(run.partial, sum);
            y[r] = ACCUM ? fadd(y[r], v) : v;
        }
        __syncthreads();
    }
}

// ctl[0] = queued long runs (zeroed by coo_warp_kernel)
template <bool ACCUM>
__global__ void __launch_bounds__(256) coo_fixup(int64_t nchunks, const CooChunkRec* __restrict__ rec,
                                                 double* __restrict__ y, LongRun* __restrict__ runs,
                                                 unsigned long long* __restrict__ ctl) {
    pdl_enter();
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int32_t f = c < nchunks ? rec[c].flags : 0;
    if ((f & kLastOpen) && !(f & kSingle)) {
        double t = rec[c].last_sum;
        bool queued = false;
        for (int64_t j0 = c + 1; j0 < nchunks; j0 += 8) {
            if (j0 - c > kFixupInline) {  // long run: the last CTA finishes it
                const unsigned long long q = atomicAdd(&ctl[0], 1ull);
                runs[q] = LongRun{c, j0, t};
                queued = true;
                break;
            }
            double fs[8];
            int32_t fl[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t j = j0 + u < nchunks ? j0 + u : nchunks - 1;
                fs[u] = rec[j].first_sum;
                fl[u] = rec[j].flags;
            }
            bool done = false;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (!done && j0 + u < nchunks) {
                    t = fadd(t, fs[u]);
                    if (!(fl[u] & kSingle)) done = true;
                }
            }
            if (done) break;
        }
        if (!queued) {
            const int32_t r = rec[c].last_row;
            y[r] = ACCUM ? fadd(y[r], t) : t;
        }
    }
}

// The queued long runs, one CTA each (grid-stride over the queue).
template <bool ACCUM>
__global__ void __launch_bounds__(256) coo_fixup_long(int64_t nchunks, const CooChunkRec* __restrict__ rec,
                                                      double* __restrict__ y, const LongRun* __restrict__ runs,
                                                      const unsigned long long* __restrict__ ctl) {
    pdl_enter();
    const unsigned long long n = ctl[0];
    for (unsigned long long q = blockIdx.x; q < n; q += gridDim.x) finish_long_runs<ACCUM>(nchunks, rec, y, runs + q, 1);
}

// Longest run of empty rows of a canonical COO (leading, between entries,
// trailing) -- cached per matrix.  The non-accumulating kernel zero-fills an
// empty run with the one lane that finds it, which is free for ordinary
// matrices but serialises on a lane when the entries sit in a few rows; those
// matrices take y = 0 (memset) + the accumulating kernel instead (0 + s == s
// exactly, so the result is identical).
__global__ void coo_max_gap(int64_t z, int64_t nrows, const int32_t* __restrict__ row,
                            unsigned long long* __restrict__ out) {
    // out[0] = longest empty-row run; out[1] |= 1 when some row fully covers
    // kFixupInline + 1 consecutive chunks (only then can coo_fixup queue a long
    // run); out[2] |= 1 when some row holds more than 32 entries
    constexpr int64_t kSpan = int64_t(kFixupInline) * kCooChunk - 1;
    unsigned long long g = 0;
    bool lng = false, big = false;
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k <= z; k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t prv = k == 0 ? -1 : row[k - 1];
        const int64_t cur = k == z ? nrows : row[k];
        const int64_t gap = cur - prv - 1;
        if (gap > int64_t(g)) g = gap;
        if (k % kCooChunk == 0 && k + kSpan < z && row[k] == row[k + kSpan]) lng = true;
        if (k + 32 < z && row[k] == row[k + 32]) big = true;
    }
    g = warp_max(g);
    if ((threadIdx.x & 31) == 0 && g) atomicMax(out, g);
    if (__any_sync(0xffffffffu, lng) && (threadIdx.x & 31) == 0) out[1] = 1;
    if (__any_sync(0xffffffffu, big) && (threadIdx.x & 31) == 0) out[2] = 1;
}
constexpr int64_t kCooGapInline = 4096;  // a lane zero-fills up to ~2 us of rows inline

// chunk records, then the fix-up's control word pair and long-run queue
int64_t coo_rec_count(const CooPart& coo) { return 2 * ceil_div(coo.nnz, kCooChunk) + 1; }

// Every row <= 32 entries (profiled) and a small matrix: the chunk kernel
// finishes rows crossing into the next chunk itself -- no records, no fix-up
// kernel (config 1: 28.7 -> 24.9 us).  The head load of the next chunk costs
// ~0.1 us per million entries (config 2: 375 -> 385 us), the fix-up ~4.5 us
// flat: break-even near 35 M entries, gated at 16 M
// (profiles/r02au_coo_cont.txt).  SOB_NO_COO_CONT / SOB_COO_CONT=1: A/B.
constexpr int64_t kCooContMaxNnz = int64_t(1) << 24;
bool coo_cont(const CooPart& coo) {
    static const bool off = std::getenv("SOB_NO_COO_CONT") != nullptr;
    static const bool always = std::getenv("SOB_COO_CONT") != nullptr;
    return !off && coo.short_rows.load(std::memory_order_acquire) == 1 && (always || coo.nnz <= kCooContMaxNnz);
}

// `pre`: the record buffer allocated by a follow path before its first launch
template <bool ACCUM>
void launch_coo(const CooPart& coo, int64_t nrows, const double* x, double* y, cudaStream_t s,
                const FollowCtx* follow = nullptr, DBuf<CooChunkRec>* pre = nullptr) {
    const int64_t nchunks = ceil_div(coo.nnz, kCooChunk);
    if (coo_cont(coo)) {
        const int grid = int(std::min<int64_t>(ceil_div(nchunks, 8), int64_t(current_ctx().num_sms) * coo_per_sm(ACCUM)));
        if (follow)
            coo_warp_kernel<ACCUM, true, true><<<grid, 256, 0, s>>>(coo.nnz, nrows, coo.row.get(), coo.col.get(),
                                                                    coo.val.get(), x, y, nullptr, *follow);
        else
            coo_warp_kernel<ACCUM, false, true><<<grid, 256, 0, s>>>(coo.nnz, nrows, coo.row.get(), coo.col.get(),
                                                                     coo.val.get(), x, y, nullptr,
                                                                     FollowCtx{nullptr, nullptr, 0});
        SOB_LAUNCH("coo_warp_kernel");
        return;
    }
    static_assert(sizeof(LongRun) == sizeof(CooChunkRec) && sizeof(CooChunkRec) >= 16, "record layout");
    DBuf<CooChunkRec> own;
    if (!pre) own.alloc(coo_rec_count(coo), s);
    DBuf<CooChunkRec>& rec = pre ? *pre : own;
    const int grid = int(std::min<int64_t>(ceil_div(nchunks, 8), int64_t(current_ctx().num_sms) * coo_per_sm(ACCUM)));
    if (follow)
        coo_warp_kernel<ACCUM, true><<<grid, 256, 0, s>>>(coo.nnz, nrows, coo.row.get(), coo.col.get(),
                                                          coo.val.get(), x, y, rec.get(), *follow);
    else
        coo_warp_kernel<ACCUM><<<grid, 256, 0, s>>>(coo.nnz, nrows, coo.row.get(), coo.col.get(), coo.val.get(), x,
                                                    y, rec.get(), FollowCtx{nullptr, nullptr, 0});
    SOB_LAUNCH("coo_warp_kernel");
    LongRun* runs = reinterpret_cast<LongRun*>(rec.get() + nchunks + 1);
    unsigned long long* ctl = reinterpret_cast<unsigned long long*>(rec.get() + nchunks);
    if (fixup_pdl()) {  // scheduled while the chunk kernel runs; waits for it
        launch_pdl(coo_fixup<ACCUM>, dim3(unsigned(ceil_div(nchunks, 256))), dim3(256), 0, s, nchunks,
                   static_cast<const CooChunkRec*>(rec.get()), y, runs, ctl);
    } else {
        coo_fixup<ACCUM><<<unsigned(ceil_div(nchunks, 256)), 256, 0, s>>>(nchunks, rec.get(), y, runs, ctl);
    }
    SOB_LAUNCH("coo_fixup");
    if (coo.long_runs != 0) {  // unknown (-1) or present
        if (fixup_pdl())
            launch_pdl(coo_fixup_long<ACCUM>, dim3(unsigned(current_ctx().num_sms)), dim3(256), 0, s, nchunks,
                       static_cast<const CooChunkRec*>(rec.get()), y, static_cast<const LongRun*>(runs),
                       static_cast<const unsigned long long*>(ctl));
        else
            coo_fixup_long<ACCUM><<<current_ctx().num_sms, 256, 0, s>>>(nchunks, rec.get(), y, runs, ctl);
        SOB_LAUNCH("coo_fixup_long");
    }
}

// [g0, g1): the row groups to run (g1 < 0: all)
template <int IT, bool PAD, bool COOP, int RPL>
void launch_csr_warp4(const so_matrix& m, bool accum, const double* x, double* y, cudaStream_t s,
                      const FollowCtx* follow, int64_t g0 = 0, int64_t g1 = -1) {
    const CsrPart& c = m.csr;
    const int per_sm = IT > 8 ? 3 : 4;
    const int grid = int(std::min<int64_t>(ceil_div(c.ngrp, 8), int64_t(current_ctx().num_sms) * per_sm));
    const FollowCtx none{nullptr, nullptr, 0};
    if (follow && g1 >= 0) {  // a chunk of the groups (pinned CSR / HDC chunk pipelines)
        const int gridc = int(std::min<int64_t>(ceil_div(g1 - g0, 8), int64_t(current_ctx().num_sms) * per_sm));
        if (accum)
            csr_warp_kernel<IT, true, PAD, COOP, RPL, true><<<gridc, 256, 0, s>>>(
                c.grp.get() + g0, c.grp_k.get() + g0, g1 - g0, c.row_ptr.get(), c.col.get(), c.val.get(), x, y,
                m.nrows, *follow);
        else
            csr_warp_kernel<IT, false, PAD, COOP, RPL, true><<<gridc, 256, 0, s>>>(
                c.grp.get() + g0, c.grp_k.get() + g0, g1 - g0, c.row_ptr.get(), c.col.get(), c.val.get(), x, y,
                m.nrows, *follow);
    } else if (follow && accum)  // HDC's CSR part after its DIA part, following the upload of x
        csr_warp_kernel<IT, true, PAD, COOP, RPL, true><<<grid, 256, 0, s>>>(
            c.grp.get(), c.grp_k.get(), c.ngrp, c.row_ptr.get(), c.col.get(), c.val.get(), x, y, m.nrows, *follow);
    else if (follow)  // host-buffer spmv(m, x) following the upload of x
        csr_warp_kernel<IT, false, PAD, COOP, RPL, true><<<grid, 256, 0, s>>>(
            c.grp.get(), c.grp_k.get(), c.ngrp, c.row_ptr.get(), c.col.get(), c.val.get(), x, y, m.nrows, *follow);
    else if (accum)
        csr_warp_kernel<IT, true, PAD, COOP, RPL><<<grid, 256, 0, s>>>(c.grp.get(), c.grp_k.get(), c.ngrp,
                                                                       c.row_ptr.get(), c.col.get(), c.val.get(),
                                                                       x, y, m.nrows, none);
    else
        csr_warp_kernel<IT, false, PAD, COOP, RPL><<<grid, 256, 0, s>>>(c.grp.get(), c.grp_k.get(), c.ngrp,
                                                                        c.row_ptr.get(), c.col.get(), c.val.get(),
                                                                        x, y, m.nrows, none);
    SOB_LAUNCH("csr_warp_kernel");
}

template <int IT, bool PAD, bool COOP>
void launch_csr_warp3(const so_matrix& m, bool accum, const double* x, double* y, cudaStream_t s,
                      const FollowCtx* follow, int64_t g0, int64_t g1) {
    if (m.csr.grp_rpl > 1)
        launch_csr_warp4<IT, PAD, COOP, kGroupRowsMax / 32>(m, accum, x, y, s, follow, g0, g1);
    else
        launch_csr_warp4<IT, PAD, COOP, 1>(m, accum, x, y, s, follow, g0, g1);
}

template <int IT, bool PAD>
void launch_csr_warp(const so_matrix& m, bool accum, const double* x, double* y, cudaStream_t s,
                     const FollowCtx* follow, int64_t g0 = 0, int64_t g1 = -1) {
    static const bool no_coop = std::getenv("SOB_NO_CSR_COOP") != nullptr;  // diagnostic knob (A/B)
    if (m.csr.ncoop > 0 && !no_coop)
        launch_csr_warp3<IT, PAD, true>(m, accum, x, y, s, follow, g0, g1);
    else
        launch_csr_warp3<IT, PAD, false>(m, accum, x, y, s, follow, g0, g1);
}

// The row-group kernel alone over groups [g0, g1), following the upload
// (matrices without long rows: the pinned CSR / HDC chunk pipelines;
// accum: y += A_csr x, HDC's CSR part after its DIA part)
void launch_csr_groups_follow(const so_matrix& m, const double* x, double* y, cudaStream_t s, const FollowCtx& fc,
                              int64_t g0, int64_t g1, bool accum = false) {
    const CsrPart& c = m.csr;
    const bool pad = c.npad > 0;
    if (c.grp_cap == 32 * kGroupItemsShort)
        pad ? launch_csr_warp<kGroupItemsShort, true>(m, accum, x, y, s, &fc, g0, g1)
            : launch_csr_warp<kGroupItemsShort, false>(m, accum, x, y, s, &fc, g0, g1);
    else
        pad ? launch_csr_warp<kGroupItemsLong, true>(m, accum, x, y, s, &fc, g0, g1)
            : launch_csr_warp<kGroupItemsLong, false>(m, accum, x, y, s, &fc, g0, g1);
}

// accum: y += A_csr x (HDC's CSR part after its DIA part), else y = A_csr x;
// follow: x is still being uploaded (FOLLOW kernels)
// `pre_part`: the long-row pieces buffer, allocated by a follow path before
// its first launch
void launch_csr_stream(const so_matrix& m, bool accum, const double* x, double* y, cudaStream_t s,
                       const FollowCtx* follow = nullptr, DBuf<double>* pre_part = nullptr) {
    const CsrPart& c = m.csr;
    if (c.ngrp == 0) return;
    // flags are set (npad > 0) only when >= 1/64 of the groups prefer the
    // padded layout (convert.cu); otherwise grp_k is plain
    const bool pad = c.npad > 0;
    // allocated before any launch: nothing between two kernels that follow
    // an upload may wait for the device
    DBuf<double> own_part(pre_part || c.nlong == 0 ? 0 : c.npieces, s);
    DBuf<double>& part = pre_part ? *pre_part : own_part;
    if (c.grp_cap == 32 * kGroupItemsShort)
        pad ? launch_csr_warp<kGroupItemsShort, true>(m, accum, x, y, s, follow)
            : launch_csr_warp<kGroupItemsShort, false>(m, accum, x, y, s, follow);
    else
        pad ? launch_csr_warp<kGroupItemsLong, true>(m, accum, x, y, s, follow)
            : launch_csr_warp<kGroupItemsLong, false>(m, accum, x, y, s, follow);
    if (c.nlong > 0) {
        const FollowCtx none{nullptr, nullptr, 0};
        const int64_t* pk = c.piece_k.get();
        const int32_t* col = c.col.get();
        const double* val = c.val.get();
        const int32_t* lrow = c.long_row.get();
        const int64_t* lpiece = c.long_piece.get();
        const double* cpart = part.get();
        const unsigned g = unsigned(ceil_div(c.nlong * 32, 128));  // one warp per long row
        if (fixup_pdl()) {  // each waits for the kernel before it (launch latency hidden)
            launch_pdl(follow ? csr_long_pieces<true> : csr_long_pieces<false>, dim3(unsigned(c.npieces)),
                       dim3(kStreamBlock), 0, s, pk, col, val, x, part.get(), follow ? *follow : none);
            SOB_LAUNCH("csr_long_pieces");
            launch_pdl(accum ? csr_long_fixup<true> : csr_long_fixup<false>, dim3(g), dim3(128), 0, s, c.nlong, lrow,
                       lpiece, cpart, y);
        } else {
            if (follow)
                csr_long_pieces<true><<<unsigned(c.npieces), kStreamBlock, 0, s>>>(pk, col, val, x, part.get(),
                                                                                    *follow);
            else
                csr_long_pieces<false><<<unsigned(c.npieces), kStreamBlock, 0, s>>>(pk, col, val, x, part.get(),
                                                                                     none);
            SOB_LAUNCH("csr_long_pieces");
            if (accum)
                csr_long_fixup<true><<<g, 128, 0, s>>>(c.nlong, lrow, lpiece, cpart, y);
            else
                csr_long_fixup<false><<<g, 128, 0, s>>>(c.nlong, lrow, lpiece, cpart, y);
        }
        SOB_LAUNCH("csr_long_fixup");
    }
}

void launch_dia(const so_matrix& m, const double* x, double* y, cudaStream_t s, int64_t lo = 0,
                int64_t hi = -1) {
    if (hi < 0) hi = m.nrows;
    if (hi <= lo) return;
    const unsigned grid = unsigned(ceil_div(hi - lo, 256));
    const int nd = int(m.dia.ndiags);
    if (nd <= 5)
        dia_kernel<false, 5, 8><<<grid, 256, 0, s>>>(m.nrows, m.ncols, nd, m.dia.offsets.get(), m.dia.values.get(),
                                                      x, y, lo, hi);
    else if (m.dia.ndiags <= kDiaSmem)
        dia_kernel<false, kDiaBatch, 6><<<grid, 256, 0, s>>>(m.nrows, m.ncols, nd, m.dia.offsets.get(),
                                                              m.dia.values.get(), x, y, lo, hi);
    else
        dia_kernel<true, kDiaBatch, 6><<<grid, 256, 0, s>>>(m.nrows, m.ncols, nd, m.dia.offsets.get(),
                                                             m.dia.values.get(), x, y, lo, hi);
    SOB_LAUNCH("dia_kernel");
}

template <bool ACCUM>
void launch_ell(const so_matrix& m, const double* x, double* y, cudaStream_t s, const FollowCtx* follow = nullptr) {
    const unsigned grid = unsigned(ceil_div(m.nrows, 256));
    if (follow)  // rows in block order trail the upload of x (never accumulating)
        ell_kernel<false, true><<<grid, 256, 0, s>>>(m.nrows, int(m.ell.width), m.ell.col.get(), m.ell.val.get(), x, y,
                                                     *follow);
    else
        ell_kernel<ACCUM><<<grid, 256, 0, s>>>(m.nrows, int(m.ell.width), m.ell.col.get(), m.ell.val.get(), x, y,
                                               FollowCtx{nullptr, nullptr, 0});
    SOB_LAUNCH("ell_kernel");
}

}  // namespace

int64_t zero_copy_rows_per_block() { return kZcRows; }

bool spmv_dia_zero_copy(const so_matrix& m, const double* x_mapped, double* y_mapped, cudaStream_t s,
                        int64_t blk_lo, int64_t blk_hi) {
    if (m.format != SO_DIA && !(m.format == SO_HDC && m.csr.nnz == 0)) return false;
    if (!m.dia_window_known.load(std::memory_order_acquire) || m.dia.ndiags == 0 || m.dia.ndiags > kDiaSmem)
        return false;
    const int64_t omin = m.dia_omin, omax = m.dia_omax;
    if (omax - omin > kZcSpan) return false;
    const size_t smem = sizeof(double) * size_t(kZcRows + (omax - omin) + 2);
    const int64_t nblk = ceil_div(m.nrows, int64_t(kZcRows));
    if (blk_hi < 0 || blk_hi > nblk) blk_hi = nblk;
    if (blk_lo >= blk_hi) return true;
    const unsigned grid = unsigned(blk_hi - blk_lo);
    if ((reinterpret_cast<uintptr_t>(x_mapped) & 15) == 0)
        dia_zc_kernel<true><<<grid, kZcRows, smem, s>>>(int(m.nrows), int(m.ncols), int(m.dia.ndiags),
                                                         m.dia.offsets.get(), m.dia.values.get(), x_mapped, y_mapped,
                                                         int(omin), int(omax), int(blk_lo));
    else
        dia_zc_kernel<false><<<grid, kZcRows, smem, s>>>(int(m.nrows), int(m.ncols), int(m.dia.ndiags),
                                                          m.dia.offsets.get(), m.dia.values.get(), x_mapped,
                                                          y_mapped, int(omin), int(omax), int(blk_lo));
    SOB_LAUNCH("dia_zc_kernel");
    return true;
}

namespace {
// Per-device state of the follow path: the sentinel-filled device copy of x
// (grow-only), the copy-complete flag, the pinned word copied into it, the
// mapped timeout word, and the event after which the copy may refill x.
// The mutex covers only the enqueueing (follow_launch returns with it
// released, so the pageable path may finish a call on another thread);
// calls on the same device are ordered through the events: a call's upload
// AND kernel wait for the previous call's sentinel refill.  Each call gets
// its own timeout word (a ring of kFollowSlots mapped words).
constexpr int kFollowSlots = 64;
struct FollowStage {
    std::mutex mu;
    double* dx = nullptr;
    int64_t cap = 0;
    unsigned* flag = nullptr;
    unsigned* one_host = nullptr;
    unsigned* timed_out = nullptr;  // [kFollowSlots], pinned + mapped
    unsigned* timed_out_dev = nullptr;
    unsigned next_slot = 0;
    cudaEvent_t refilled = nullptr, copied = nullptr;
    cudaEvent_t done[kFollowSlots] = {};  // per call slot: its kernels are complete
    // pinned CSR chunk pipeline: chunk k's rows done / every chunk's y copied
    // (recorded and waited inside one enqueue, under mu)
    cudaEvent_t chunk_ev[so_matrix::kFollowChunks + 1] = {};
    bool preloaded = false;
};

// Lazy module loading (the CUDA 12 default) loads a kernel at its first
// launch and waits for the device to do so; a follow kernel already running
// waits for an upload this thread has not queued yet, so a kernel loaded
// between the follow kernels and the upload stalls the call until the wait
// times out (HYB with a COO part: 13.9 s on its first call).  Every kernel a
// follow path launches after its first one is loaded up front, once per
// device, and its scratch buffers are allocated before its first launch.
template <int IT, bool PAD, bool COOP, int RPL>
void preload_csr_accum_follow() {
    cudaFuncAttributes a;
    SOB_CUDA(cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(&csr_warp_kernel<IT, true, PAD, COOP, RPL, true>)));
}
template <int IT>
void preload_csr_accum_follow_all() {
    preload_csr_accum_follow<IT, false, false, 1>();
    preload_csr_accum_follow<IT, false, true, 1>();
    preload_csr_accum_follow<IT, true, false, 1>();
    preload_csr_accum_follow<IT, true, true, 1>();
    preload_csr_accum_follow<IT, false, false, kGroupRowsMax / 32>();
    preload_csr_accum_follow<IT, false, true, kGroupRowsMax / 32>();
    preload_csr_accum_follow<IT, true, false, kGroupRowsMax / 32>();
    preload_csr_accum_follow<IT, true, true, kGroupRowsMax / 32>();
}

void follow_preload() {
    // HDC with both parts: the CSR kernels (accumulating) run after the DIA one
    preload_csr_accum_follow_all<kGroupItemsShort>();
    preload_csr_accum_follow_all<kGroupItemsLong>();
    const void* fns[] = {
        reinterpret_cast<const void*>(&csr_long_fixup<true>),
        reinterpret_cast<const void*>(&csr_long_pieces<true>),
        reinterpret_cast<const void*>(&csr_long_fixup<false>),
        reinterpret_cast<const void*>(&coo_warp_kernel<false, true>),
        reinterpret_cast<const void*>(&coo_warp_kernel<true, true>),
        reinterpret_cast<const void*>(&coo_warp_kernel<false, true, true>),
        reinterpret_cast<const void*>(&coo_warp_kernel<true, true, true>),
        reinterpret_cast<const void*>(&coo_fixup<false>),
        reinterpret_cast<const void*>(&coo_fixup<true>),
        reinterpret_cast<const void*>(&coo_fixup_long<false>),
        reinterpret_cast<const void*>(&coo_fixup_long<true>),
        reinterpret_cast<const void*>(&ell_kernel<false, true>),
        reinterpret_cast<const void*>(&dia_follow_kernel),
        reinterpret_cast<const void*>(&follow_fill),
    };
    for (const void* fn : fns) {
        cudaFuncAttributes a;
        SOB_CUDA(cudaFuncGetAttributes(&a, fn));
    }
}
FollowStage g_follow[64];
}  // namespace

// SOB_NO_FOLLOW: diagnostic knob (A/B).  Under an injected CUDA tool (ncu /
// nsys: NV_NSIGHT_INJECTION_*, compute-sanitizer: NV_SANITIZER_INJECTION_*,
// or CUDA_INJECTION64_PATH) kernels may be serialised against the copy they
// follow -- every call would wait for the timeout -- so the follow paths are
// off.  SOB_FOLLOW_UNDER_TOOLS=1 keeps them (the sanitizer driver: a
// timed-out call falls back and stays correct).
bool follow_disabled() {
    static const bool off = [] {
        if (std::getenv("SOB_NO_FOLLOW")) return true;
        if (std::getenv("SOB_FOLLOW_UNDER_TOOLS")) return false;
        for (const char* v : {"CUDA_INJECTION64_PATH", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE",
                              "NV_SANITIZER_INJECTION_TRANSPORT_TYPE", "NV_TPS_LAUNCH_TOKEN"})
            if (std::getenv(v)) return true;
        return false;
    }();
    return off;
}

// The shared part of every follow path: the device's sentinel-filled copy of
// x (allocated / refilled as needed, ordered after the previous call), this
// call's timeout word, the caller's kernels (launched before the upload so
// they trail it), the upload, the copy-complete flag and the refill for the
// next call.
void follow_run(int device, int64_t nc, cudaStream_t s, cudaStream_t copy,
                const std::function<void(const double* dx, const FollowCtx& f)>& kernels,
                const std::function<void(double*)>& upload, FollowToken& tok) {
    FollowStage& f = g_follow[device];
    std::lock_guard<std::mutex> lk(f.mu);
    if (!f.flag) {
        SOB_CUDA(cudaMalloc(reinterpret_cast<void**>(&f.flag), sizeof(unsigned)));
        SOB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&f.one_host), sizeof(unsigned), cudaHostAllocPortable));
        *f.one_host = 1;
        SOB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&f.timed_out), kFollowSlots * sizeof(unsigned),
                               cudaHostAllocMapped | cudaHostAllocPortable));
        for (int i = 0; i < kFollowSlots; ++i) f.timed_out[i] = 0;
        SOB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&f.timed_out_dev), f.timed_out, 0));
        SOB_CUDA(cudaEventCreateWithFlags(&f.refilled, cudaEventDisableTiming));
        SOB_CUDA(cudaEventCreateWithFlags(&f.copied, cudaEventDisableTiming));
        for (int i = 0; i < kFollowSlots; ++i) SOB_CUDA(cudaEventCreateWithFlags(&f.done[i], cudaEventDisableTiming));
        for (auto& e : f.chunk_ev) SOB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (!f.preloaded) {
        follow_preload();
        f.preloaded = true;
    }
    const unsigned slot = f.next_slot++ % kFollowSlots;
    f.timed_out[slot] = 0;
    tok.timed_out = f.timed_out + slot;
    tok.done = f.done[slot];
    const int grid_fill = current_ctx().num_sms * 4;
    // everything of the previous call (its kernels, copy and refill, possibly
    // on another stream) precedes this call's use -- or release -- of dx
    if (f.dx) SOB_CUDA(cudaStreamWaitEvent(s, f.refilled, 0));
    if (f.cap < nc) {
        if (f.dx) SOB_CUDA(cudaFreeAsync(f.dx, s));
        f.dx = nullptr;
        f.cap = 0;
        SOB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&f.dx), sizeof(double) * size_t(nc), s));
        f.cap = nc;
        follow_fill<<<grid_fill, 256, 0, s>>>(reinterpret_cast<unsigned*>(f.dx), 2 * f.cap, f.flag);
        SOB_LAUNCH("follow_fill");
        SOB_CUDA(cudaEventRecord(f.refilled, s));
    }
    // the upload starts once the device copy holds sentinels again
    SOB_CUDA(cudaStreamWaitEvent(copy, f.refilled, 0));
    // 250 ms plus 1 ns per byte of x (a slowly staged pageable x still arrives)
    const FollowCtx fc{f.flag, f.timed_out_dev + slot, 250ull * 1000 * 1000 + 8ull * uint64_t(nc)};
    // pinned x: the copy is queued first (it starts a kernel launch earlier;
    // the kernels still trail it).  Staged x: the upload blocks on host
    // threads, so the kernels go first.  SOB_FOLLOW_KERNEL_FIRST: A/B.
    static const bool kernel_first = std::getenv("SOB_FOLLOW_KERNEL_FIRST") != nullptr;
    if (tok.upload_first && !kernel_first) {
        upload(f.dx);
        kernels(f.dx, fc);
    } else {
        kernels(f.dx, fc);
        upload(f.dx);  // the caller's H2D copies of x into f.dx on `copy`
    }
    SOB_CUDA(cudaMemcpyAsync(f.flag, f.one_host, sizeof(unsigned), cudaMemcpyHostToDevice, copy));
    SOB_CUDA(cudaEventRecord(f.copied, copy));
    // refill the sentinels for the next call once the copy has finished (x
    // columns no row reads are not waited for by the kernels)
    SOB_CUDA(cudaStreamWaitEvent(s, f.copied, 0));
    // the caller waits for this -- kernels and copy done (the caller's x may
    // be reused once it returns) -- not for the refill below
    SOB_CUDA(cudaEventRecord(tok.done, s));
    follow_fill<<<grid_fill, 256, 0, s>>>(reinterpret_cast<unsigned*>(f.dx), 2 * nc, f.flag);
    SOB_LAUNCH("follow_fill");
    SOB_CUDA(cudaEventRecord(f.refilled, s));
}

// The DIA part's window fits the follow kernel (offsets known, staged in
// shared memory, x window of a 1024-row block <= kFollowSpan).
bool dia_follow_ok(const so_matrix& m) {
    if (!m.dia_window_known.load(std::memory_order_acquire) || m.dia.ndiags == 0 || m.dia.ndiags > kDiaSmem)
        return false;
    // x comes from device memory here (no read amplification over the link):
    // any window that fits a CTA's shared memory with its 1024 rows
    return m.dia_omax - m.dia_omin <= kFollowSpan;
}

// dia_follow_kernel over row blocks [b0, b1) (persistent: <= one CTA per SM)
void launch_dia_follow(const so_matrix& m, const double* dx, double* y, cudaStream_t s, const FollowCtx& fc,
                       int64_t b0, int64_t b1) {
    const int64_t omin = m.dia_omin, omax = m.dia_omax;
    const size_t smem = sizeof(double) * size_t(kZcRows + (omax - omin) + 2);
    const unsigned grid = unsigned(std::min<int64_t>(b1 - b0, current_ctx().num_sms));
    dia_follow_kernel<<<grid, kZcRows, smem, s>>>(int(m.nrows), int(m.ncols), int(m.dia.ndiags), m.dia.offsets.get(),
                                                  m.dia.values.get(), dx, y, fc.flag, int(omin), int(omax),
                                                  fc.timed_out, fc.timeout_ns, int(b0), int(b1));
    SOB_LAUNCH("dia_follow_kernel");
}

// wide windows (2-D stencils): opt in to > 48 KB of shared memory, once per device
void dia_follow_smem_attr(const so_matrix& m) {
    const size_t smem = sizeof(double) * size_t(kZcRows + (m.dia_omax - m.dia_omin) + 2);
    if (smem > 48 * 1024) {
        static std::mutex attr_mu;
        static uint64_t attr_done = 0;
        std::lock_guard<std::mutex> alk(attr_mu);
        if (m.device >= 64 || !((attr_done >> m.device) & 1)) {
            SOB_CUDA(cudaFuncSetAttribute(dia_follow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(sizeof(double) * size_t(kZcRows + kFollowSpan + 2))));
            if (m.device < 64) attr_done |= uint64_t(1) << m.device;
        }
    }
}

bool follow_launch(const so_matrix& m, double* y_mapped, cudaStream_t s, cudaStream_t copy, int64_t rows_per_chunk,
                   const std::function<void(int64_t)>* after_chunk, const std::function<void(double*)>& upload,
                   FollowToken& tok) {
    if (follow_disabled()) return false;
    if (m.format != SO_DIA && !(m.format == SO_HDC && m.csr.nnz == 0)) return false;
    if (!dia_follow_ok(m)) return false;
    if (rows_per_chunk < 0 || rows_per_chunk % kZcRows) return false;
    const int64_t nc = m.ncols;
    dia_follow_smem_attr(m);
    const int64_t nblk = ceil_div(m.nrows, int64_t(kZcRows));
    const int64_t per = rows_per_chunk > 0 ? rows_per_chunk / kZcRows : nblk;  // blocks per launch
    follow_run(m.device, nc, s, copy, [&](const double* dx, const FollowCtx& fc) {
        for (int64_t b0 = 0, j = 0; b0 < nblk; b0 += per, ++j) {
            launch_dia_follow(m, dx, y_mapped, s, fc, b0, std::min(nblk, b0 + per));
            if (after_chunk) (*after_chunk)(j);
        }
    }, upload, tok);
    return true;
}

static void coo_profile(const CooPart& coo, int64_t nrows, cudaStream_t s);

// Group / row at each chunk boundary of the pinned CSR pipeline (equal group
// counts), read once per matrix.  False when the groups do not tile the rows.
static bool csr_follow_chunks(const so_matrix& m, cudaStream_t s) {
    constexpr int K = so_matrix::kFollowChunks;
    if (m.csr_chunks_known.load(std::memory_order_acquire)) return m.csr_chunk_row[K].load() == m.nrows;
    int64_t gs[K + 1];
    int32_t rows[K + 1];
    for (int k = 0; k <= K; ++k) {
        gs[k] = m.csr.ngrp * k / K;
        SOB_CUDA(cudaMemcpyAsync(&rows[k], m.csr.grp.get() + gs[k], sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    }
    SOB_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k <= K; ++k) {
        m.csr_chunk_grp[k].store(gs[k], std::memory_order_relaxed);
        m.csr_chunk_row[k].store(rows[0] == 0 ? rows[k] : -1, std::memory_order_relaxed);
    }
    m.csr_chunks_known.store(true, std::memory_order_release);
    return rows[0] == 0 && rows[K] == m.nrows;
}

// Entry-chunk ranges of the pinned COO pipeline (equal chunk counts) and the
// row bound after each.  A CONT chunk writes only rows above the previous
// chunk's last row (its orphan head is skipped, the empty rows before its
// first row are zeroed by it) up to its own last row (finished with the head
// of the next chunk), so rows below row[c_k * kCooChunk - 1] + 1 are final
// once ranges 0..k-1 are done.  Read once per matrix.
static void coo_follow_chunks(const so_matrix& m, cudaStream_t s) {
    constexpr int K = so_matrix::kFollowChunks;
    if (m.coo_chunks_known.load(std::memory_order_acquire)) return;
    const int64_t nch = ceil_div(m.coo.nnz, int64_t(kCooChunk));
    int64_t cs[K + 1];
    int32_t rows[K + 1] = {};
    for (int k = 0; k <= K; ++k) {
        cs[k] = nch * k / K;
        if (k > 0 && k < K)
            SOB_CUDA(cudaMemcpyAsync(&rows[k], m.coo.row.get() + cs[k] * kCooChunk - 1, sizeof(int32_t),
                                     cudaMemcpyDeviceToHost, s));
    }
    SOB_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k <= K; ++k) {
        m.coo_chunk_c[k].store(cs[k], std::memory_order_relaxed);
        m.coo_chunk_row[k].store(k == 0 ? 0 : k == K ? m.nrows : int64_t(rows[k]) + 1, std::memory_order_relaxed);
    }
    m.coo_chunks_known.store(true, std::memory_order_release);
}

// The CONT chunk kernel over entry chunks [c0, c1), following the upload
template <bool ACCUM>
static void launch_coo_cont_range(const CooPart& coo, int64_t nrows, const double* x, double* y, cudaStream_t s,
                                  const FollowCtx& fc, int64_t c0, int64_t c1) {
    const int grid = int(std::min<int64_t>(ceil_div(c1 - c0, 8), int64_t(current_ctx().num_sms) * coo_per_sm(ACCUM)));
    coo_warp_kernel<ACCUM, true, true><<<grid, 256, 0, s>>>(coo.nnz, nrows, coo.row.get(), coo.col.get(),
                                                            coo.val.get(), x, y, nullptr, fc, c0, c1);
    SOB_LAUNCH("coo_warp_kernel");
}

// Pinned spmv(m, x) on a CSR matrix (or HDC without a DIA part) or an ELL
// matrix (or HYB without a COO part): the kernels launched with FOLLOW trail
// ONE upload of x (each x gather waits for its element) and store y straight
// into mapped host memory, so y goes down while x still comes up.  The
// persistent CSR warp kernel walks its groups in address order (group g,
// g + grid, ...) and the ELL grid runs its row blocks in order, so on banded
// / stencil rows the kernels follow the copy front; scattered columns just
// wait longer.  COO (and HYB with a COO part) follow the upload the same way
// but into device y, copied down after the fix-up: their row sums end at
// scattered lanes, and 8-byte stores into mapped memory each cost a link
// transaction (profiles/r02ac_ab_mapped_y.txt).
bool follow_launch_rows(const so_matrix& m, double* y_mapped, cudaStream_t s, cudaStream_t copy,
                        const std::function<void(const double* y_dev)>* after_kernels,
                        const std::function<void(double*)>& upload, FollowToken& tok) {
    static const bool off = std::getenv("SOB_NO_CSR_FOLLOW") != nullptr;  // diagnostic knob (A/B)
    static const bool coo_off = std::getenv("SOB_NO_COO_FOLLOW") != nullptr;  // diagnostic knob (A/B)
    static const bool hdc_off = std::getenv("SOB_NO_HDC_FOLLOW") != nullptr;  // diagnostic knob (A/B)
    if (off || follow_disabled()) return false;
    const bool csr = (m.format == SO_CSR || (m.format == SO_HDC && m.dia.ndiags == 0)) && m.csr.nnz > 0;
    const bool ell = (m.format == SO_ELL || (m.format == SO_HYB && m.coo.nnz == 0)) && m.ell.width > 0;
    const bool coo = !coo_off && (m.format == SO_COO || m.format == SO_HYB) && m.coo.nnz > 0;
    // HDC with both parts: the DIA follow kernel, then the CSR part
    // accumulating (spmv_device's order), into device y
    bool hdc2 = !hdc_off && m.format == SO_HDC && m.dia.ndiags > 0 && m.csr.nnz > 0;
    if (hdc2) {
        ensure_dia_window(m, s);  // cached after the first call
        hdc2 = dia_follow_ok(m);
        if (hdc2) dia_follow_smem_attr(m);
    }
    if (!csr && !ell && !coo && !hdc2) return false;
    if (coo) coo_profile(m.coo, m.nrows, s);  // cached after the first multiply
    // pinned CSR without long rows: kFollowChunks launches over equal group
    // ranges into device y, each chunk's y copied down on copy_out as soon as
    // it is done -- the rows kernel's short, partly filled y stores into
    // mapped memory made the y leg the slow one.  SOB_NO_CSR_CHUNKS: A/B.
    static const bool no_chunks = std::getenv("SOB_NO_CSR_CHUNKS") != nullptr;
    const bool chunks = csr && !after_kernels && !no_chunks && m.csr.nlong == 0 &&
                        m.csr.ngrp >= 64 * so_matrix::kFollowChunks && csr_follow_chunks(m, s);
    // pinned COO of short rows (every row <= 32 entries): the CONT chunk
    // kernel (no records, no fix-up) over kFollowChunks entry-chunk ranges,
    // each range's rows copied down as it completes.  SOB_NO_COO_CHUNKS: A/B.
    static const bool no_coo_chunks = std::getenv("SOB_NO_COO_CHUNKS") != nullptr;
    const bool coo_chunks = coo && m.format == SO_COO && !after_kernels && !no_coo_chunks &&
                            m.coo.short_rows.load(std::memory_order_acquire) == 1 &&
                            ceil_div(m.coo.nnz, int64_t(kCooChunk)) >= 64 * so_matrix::kFollowChunks;
    if (coo_chunks) coo_follow_chunks(m, s);
    // pinned HDC with both parts, no long rows: per CSR chunk, the DIA row
    // blocks starting in its rows, then its groups accumulating, then its
    // rows copied down (the same pipeline; SOB_NO_CSR_CHUNKS: A/B)
    const bool hdc_chunks = hdc2 && !after_kernels && !no_chunks && m.csr.nlong == 0 &&
                            m.csr.ngrp >= 64 * so_matrix::kFollowChunks && csr_follow_chunks(m, s);
    follow_run(m.device, m.ncols, s, copy, [&](const double* dx, const FollowCtx& fc) {
        if (chunks) {
            constexpr int K = so_matrix::kFollowChunks;
            FollowStage& st = g_follow[m.device];  // follow_run holds st.mu here
            cudaStream_t out = current_ctx().copy_out;
            DBuf<double> yd(m.nrows, s);  // released stream-ordered after the copies
            for (int k = 0; k < K; ++k) {
                const int64_t g0 = m.csr_chunk_grp[k].load(), g1 = m.csr_chunk_grp[k + 1].load();
                const int64_t r0 = m.csr_chunk_row[k].load(), r1 = m.csr_chunk_row[k + 1].load();
                if (g1 > g0) launch_csr_groups_follow(m, dx, yd.get(), s, fc, g0, g1);
                SOB_CUDA(cudaEventRecord(st.chunk_ev[k], s));
                SOB_CUDA(cudaStreamWaitEvent(out, st.chunk_ev[k], 0));
                if (r1 > r0)
                    SOB_CUDA(cudaMemcpyAsync(y_mapped + r0, yd.get() + r0, sizeof(double) * size_t(r1 - r0),
                                             cudaMemcpyDefault, out));
            }
            SOB_CUDA(cudaEventRecord(st.chunk_ev[K], out));
            SOB_CUDA(cudaStreamWaitEvent(s, st.chunk_ev[K], 0));
        } else if (csr) {
            launch_csr_stream(m, false, dx, y_mapped, s, &fc);
            if (after_kernels) (*after_kernels)(nullptr);
        } else if (ell) {
            launch_ell<false>(m, dx, y_mapped, s, &fc);
            if (after_kernels) (*after_kernels)(nullptr);
        } else if (hdc_chunks) {
            constexpr int K = so_matrix::kFollowChunks;
            FollowStage& st = g_follow[m.device];  // follow_run holds st.mu here
            cudaStream_t out = current_ctx().copy_out;
            DBuf<double> yd(m.nrows, s);  // released stream-ordered after the copies
            // a DIA block is run with the chunk its first row is in: every
            // row's block is done before (or with) the chunk accumulating it
            for (int k = 0; k < K; ++k) {
                const int64_t g0 = m.csr_chunk_grp[k].load(), g1 = m.csr_chunk_grp[k + 1].load();
                const int64_t r0 = m.csr_chunk_row[k].load(), r1 = m.csr_chunk_row[k + 1].load();
                const int64_t b0 = ceil_div(r0, int64_t(kZcRows)), b1 = ceil_div(r1, int64_t(kZcRows));
                if (b1 > b0) launch_dia_follow(m, dx, yd.get(), s, fc, b0, b1);
                if (g1 > g0) launch_csr_groups_follow(m, dx, yd.get(), s, fc, g0, g1, true);
                SOB_CUDA(cudaEventRecord(st.chunk_ev[k], s));
                SOB_CUDA(cudaStreamWaitEvent(out, st.chunk_ev[k], 0));
                if (r1 > r0)
                    SOB_CUDA(cudaMemcpyAsync(y_mapped + r0, yd.get() + r0, sizeof(double) * size_t(r1 - r0),
                                             cudaMemcpyDefault, out));
            }
            SOB_CUDA(cudaEventRecord(st.chunk_ev[K], out));
            SOB_CUDA(cudaStreamWaitEvent(s, st.chunk_ev[K], 0));
        } else if (hdc2) {
            // released stream-ordered after the copy below; allocated before
            // the first launch (see follow_preload)
            DBuf<double> yd(m.nrows, s);
            DBuf<double> part(m.csr.nlong > 0 ? m.csr.npieces : 0, s);
            launch_dia_follow(m, dx, yd.get(), s, fc, 0, ceil_div(m.nrows, int64_t(kZcRows)));
            launch_csr_stream(m, true, dx, yd.get(), s, &fc, &part);
            if (after_kernels)
                (*after_kernels)(yd.get());
            else
                SOB_CUDA(cudaMemcpyAsync(y_mapped, yd.get(), sizeof(double) * size_t(m.nrows), cudaMemcpyDefault, s));
        } else if (coo_chunks) {
            constexpr int K = so_matrix::kFollowChunks;
            FollowStage& st = g_follow[m.device];  // follow_run holds st.mu here
            cudaStream_t out = current_ctx().copy_out;
            DBuf<double> yd(m.nrows, s);  // released stream-ordered after the copies
            const int64_t gap = m.coo.max_gap.load(std::memory_order_acquire);
            const bool zeroed = gap < 0 || gap > kCooGapInline;  // spmv_device's safe path: y zeroed, accumulate
            if (zeroed) SOB_CUDA(cudaMemsetAsync(yd.get(), 0, sizeof(double) * size_t(m.nrows), s));
            for (int k = 0; k < K; ++k) {
                const int64_t c0 = m.coo_chunk_c[k].load(), c1 = m.coo_chunk_c[k + 1].load();
                const int64_t r0 = m.coo_chunk_row[k].load(), r1 = m.coo_chunk_row[k + 1].load();
                if (c1 > c0) {
                    if (zeroed)
                        launch_coo_cont_range<true>(m.coo, m.nrows, dx, yd.get(), s, fc, c0, c1);
                    else
                        launch_coo_cont_range<false>(m.coo, m.nrows, dx, yd.get(), s, fc, c0, c1);
                }
                SOB_CUDA(cudaEventRecord(st.chunk_ev[k], s));
                SOB_CUDA(cudaStreamWaitEvent(out, st.chunk_ev[k], 0));
                if (r1 > r0)
                    SOB_CUDA(cudaMemcpyAsync(y_mapped + r0, yd.get() + r0, sizeof(double) * size_t(r1 - r0),
                                             cudaMemcpyDefault, out));
            }
            SOB_CUDA(cudaEventRecord(st.chunk_ev[K], out));
            SOB_CUDA(cudaStreamWaitEvent(s, st.chunk_ev[K], 0));
        } else {
            // both released stream-ordered after the copy below; allocated
            // before the first launch (see follow_preload)
            DBuf<double> yd(m.nrows, s);
            DBuf<CooChunkRec> rec(coo_cont(m.coo) ? 0 : coo_rec_count(m.coo), s);
            if (m.format == SO_HYB) {
                launch_ell<false>(m, dx, yd.get(), s, m.ell.width > 0 ? &fc : nullptr);
                launch_coo<true>(m.coo, m.nrows, dx, yd.get(), s, &fc, &rec);
            } else if (m.coo.max_gap < 0 || m.coo.max_gap > kCooGapInline) {  // spmv_device's safe path
                SOB_CUDA(cudaMemsetAsync(yd.get(), 0, sizeof(double) * size_t(m.nrows), s));
                launch_coo<true>(m.coo, m.nrows, dx, yd.get(), s, &fc, &rec);
            } else {
                launch_coo<false>(m.coo, m.nrows, dx, yd.get(), s, &fc, &rec);
            }
            if (after_kernels)
                (*after_kernels)(yd.get());
            else
                SOB_CUDA(cudaMemcpyAsync(y_mapped, yd.get(), sizeof(double) * size_t(m.nrows), cudaMemcpyDefault, s));
        }
    }, upload, tok);
    return true;
}

// A pinned call returns once its kernels are done (y is in host memory);
// the sentinel refill queued behind them on `s` is not waited for.
static void follow_wait_done(const FollowToken& tok, cudaStream_t s) {
    static const bool stream_sync = std::getenv("SOB_FOLLOW_KERNEL_FIRST") != nullptr;  // A/B (as before)
    if (stream_sync)
        SOB_CUDA(cudaStreamSynchronize(s));
    else
        SOB_CUDA(cudaEventSynchronize(tok.done));
}

bool spmv_csr_follow(const so_matrix& m, const double* x_host, double* y_mapped, cudaStream_t s,
                     cudaStream_t copy) {
    const int64_t nc = m.ncols;
    FollowToken tok;
    tok.upload_first = true;
    if (!follow_launch_rows(m, y_mapped, s, copy, nullptr, [&](double* dx) {
            SOB_CUDA(cudaMemcpyAsync(dx, x_host, sizeof(double) * size_t(nc), cudaMemcpyHostToDevice, copy));
        }, tok))
        return false;
    follow_wait_done(tok, s);
    if (!follow_finish(tok)) {  // the copy never showed up: recompute elsewhere
        SOB_CUDA(cudaStreamSynchronize(copy));
        return false;
    }
    return true;
}

bool follow_finish(FollowToken& tok) {
    bool ok = true;
    if (tok.timed_out && *reinterpret_cast<volatile unsigned*>(tok.timed_out)) {
        ok = false;
    }
    return ok;
}

bool spmv_dia_follow(const so_matrix& m, const double* x_host, double* y_mapped, cudaStream_t s,
                     cudaStream_t copy) {
    FollowToken tok;
    tok.upload_first = true;
    const int64_t nc = m.ncols;
    const bool launched = follow_launch(m, y_mapped, s, copy, 0, nullptr, [&](double* dx) {
        SOB_CUDA(cudaMemcpyAsync(dx, x_host, sizeof(double) * size_t(nc), cudaMemcpyHostToDevice, copy));
    }, tok);
    if (!launched) return false;
    follow_wait_done(tok, s);
    if (!follow_finish(tok)) {  // the copy never showed up: recompute elsewhere
        SOB_CUDA(cudaStreamSynchronize(copy));
        return false;
    }
    return true;
}

void spmv_device_rows(const so_matrix& m, const double* x, double* y, int64_t lo, int64_t hi, cudaStream_t s) {
    if (m.format != SO_DIA && !(m.format == SO_HDC && m.csr.nnz == 0))
        fail(SO_INVALID_INPUT, "row-range SpMV is implemented for DIA matrices (and HDC with an empty CSR part)");
    if (lo < 0 || hi > m.nrows || lo > hi) fail(SO_INVALID_INPUT, "row range outside the matrix");
    launch_dia(m, x, y, s, lo, hi);
}

void spmv_rows_push(const so_matrix& m, const double* x, double* y, int64_t lo, int64_t hi, double* remote,
                    unsigned* ticket, unsigned long long* remote_flag, unsigned long long flag_value,
                    cudaStream_t s) {
    if (m.format != SO_DIA && !(m.format == SO_HDC && m.csr.nnz == 0))
        fail(SO_INVALID_INPUT, "row-range SpMV is implemented for DIA matrices (and HDC with an empty CSR part)");
    if (lo < 0 || hi > m.nrows || lo >= hi) fail(SO_INVALID_INPUT, "row range outside the matrix or empty");
    if (!remote || !ticket || !remote_flag) fail(SO_INVALID_INPUT, "null peer pointer");
    const unsigned grid = unsigned(ceil_div(hi - lo, 256));
    if (m.dia.ndiags <= kDiaSmem)
        dia_push_kernel<false><<<grid, 256, 0, s>>>(m.nrows, m.ncols, int(m.dia.ndiags), m.dia.offsets.get(),
                                                    m.dia.values.get(), x, y, lo, hi, remote, ticket, remote_flag,
                                                    flag_value);
    else
        dia_push_kernel<true><<<grid, 256, 0, s>>>(m.nrows, m.ncols, int(m.dia.ndiags), m.dia.offsets.get(),
                                                   m.dia.values.get(), x, y, lo, hi, remote, ticket, remote_flag,
                                                   flag_value);
    SOB_LAUNCH("dia_push_kernel");
}

unsigned long long wait_flag_timeouts() {
    unsigned long long v = 0;
    SOB_CUDA(cudaMemcpyFromSymbol(&v, g_wait_timeouts, sizeof(v)));
    return v;
}

void wait_flag(const unsigned long long* flag, unsigned long long value, cudaStream_t s) {
    if (!flag) fail(SO_INVALID_INPUT, "null flag");
    wait_flag_kernel<<<1, 1, 0, s>>>(flag, value);
    SOB_LAUNCH("wait_flag_kernel");
}

// First multiply of a COO part (outside stream capture): the longest empty
// run and whether any row is long enough to need coo_fixup_long; cached.
static void coo_profile(const CooPart& coo, int64_t nrows, cudaStream_t s) {
    if (coo.max_gap >= 0 || coo.nnz == 0) return;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    SOB_CUDA(cudaStreamIsCapturing(s, &cap));
    if (cap != cudaStreamCaptureStatusNone) return;  // stays unknown: safe paths
    DBuf<unsigned long long> g(3, s);
    SOB_CUDA(cudaMemsetAsync(g.get(), 0, 3 * sizeof(unsigned long long), s));
    coo_max_gap<<<grid_for(coo.nnz + 1, 256, 4), 256, 0, s>>>(coo.nnz, nrows, coo.row.get(), g.get());
    SOB_LAUNCH("coo_max_gap");
    unsigned long long h[3];
    SOB_CUDA(cudaMemcpyAsync(h, g.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    SOB_CUDA(cudaStreamSynchronize(s));
    coo.long_runs = h[1] ? 1 : 0;
    coo.short_rows = h[2] ? 0 : 1;
    coo.max_gap = int64_t(h[0]);
}

void spmv_device(const so_matrix& m, const double* x, double* y, cudaStream_t s) {
    if (m.nrows <= 0) return;
    switch (m.format) {
        case SO_COO: {
            coo_profile(m.coo, m.nrows, s);
            if (m.coo.nnz == 0) {
                SOB_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * size_t(m.nrows), s));
            } else if (m.coo.max_gap < 0 || m.coo.max_gap > kCooGapInline) {  // unknown under capture: safe path
                SOB_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * size_t(m.nrows), s));
                launch_coo<true>(m.coo, m.nrows, x, y, s);
            } else {
                launch_coo<false>(m.coo, m.nrows, x, y, s);
            }
            break;
        }
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
            coo_profile(m.coo, m.nrows, s);
            launch_ell<false>(m, x, y, s);
            if (m.coo.nnz > 0) launch_coo<true>(m.coo, m.nrows, x, y, s);
            break;
        case SO_HDC:
            // one kernel per non-empty part; both parts: the DIA kernel, then
            // the CSR part accumulating into y (spmv.cpp:101-106 order).  A
            // fused per-row DIA+CSR kernel measured slower on every shape
            // tried (0.34-0.74 vs 0.38-0.90 of peak)
            if (m.csr.nnz == 0) {
                launch_dia(m, x, y, s);
            } else if (m.dia.ndiags == 0) {
                launch_csr_stream(m, false, x, y, s);
            } else {
                launch_dia(m, x, y, s);
                launch_csr_stream(m, true, x, y, s);
            }
            break;
        default:
            fail(SO_INVALID_INPUT, "unknown format");
    }
}

}  // namespace sob
