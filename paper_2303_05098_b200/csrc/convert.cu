// Device conversions, CSR -> {COO, DIA, ELL, HYB, HDC} and back.
//
// The reference converts through canonical COO on the host (formats.cpp:
// 411-467).  Here the canonical source is the device CSR (identical content:
// to_coo(CSR) is canonical), and every conversion is two-phase: a size pass
// on the device, the PaddingOverflow cap check on the host BEFORE the dense
// allocation (formats.cpp:81-84, 111-112), then a fill pass.  Host-visible
// arrays are bit-identical to the reference's (tests/test_gpu_formats.py).
#include <cmath>
#include <limits>
#include <memory>
#include <vector>

#include "hist.cuh"
#include "matrix.cuh"

namespace sob {

// ---------------------------------------------------------------- host rules

int64_t checked_mul(int64_t a, int64_t b) {  // formats.cpp:14-20
    if (a == 0 || b == 0) return 0;
    if (a > std::numeric_limits<int64_t>::max() / b) return std::numeric_limits<int64_t>::max();
    return a * b;
}

int64_t padded_entry_cap(const so_conversion_config& c, int64_t nnz) {  // formats.cpp:348-355
    if (c.max_padded_entries > 0) return c.max_padded_entries;
    const double cap = c.max_padding_factor * double(nnz);
    if (cap >= double(std::numeric_limits<int64_t>::max())) return std::numeric_limits<int64_t>::max();
    return int64_t(cap);
}

int64_t effective_kh(const so_conversion_config& c, int64_t nnz, int64_t nrows) {  // :357-361
    if (c.kh_override > 0) return c.kh_override;
    if (nrows <= 0 || nnz <= 0) return 0;
    return (nnz + nrows - 1) / nrows;
}

int64_t true_diag_threshold(double ratio, int64_t nrows, int64_t ncols) {  // :363-367
    const double len = double(nrows < ncols ? nrows : ncols);
    return int64_t(std::ceil(ratio * len));
}

static void check_cap(int64_t allocation, int64_t cap, const char* what) {  // formats.cpp:36-43
    if (allocation > cap)
        fail(SO_PADDING_OVERFLOW, std::string(what) + " allocation of " + std::to_string(allocation) +
                                      " entries exceeds padding cap " + std::to_string(cap));
}

namespace {

constexpr int kB = 256;

// ------------------------------------------------------- generic entry sweep
// CTA-per-row-block sweep over the entries of a CSR (grid-stride over blocks).
// op(row, k) is called for every entry; rows are found by binary search in the
// block's row_ptr slice staged in shared memory.  Loop trip counts are
// block-uniform so ops may use warp-synchronous primitives (valid=false lanes).
template <class Op>
__global__ void __launch_bounds__(kB) csr_sweep(const int32_t* __restrict__ blk, int64_t nblk,
                                                 const int64_t* __restrict__ rp, Op op) {
    __shared__ int64_t srp[kRowsPerBlock + 1];
    op.begin();
    for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
        const int r0 = blk[b], nr = blk[b + 1] - r0;
        __syncthreads();
        for (int j = threadIdx.x; j <= nr; j += kB) srp[j] = rp[r0 + j];
        __syncthreads();
        const int64_t k0 = srp[0], k1 = srp[nr];
        for (int64_t base = k0; base < k1; base += kB) {
            const int64_t k = base + threadIdx.x;
            const bool valid = k < k1;
            const int r = valid ? r0 + row_in_block(srp, nr, k) : -1;
            op(r, k, valid);
        }
    }
    op.end();
}

struct OpBase {
    static constexpr bool kHasEntry = false;  // op.entry(r, col, valid): column-prefetching sweep
    static constexpr bool kHasEntry8 = false;
    __device__ void begin() {}
    __device__ void row(int, bool, int64_t) {}
    __device__ void end() {}
};

template <class Op>
void sweep(const so_matrix& csr, Op op, cudaStream_t s, int per_sm = 4) {
    if (csr.csr.nblk == 0) return;
    csr_sweep<Op><<<grid_for(csr.csr.nblk * kB, kB, per_sm), kB, 0, s>>>(csr.csr.blk.get(), csr.csr.nblk,
                                                                         csr.csr.row_ptr.get(), op);
    SOB_LAUNCH("csr_sweep");
}

// Row-lockstep sweep of every entry; rows longer than grp_cap go
// through the piece-parallel sweep (no single-warp tail on skewed rows).
template <class Op>
void row_sweep_launch(const so_matrix& csr, Op op, cudaStream_t s, bool prefetch_cols = false) {
    if (csr.nrows <= 0) return;
    const CsrPart& c = csr.csr;
    const int64_t skip = c.nlong > 0 ? int64_t(c.grp_cap) : INT64_MAX;
    DBuf<unsigned> ticket;  // dynamic row groups when the row lengths are skewed
    if (c.nlong > 0) {
        ticket.alloc(1, s);
        SOB_CUDA(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned), s));
    }
    const int g = grid_for(ceil_div(csr.nrows, 32) * 256 / 8, 256, 8);
    if constexpr (Op::kHasEntry) {
        if (prefetch_cols) {
            row_sweep_cols<Op><<<g, 256, 0, s>>>(c.row_ptr.get(), c.col.get(), csr.nrows, op, skip, ticket.get());
        } else {
            row_sweep<Op><<<g, 256, 0, s>>>(c.row_ptr.get(), csr.nrows, op, skip, ticket.get());
        }
    } else {
        row_sweep<Op><<<g, 256, 0, s>>>(c.row_ptr.get(), csr.nrows, op, skip, ticket.get());
    }
    SOB_LAUNCH("row_sweep");
    if (c.nlong > 0) {
        piece_sweep<Op><<<unsigned(c.npieces), 256, 0, s>>>(c.piece_k.get(), c.long_row.get(), c.long_piece.get(),
                                                            c.nlong, op);
        SOB_LAUNCH("piece_sweep");
    }
}

// ---------------------------------------------------------- row-block build

__device__ __forceinline__ int64_t ceil_div_d(int64_t a, int64_t b) { return (a + b - 1) / b; }

__global__ void row_block_flags(const int64_t* __restrict__ rp, int64_t n, int32_t* __restrict__ flag) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t len = rp[i + 1] - rp[i];
    bool start = (i == 0) || (i % kRowsPerBlock == 0) || len > kWindow;
    if (i > 0) {
        const int64_t plen = rp[i] - rp[i - 1];
        start = start || plen > kWindow || (rp[i] / kWindow) != (rp[i - 1] / kWindow);
    }
    flag[i] = start ? 1 : 0;
}

__global__ void row_block_scatter(const int32_t* __restrict__ flag, const int64_t* __restrict__ pos,
                                  const int64_t* __restrict__ rp, int64_t n, int32_t* __restrict__ blk,
                                  int64_t* __restrict__ blk_k) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) {
        blk[pos[i]] = int32_t(i);
        blk_k[pos[i]] = rp[i];
    }
    if (i == n) {
        blk[pos[n]] = int32_t(n);
        blk_k[pos[n]] = rp[n];
    }
}

// rows of kCoopLen < length <= cap (the SpMV's warp-cooperative rows)
__global__ void count_coop_rows(const int64_t* __restrict__ rp, int64_t n, int64_t cap,
                                unsigned long long* __restrict__ out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t len = i < n ? rp[i + 1] - rp[i] : 0;
    const unsigned b = __ballot_sync(0xffffffffu, len > kCoopLen && len <= cap);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(out, (unsigned long long)__popc(b));
}

__global__ void long_row_flags(const int64_t* __restrict__ rp, int64_t n, int64_t limit, int32_t* __restrict__ flag) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = (rp[i + 1] - rp[i]) > limit ? 1 : 0;
}

// SpMV warp groups, greedy: a group is <= 32 consecutive rows holding <= cap
// entries; a row longer than cap stands alone (and is split into pieces).
// One warp per kGroupChunk rows (chunk starts are forced group starts, so
// the partition is deterministic and parallel) flags group starts: the
// chunk's row_ptr is staged in shared memory (coalesced), then each group
// costs one ballot -- the next start is the first row whose end passes
// base + cap (or base row itself when it is longer than cap), at most 32
// rows on.  (A thread walking its chunk row by row took ~150 us at any size.)
// Shared-memory layout of each warp group's products (csr_warp_kernel):
// lane i walks prod[pa_i + j], so rows of one even length (16 entries: every
// lane on one bank) serialise the walk.  The padded layout stores entry e at
// e + e / 16; a group takes it when its row starts cover more of the 16
// double-wide banks that way, flagged in bit kGrpPadBit of grp_k[g] (decided
// once here, so the SpMV pays no vote).
// Two launches: count (SET = false), then -- only when at least 1/64 of the
// groups prefer the padded layout, i.e. when the SpMV will run the padded
// kernel -- flag (SET = true); otherwise grp_k stays plain and the
// plain-layout kernel reads it unmasked.
// npad[1] (count pass) counts groups of more than 32 rows.
template <bool SET>
__global__ void group_pad_flags(const int32_t* __restrict__ grp, int64_t* __restrict__ grp_k, int64_t ngrp,
                                const int64_t* __restrict__ rp, int cap, unsigned long long* npad) {
    const int lane = threadIdx.x & 31;
    const int64_t g = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (g >= ngrp) return;
    const int r0 = grp[g], r1 = grp[g + 1];
    if (!SET && lane == 0 && r1 - r0 > 32) atomicAdd(npad + 1, 1ull);
    const int64_t k0 = grp_k[g];
    if (grp_k[g + 1] - k0 > cap) return;  // a long row: pieces, no walk
    const bool act = r0 + lane < r1;
    const int pa = act ? int(rp[r0 + lane] - k0) : 0;
    const unsigned o0 = __reduce_or_sync(~0u, act ? 1u << (pa & 15) : 0u);
    const unsigned o1 = __reduce_or_sync(~0u, act ? 1u << ((pa + (pa >> 4)) & 15) : 0u);
    if (lane == 0 && __popc(o1) > __popc(o0)) {
        if (SET)
            grp_k[g] = k0 | kGrpPad;
        else
            atomicAdd(npad, 1ull);
    }
}

constexpr int kGroupChunk = 1024;
constexpr int kGroupWarps = 4;
__global__ void __launch_bounds__(32 * kGroupWarps)
    group_flags(const int64_t* __restrict__ rp, int64_t n, int64_t cap, int32_t* __restrict__ flag) {
    __shared__ int64_t srp[kGroupWarps][kGroupChunk + 1];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t lo = (int64_t(blockIdx.x) * kGroupWarps + w) * kGroupChunk;
    if (lo >= n) return;
    const int len = int(lo + kGroupChunk < n ? kGroupChunk : n - lo);
    int64_t* r = srp[w];
    for (int j = lane; j <= len; j += 32) r[j] = rp[lo + j];
    for (int j = lane; j < len; j += 32) flag[lo + j] = 0;
    __syncwarp();
    for (int g = 0; g < len;) {
        if (lane == 0) flag[lo + g] = 1;
        const int64_t base = r[g];
        // the next start: the first row whose end passes base + cap, at most
        // kGroupRowsMax rows on (one ballot per 32 rows)
        int step = kGroupRowsMax;
        for (int w = 0; w < kGroupRowsMax; w += 32) {
            const int j = g + w + lane;
            const bool over = j < len && r[j + 1] - base > cap;
            const unsigned b = __ballot_sync(0xffffffffu, over);
            if (b) {
                step = w + __ffs(b) - 1;
                break;
            }
            if (g + w + 32 >= len) break;  // the chunk ends first
        }
        g += step ? step : 1;  // step 0: the base row alone exceeds cap
    }
}

__global__ void long_row_list(const int64_t* __restrict__ rp, const int32_t* __restrict__ flag,
                              const int64_t* __restrict__ pos, int64_t n, int32_t* __restrict__ lrow,
                              int64_t* __restrict__ npc) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n || !flag[i]) return;
    lrow[pos[i]] = int32_t(i);
    npc[pos[i]] = ceil_div_d(rp[i + 1] - rp[i], kPiece);
}

__global__ void long_row_pieces(const int64_t* __restrict__ rp, const int32_t* __restrict__ lrow,
                                const int64_t* __restrict__ lpiece, int64_t nlong, int64_t* __restrict__ pk) {
    const int64_t l = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (l >= nlong) return;
    const int64_t a = rp[lrow[l]], e = rp[lrow[l] + 1];
    for (int64_t p = lpiece[l], k = a; p < lpiece[l + 1]; ++p, k += kPiece) {
        pk[2 * p] = k;
        pk[2 * p + 1] = k + kPiece < e ? k + kPiece : e;
    }
}

// ------------------------------------------------------------ COO -> CSR

__global__ void coo_canonical_check(const int32_t* __restrict__ row, const int32_t* __restrict__ col,
                                    int64_t z, int* __restrict__ bad) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x + 1;
    if (k >= z) return;
    const int32_t r0 = row[k - 1], r1 = row[k];
    if (!(r0 < r1 || (r0 == r1 && col[k - 1] < col[k]))) atomicExch(bad, 1);
}

// row_ptr from a row-sorted row array: every row_ptr slot written exactly once.
__global__ void coo_row_ptr(const int32_t* __restrict__ row, int64_t z, int64_t n, int64_t* __restrict__ rp) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k > z) return;
    const int64_t lo = k == 0 ? 0 : int64_t(row[k - 1]) + 1;
    const int64_t hi = k == z ? n : int64_t(row[k]);
    for (int64_t r = lo; r <= hi; ++r) rp[r] = k;
}

// --------------------------------------------------------------- reductions

__global__ void row_len_max(const int64_t* __restrict__ rp, int64_t n, int64_t cap_at,
                            unsigned long long* __restrict__ out) {
    int64_t m = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        int64_t len = rp[i + 1] - rp[i];
        if (cap_at >= 0 && len > cap_at) len = cap_at;
        m = len > m ? len : m;
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)m);
}

// ------------------------------------------------------------------- DIA
// formats.cpp:64-96: seen[key] -> ascending offsets -> cap -> fill.

// flag[key] = a diagonal with >= max(1, thr) entries exists (thr = 0: DIA,
// thr = ceil(ratio*min(n,m)): HDC's true diagonals)
__global__ void bins_to_flags(const int32_t* __restrict__ bins, int64_t nkeys, int64_t thr,
                              int32_t* __restrict__ flag) {
    const int64_t key = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (key < nkeys) flag[key] = (bins[key] >= 1 && bins[key] >= thr) ? 1 : 0;
}

__global__ void keys_to_offsets(const int32_t* __restrict__ flag, const int64_t* __restrict__ pos,
                                int64_t nkeys, int64_t nrows, int64_t* __restrict__ offsets) {
    const int64_t key = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (key < nkeys && flag[key]) offsets[pos[key]] = key - (nrows - 1);
}

struct FillDia : OpBase {
    const int32_t* col;
    const double* val;
    int64_t nrows;
    const int64_t* pos;  // key -> diagonal slot
    const int32_t* bins;
    int64_t thr;
    double* values;
    unsigned long long* stored;
    unsigned long long count = 0;  // per-thread, flushed once in end()
    __device__ void operator()(int r, int64_t k, bool valid) {
        if (!valid) return;
        const int64_t key = int64_t(__ldg(col + k)) - r + nrows - 1;
        if (!bins || __ldg(bins + key) >= thr) {
            const double v = __ldg(val + k);
            values[__ldg(pos + key) * nrows + r] = v;
            count += v != 0.0;  // formats.cpp:93 -- stored_nnz counts nonzero cells
        }
    }
    __device__ void end() {
        const unsigned long long c = warp_sum(count);
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(stored, c);
    }
};

// -------------------------------------------------------------- ELL / HYB

// Row-major traversal, column-major writes: thread per row walks its slots;
// consecutive threads write consecutive cells of each slot (coalesced) and
// read their own contiguous row (L1-resident for a warp).  Every padded slot
// is written exactly once: real entries first, then sentinel -1 / 0.0.
__global__ void ell_fill(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                         const double* __restrict__ val, int64_t nrows, int64_t width,
                         int32_t* __restrict__ ecol, double* __restrict__ eval) {
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows;
         r += int64_t(gridDim.x) * blockDim.x) {
        const int64_t a = rp[r], len = rp[r + 1] - a;
        for (int64_t j = 0; j < width; ++j) {
            const bool real = j < len;
            ecol[j * nrows + r] = real ? col[a + j] : -1;
            eval[j * nrows + r] = real ? val[a + j] : 0.0;
        }
    }
}

__global__ void hyb_surplus(const int64_t* __restrict__ rp, int64_t n, int64_t kh, int64_t* __restrict__ cnt) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t len = rp[i + 1] - rp[i];
    cnt[i] = len > kh ? len - kh : 0;
}

struct FillHybCoo : OpBase {
    const int64_t* rp;
    const int32_t* col;
    const double* val;
    int64_t kh;
    const int64_t* coo_off;
    int32_t *crow, *ccol;
    double* cval;
    __device__ void operator()(int r, int64_t k, bool valid) const {
        if (!valid) return;
        const int64_t j = k - rp[r];
        if (j < kh) return;
        const int64_t p = coo_off[r] + (j - kh);
        crow[p] = r;
        ccol[p] = col[k];
        cval[p] = val[k];
    }
};

// ------------------------------------------------------------------- HDC

struct DiagHist : OpBase {
    static constexpr bool kHasEntry = true;
    const int32_t* col;
    int64_t nrows;
    int32_t* bins;
    SmemHash* h;
    __device__ void begin() {
        __shared__ SmemHash sh;
        h = &sh;
        hash_init(sh);
        __syncthreads();
    }
    __device__ void operator()(int r, int64_t k, bool valid) {
        const int32_t key = valid ? int32_t(int64_t(col[k]) - r + nrows - 1) : -1;
        hash_add(*h, bins, key);
    }
    static constexpr bool kPieceDirect = true;  // piece_sweep (hist.cuh)
    __device__ void piece(int r, int64_t k, bool valid) {
        if (valid) atomicAdd(bins + (int64_t(col[k]) - r + nrows - 1), 1);
    }
    __device__ bool scattered() const { return __shfl_sync(0xffffffffu, h->used >= kHashSlots / 2, 0); }
    __device__ void direct(int r, int32_t c, bool valid) {
        if (valid) hash_insert_one(*h, bins, int32_t(int64_t(c) - r + nrows - 1), 1);
    }
    SlotCache cache;
    static constexpr bool kHasEntry8 = true;
    __device__ void entry(int r, int32_t c, bool valid, int slot) {
        const int32_t key = valid ? int32_t(int64_t(c) - r + nrows - 1) : -1;
        if (!cache.add(*h, bins, key, slot)) hash_add(*h, bins, key);
    }
    // eight full lockstep slots of one warp (row_sweep_cols)
    __device__ bool entry8(int r, const int32_t (&c)[8], int j0, bool all_valid) {
        int32_t k[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) k[u] = int32_t(int64_t(c[u]) - r + nrows - 1);
        return cache.add8(*h, bins, k, j0, all_valid);
    }
    __device__ void end() {
        cache.flush(*h, bins);
        __syncthreads();
        hash_flush(*h, bins);
    }
};

// HDC CSR part, entry-parallel (no per-row serial loop: an R-MAT hub row of
// ~10^5 entries used to cost one thread milliseconds).  keep[k] = the entry's
// diagonal count is below the threshold (formats.cpp:191); an exclusive scan
// of keep gives every kept entry its slot, which is also the stable per-row
// compaction because entries are in row order; row_ptr[i] = pos[rp[i]].
struct KeepFlag : OpBase {
    const int32_t* col;
    const int32_t* bins;
    int64_t nrows, thr;
    int32_t* keep;
    __device__ void operator()(int r, int64_t k, bool valid) const {
        if (valid) keep[k] = bins[int64_t(col[k]) - r + nrows - 1] < thr ? 1 : 0;
    }
};

// entries on diagonals below the threshold = the CSR part's size
__global__ void hdc_rest_total(const int32_t* __restrict__ bins, int64_t nbins, int64_t thr,
                               unsigned long long* __restrict__ total) {
    unsigned long long t = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nbins; i += int64_t(gridDim.x) * blockDim.x)
        if (bins[i] < thr) t += unsigned(bins[i]);
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(total, t);
}

__global__ void hdc_rest_rowptr(const int64_t* __restrict__ rp, const int64_t* __restrict__ pos, int64_t nrows,
                                int64_t* __restrict__ orp) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i <= nrows) orp[i] = pos[rp[i]];
}

__global__ void hdc_rest_fill(const int32_t* __restrict__ keep, const int64_t* __restrict__ pos, int64_t z,
                              const int32_t* __restrict__ col, const double* __restrict__ val,
                              int32_t* __restrict__ ocol, double* __restrict__ oval) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < z && keep[k]) {
        ocol[pos[k]] = col[k];
        oval[pos[k]] = val[k];
    }
}

// ------------------------------------------------------------ to CSR (any)

struct RowOfEntry : OpBase {
    int32_t* row;
    __device__ void operator()(int r, int64_t k, bool valid) const {
        if (valid) row[k] = r;
    }
};

__global__ void dia_row_counts(int64_t nrows, int64_t ncols, int ndiags, const int64_t* __restrict__ off,
                               const double* __restrict__ vals, int64_t* __restrict__ cnt, bool accumulate) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    int64_t c = 0;
    for (int d = 0; d < ndiags; ++d) {
        const int64_t j = i + off[d];
        if (j >= 0 && j < ncols && vals[int64_t(d) * nrows + i] != 0.0) ++c;
    }
    cnt[i] = accumulate ? cnt[i] + c : c;
}

__global__ void ell_row_counts(int64_t nrows, int64_t width, const int32_t* __restrict__ ecol,
                               int64_t* __restrict__ cnt) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    int64_t c = 0;
    while (c < width && ecol[c * nrows + i] != -1) ++c;
    cnt[i] = c;
}

__global__ void csr_row_counts(const int64_t* __restrict__ rp, int64_t nrows, int64_t* __restrict__ cnt,
                               bool accumulate) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    const int64_t c = rp[i + 1] - rp[i];
    cnt[i] = accumulate ? cnt[i] + c : c;
}

__global__ void coo_row_counts_atomic(const int32_t* __restrict__ row, int64_t z,
                                      unsigned long long* __restrict__ cnt) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= z) return;
    atomicAdd(cnt + row[k], 1ull);
}

// Entries of DIA cells (nonzero, in range) of row i, appended at rp[i]+fill[i].
__global__ void dia_to_rows(int64_t nrows, int64_t ncols, int ndiags, const int64_t* __restrict__ off,
                            const double* __restrict__ vals, const int64_t* __restrict__ rp,
                            int64_t* __restrict__ fill, int32_t* __restrict__ ocol, double* __restrict__ oval) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    int64_t p = rp[i] + fill[i];
    for (int d = 0; d < ndiags; ++d) {
        const int64_t j = i + off[d];
        if (j < 0 || j >= ncols) continue;
        const double v = vals[int64_t(d) * nrows + i];
        if (v != 0.0) {  // formats.cpp:225: holes and padding are skipped
            ocol[p] = int32_t(j);
            oval[p] = v;
            ++p;
        }
    }
    fill[i] = p - rp[i];
}

__global__ void ell_to_rows(int64_t nrows, int64_t width, const int32_t* __restrict__ ecol,
                            const double* __restrict__ evals, const int64_t* __restrict__ rp,
                            int64_t* __restrict__ fill, int32_t* __restrict__ ocol, double* __restrict__ oval) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    int64_t p = rp[i] + fill[i];
    for (int64_t k = 0; k < width; ++k) {
        const int32_t c = ecol[k * nrows + i];
        if (c == -1) break;  // formats.cpp:234
        ocol[p] = c;
        oval[p] = evals[k * nrows + i];
        ++p;
    }
    fill[i] = p - rp[i];
}

__global__ void csr_to_rows(int64_t nrows, const int64_t* __restrict__ srp, const int32_t* __restrict__ scol,
                            const double* __restrict__ sval, const int64_t* __restrict__ rp,
                            int64_t* __restrict__ fill, int32_t* __restrict__ ocol, double* __restrict__ oval) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    int64_t p = rp[i] + fill[i];
    for (int64_t k = srp[i]; k < srp[i + 1]; ++k) {
        ocol[p] = scol[k];
        oval[p] = sval[k];
        ++p;
    }
    fill[i] = p - rp[i];
}

__global__ void coo_to_rows(int64_t z, const int32_t* __restrict__ row, const int32_t* __restrict__ col,
                            const double* __restrict__ val, const int64_t* __restrict__ rp,
                            unsigned long long* __restrict__ fill, int32_t* __restrict__ ocol,
                            double* __restrict__ oval) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= z) return;
    const int32_t r = row[k];
    const int64_t p = rp[r] + int64_t(atomicAdd(fill + r, 1ull));
    ocol[p] = col[k];
    oval[p] = val[k];
}

// Per-row sortedness check + insertion sort of unsorted rows (to_coo's
// std::sort, formats.cpp:247-265).  Valid containers are already sorted;
// this only runs on rows assembled from several parts (HDC, HYB) or on
// user-mutated host arrays.
__global__ void sort_rows(const int64_t* __restrict__ rp, int64_t nrows, int32_t* __restrict__ col,
                          double* __restrict__ val) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    const int64_t a = rp[i], e = rp[i + 1];
    bool sorted = true;
    for (int64_t k = a + 1; k < e && sorted; ++k) sorted = col[k - 1] <= col[k];
    if (sorted) return;
    for (int64_t k = a + 1; k < e; ++k) {
        const int32_t c = col[k];
        const double v = val[k];
        int64_t j = k - 1;
        while (j >= a && col[j] > c) {
            col[j + 1] = col[j];
            val[j + 1] = val[j];
            --j;
        }
        col[j + 1] = c;
        val[j + 1] = v;
    }
}

// ------------------------------------------------------------ helpers

so_matrix* new_matrix(const so_matrix& like, int32_t fmt) {
    auto* m = new so_matrix();
    m->device = like.device;
    m->format = fmt;
    m->nrows = like.nrows;
    m->ncols = like.ncols;
    return m;
}

unsigned long long reduce_max_len(const so_matrix& csr, int64_t cap_at, cudaStream_t s) {
    DBuf<unsigned long long> out(1, s);
    SOB_CUDA(cudaMemsetAsync(out.get(), 0, sizeof(unsigned long long), s));
    if (csr.nrows > 0) {
        row_len_max<<<grid_for(csr.nrows, 256), 256, 0, s>>>(csr.csr.row_ptr.get(), csr.nrows, cap_at, out.get());
        SOB_LAUNCH("row_len_max");
    }
    return d2h_scalar(out.get(), s);
}

// Distinct flagged keys -> ascending offsets.  Returns ndiags; pos holds the
// key -> slot map (exclusive scan of flags).
int64_t compact_keys(const DBuf<int32_t>& flag, int64_t nkeys, int64_t nrows, DBuf<int64_t>& pos,
                     DBuf<int64_t>& offsets, int64_t cap, cudaStream_t s) {
    pos.alloc(nkeys + 1, s);
    exclusive_scan_i32_to_i64(flag.get(), pos.get(), nkeys, s);
    const int64_t nd = d2h_scalar(pos.get() + nkeys, s);
    check_cap(checked_mul(nd, nrows), cap, "DIA");  // formats.cpp:81-82, before allocation
    offsets.alloc(nd, s);
    if (nd > 0) {
        keys_to_offsets<<<unsigned(ceil_div(nkeys, 256)), 256, 0, s>>>(flag.get(), pos.get(), nkeys, nrows,
                                                                       offsets.get());
        SOB_LAUNCH("keys_to_offsets");
    }
    return nd;
}

// Diagonal histogram of a CSR into dense bins (shared-memory hash,
// row-lockstep sweep: banded rows aggregate to one update per warp).
void diag_histogram(const so_matrix& csr, int32_t* bins, cudaStream_t s) {
    DiagHist dh;
    dh.col = csr.csr.col.get();
    dh.nrows = csr.nrows;
    dh.bins = bins;
    row_sweep_launch(csr, dh, s, /*prefetch_cols=*/true);
}

void build_dia_part(const so_matrix& csr, const int32_t* bins_in, int64_t thr, DiaPart& dia, int64_t cap,
                    cudaStream_t s) {
    const int64_t n = csr.nrows;
    const int64_t nkeys = (n > 0 && csr.ncols > 0) ? n + csr.ncols - 1 : 0;
    DBuf<int32_t> own_bins;
    const int32_t* bins = bins_in;
    if (!bins && nkeys) {
        own_bins.alloc(n + csr.ncols, s);
        SOB_CUDA(cudaMemsetAsync(own_bins.get(), 0, own_bins.bytes(), s));
        diag_histogram(csr, own_bins.get(), s);
        bins = own_bins.get();
    }
    DBuf<int32_t> flag(nkeys, s);
    if (nkeys) {
        bins_to_flags<<<unsigned(ceil_div(nkeys, 256)), 256, 0, s>>>(bins, nkeys, thr, flag.get());
        SOB_LAUNCH("bins_to_flags");
    }
    DBuf<int64_t> pos;
    dia.ndiags = compact_keys(flag, nkeys, n, pos, dia.offsets, cap, s);
    dia.values.alloc(dia.ndiags * n, s);
    if (dia.values.n) SOB_CUDA(cudaMemsetAsync(dia.values.get(), 0, dia.values.bytes(), s));
    DBuf<unsigned long long> stored(1, s);
    SOB_CUDA(cudaMemsetAsync(stored.get(), 0, sizeof(unsigned long long), s));
    FillDia fd;
    fd.col = csr.csr.col.get();
    fd.val = csr.csr.val.get();
    fd.nrows = n;
    fd.pos = pos.get();
    fd.bins = bins_in;  // HDC: only entries on true diagonals go to the DIA part
    fd.thr = thr;
    fd.values = dia.values.get();
    fd.stored = stored.get();
    if (dia.ndiags > 0) row_sweep_launch(csr, fd, s);
    dia.stored_nnz = int64_t(d2h_scalar(stored.get(), s));
}

void fill_ell_part(const so_matrix& csr, int64_t width, EllPart& ell, cudaStream_t s) {
    const int64_t n = csr.nrows;
    ell.width = width;
    ell.col.alloc(width * n, s);
    ell.val.alloc(width * n, s);
    if (width * n > 0) {
        ell_fill<<<grid_for(n, 256), 256, 0, s>>>(csr.csr.row_ptr.get(), csr.csr.col.get(),
                                                          csr.csr.val.get(), n, width, ell.col.get(),
                                                          ell.val.get());
        SOB_LAUNCH("ell_fill");
    }
}

}  // namespace

// ======================================================== public (internal)

void build_row_blocks(CsrPart& csr, int64_t n, cudaStream_t s) {
    if (n <= 0) {
        csr.nblk = 0;
        csr.ngrp = 0;
        csr.ncoop = 0;
        csr.nlong = 0;
        csr.npieces = 0;
        csr.blk.alloc(1, s);
        csr.blk_k.alloc(1, s);
        SOB_CUDA(cudaMemsetAsync(csr.blk.get(), 0, sizeof(int32_t), s));
        SOB_CUDA(cudaMemsetAsync(csr.blk_k.get(), 0, sizeof(int64_t), s));
        return;
    }
    DBuf<int32_t> flag(n, s);
    DBuf<int64_t> pos(n + 1, s);
    row_block_flags<<<unsigned(ceil_div(n, 256)), 256, 0, s>>>(csr.row_ptr.get(), n, flag.get());
    SOB_LAUNCH("row_block_flags");
    exclusive_scan_i32_to_i64(flag.get(), pos.get(), n, s);
    csr.nblk = d2h_scalar(pos.get() + n, s);
    csr.blk.alloc(csr.nblk + 1, s);
    csr.blk_k.alloc(csr.nblk + 1, s);
    row_block_scatter<<<unsigned(ceil_div(n + 1, 256)), 256, 0, s>>>(flag.get(), pos.get(), csr.row_ptr.get(), n,
                                                                     csr.blk.get(), csr.blk_k.get());
    SOB_LAUNCH("row_block_scatter");
    // SpMV warp groups; entries per lane follow the mean row length
    const int64_t nnz_total = d2h_scalar(csr.row_ptr.get() + n, s);
    csr.grp_cap = 32 * ((nnz_total <= 8 * n) ? kGroupItemsShort : kGroupItemsLong);
    group_flags<<<unsigned(ceil_div(ceil_div(n, kGroupChunk), kGroupWarps)), 32 * kGroupWarps, 0, s>>>(
        csr.row_ptr.get(), n, csr.grp_cap, flag.get());
    SOB_LAUNCH("group_flags");
    exclusive_scan_i32_to_i64(flag.get(), pos.get(), n, s);
    csr.ngrp = d2h_scalar(pos.get() + n, s);
    csr.grp.alloc(csr.ngrp + 1, s);
    csr.grp_k.alloc(csr.ngrp + 1, s);
    row_block_scatter<<<unsigned(ceil_div(n + 1, 256)), 256, 0, s>>>(flag.get(), pos.get(), csr.row_ptr.get(), n,
                                                                     csr.grp.get(), csr.grp_k.get());
    SOB_LAUNCH("row_block_scatter");
    csr.npad = 0;
    csr.ncoop = 0;
    csr.grp_rpl = 1;
    if (csr.ngrp > 0) {
        // the counter lives in the (free until long_row_flags) flag scratch:
        // no allocation between the matrix arrays
        unsigned long long* npad = reinterpret_cast<unsigned long long*>(pos.get());
        SOB_CUDA(cudaMemsetAsync(npad, 0, 2 * sizeof(unsigned long long), s));
        const unsigned g = unsigned(ceil_div(csr.ngrp * 32, 256));
        group_pad_flags<false><<<g, 256, 0, s>>>(csr.grp.get(), csr.grp_k.get(), csr.ngrp, csr.row_ptr.get(),
                                                 csr.grp_cap, npad);
        SOB_LAUNCH("group_pad_flags");
        unsigned long long cnt[2];
        SOB_CUDA(cudaMemcpyAsync(cnt, npad, sizeof(cnt), cudaMemcpyDeviceToHost, s));
        SOB_CUDA(cudaStreamSynchronize(s));
        csr.npad = int64_t(cnt[0]);
        csr.grp_rpl = cnt[1] > 0 ? kGroupRowsMax / 32 : 1;
        if (csr.npad * kGrpPadShare >= csr.ngrp) {
            group_pad_flags<true><<<g, 256, 0, s>>>(csr.grp.get(), csr.grp_k.get(), csr.ngrp, csr.row_ptr.get(),
                                                    csr.grp_cap, npad);
            SOB_LAUNCH("group_pad_flags");
        } else {
            csr.npad = 0;  // too few to pay for the padded kernel: plain layout everywhere
        }
        SOB_CUDA(cudaMemsetAsync(npad, 0, sizeof(unsigned long long), s));
        count_coop_rows<<<unsigned(ceil_div(n, 256)), 256, 0, s>>>(csr.row_ptr.get(), n, csr.grp_cap, npad);
        SOB_LAUNCH("count_coop_rows");
        csr.ncoop = int64_t(d2h_scalar(npad, s));
    }
    // long rows -> kPiece-entry pieces (SpMV splits them over many CTAs)
    long_row_flags<<<unsigned(ceil_div(n, 256)), 256, 0, s>>>(csr.row_ptr.get(), n, int64_t(csr.grp_cap),
                                                              flag.get());
    SOB_LAUNCH("long_row_flags");
    exclusive_scan_i32_to_i64(flag.get(), pos.get(), n, s);
    csr.nlong = d2h_scalar(pos.get() + n, s);
    csr.npieces = 0;
    if (csr.nlong > 0) {
        csr.long_row.alloc(csr.nlong, s);
        DBuf<int64_t> npc(csr.nlong, s);
        long_row_list<<<unsigned(ceil_div(n, 256)), 256, 0, s>>>(csr.row_ptr.get(), flag.get(), pos.get(), n,
                                                                 csr.long_row.get(), npc.get());
        SOB_LAUNCH("long_row_list");
        csr.long_piece.alloc(csr.nlong + 1, s);
        exclusive_scan_i64(npc.get(), csr.long_piece.get(), csr.nlong, s);
        csr.npieces = d2h_scalar(csr.long_piece.get() + csr.nlong, s);
        csr.piece_k.alloc(2 * csr.npieces, s);
        long_row_pieces<<<unsigned(ceil_div(csr.nlong, 128)), 128, 0, s>>>(
            csr.row_ptr.get(), csr.long_row.get(), csr.long_piece.get(), csr.nlong, csr.piece_k.get());
        SOB_LAUNCH("long_row_pieces");
    }
}

bool coo_is_canonical(const so_matrix& coo, cudaStream_t s) {  // formats.cpp:324-340
    if (coo.coo.nnz <= 1) return true;
    DBuf<int> bad(1, s);
    SOB_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    coo_canonical_check<<<unsigned(ceil_div(coo.coo.nnz - 1, 256)), 256, 0, s>>>(
        coo.coo.row.get(), coo.coo.col.get(), coo.coo.nnz, bad.get());
    SOB_LAUNCH("coo_canonical_check");
    return d2h_scalar(bad.get(), s) == 0;
}

so_matrix* coo_to_csr_device(const so_matrix& coo, cudaStream_t s) {  // formats.cpp:45-60
    auto* m = new_matrix(coo, SO_CSR);
    const int64_t z = coo.coo.nnz, n = coo.nrows;
    CsrPart& c = m->csr;
    c.nnz = z;
    c.row_ptr.alloc(n + 1, s);
    c.col.alloc(z, s);
    c.val.alloc(z, s);
    if (z) {
        SOB_CUDA(cudaMemcpyAsync(c.col.get(), coo.coo.col.get(), c.col.bytes(), cudaMemcpyDeviceToDevice, s));
        SOB_CUDA(cudaMemcpyAsync(c.val.get(), coo.coo.val.get(), c.val.bytes(), cudaMemcpyDeviceToDevice, s));
    }
    coo_row_ptr<<<unsigned(ceil_div(z + 1, 256)), 256, 0, s>>>(coo.coo.row.get(), z, n, c.row_ptr.get());
    SOB_LAUNCH("coo_row_ptr");
    c.canonical = 1;  // from canonical COO
    build_row_blocks(c, n, s);
    return m;
}

so_matrix* csr_to_coo(const so_matrix& csr, cudaStream_t s) {
    auto* m = new_matrix(csr, SO_COO);
    const int64_t z = csr.csr.nnz;
    CooPart& c = m->coo;
    c.nnz = z;
    c.row.alloc(z, s);
    c.col.alloc(z, s);
    c.val.alloc(z, s);
    if (z) {
        SOB_CUDA(cudaMemcpyAsync(c.col.get(), csr.csr.col.get(), c.col.bytes(), cudaMemcpyDeviceToDevice, s));
        SOB_CUDA(cudaMemcpyAsync(c.val.get(), csr.csr.val.get(), c.val.bytes(), cudaMemcpyDeviceToDevice, s));
        RowOfEntry op;
        op.row = c.row.get();
        sweep(csr, op, s);
    }
    return m;
}

so_matrix* clone_matrix(const so_matrix& src, cudaStream_t s) {
    auto* m = new_matrix(src, src.format);
    auto cp = [&](auto& dst, const auto& from) {
        dst.alloc(from.n, s);
        if (from.n) SOB_CUDA(cudaMemcpyAsync(dst.get(), from.get(), from.bytes(), cudaMemcpyDeviceToDevice, s));
    };
    m->coo.nnz = src.coo.nnz;
    cp(m->coo.row, src.coo.row);
    cp(m->coo.col, src.coo.col);
    cp(m->coo.val, src.coo.val);
    m->csr.nnz = src.csr.nnz;
    m->csr.nblk = src.csr.nblk;
    cp(m->csr.row_ptr, src.csr.row_ptr);
    cp(m->csr.col, src.csr.col);
    cp(m->csr.val, src.csr.val);
    cp(m->csr.blk, src.csr.blk);
    cp(m->csr.blk_k, src.csr.blk_k);
    m->csr.canonical.store(src.csr.canonical.load());
    m->csr.ngrp = src.csr.ngrp;
    m->csr.grp_cap = src.csr.grp_cap;
    cp(m->csr.grp, src.csr.grp);
    cp(m->csr.grp_k, src.csr.grp_k);
    m->csr.npad = src.csr.npad;
    m->csr.ncoop = src.csr.ncoop;
    m->csr.grp_rpl = src.csr.grp_rpl;
    m->csr.nlong = src.csr.nlong;
    m->csr.npieces = src.csr.npieces;
    cp(m->csr.long_row, src.csr.long_row);
    cp(m->csr.long_piece, src.csr.long_piece);
    cp(m->csr.piece_k, src.csr.piece_k);
    m->dia.ndiags = src.dia.ndiags;
    m->dia.stored_nnz = src.dia.stored_nnz;
    cp(m->dia.offsets, src.dia.offsets);
    cp(m->dia.values, src.dia.values);
    m->ell.width = src.ell.width;
    m->ell.stored_nnz = src.ell.stored_nnz;
    cp(m->ell.col, src.ell.col);
    cp(m->ell.val, src.ell.val);
    m->kh = src.kh;
    m->threshold = src.threshold;
    return m;
}

so_matrix* csr_to_format(const so_matrix& csr, int32_t target, const so_conversion_config& cfg, cudaStream_t s) {
    const int64_t n = csr.nrows, z = csr.csr.nnz;
    const int64_t cap = padded_entry_cap(cfg, z);  // formats.cpp:414
    switch (target) {
        case SO_COO:
            return csr_to_coo(csr, s);
        case SO_CSR:
            return clone_matrix(csr, s);
        case SO_DIA: {  // formats.cpp:98-105
            std::unique_ptr<so_matrix> m(new_matrix(csr, SO_DIA));
            build_dia_part(csr, nullptr, 0, m->dia, cap, s);
            return m.release();
        }
        case SO_ELL: {  // formats.cpp:132-138
            const int64_t width = int64_t(reduce_max_len(csr, -1, s));
            check_cap(checked_mul(width, n), cap, "ELL");
            std::unique_ptr<so_matrix> m(new_matrix(csr, SO_ELL));
            fill_ell_part(csr, width, m->ell, s);
            m->ell.stored_nnz = z;
            return m.release();
        }
        case SO_HYB: {  // formats.cpp:140-172
            const int64_t kh = effective_kh(cfg, z, n);
            const int64_t width = int64_t(reduce_max_len(csr, kh, s));
            check_cap(checked_mul(width, n), cap, "ELL");
            std::unique_ptr<so_matrix> m(new_matrix(csr, SO_HYB));
            m->kh = kh;
            fill_ell_part(csr, width, m->ell, s);
            DBuf<int64_t> cnt(n, s), off(n + 1, s);
            if (n) {
                hyb_surplus<<<unsigned(ceil_div(n, 256)), 256, 0, s>>>(csr.csr.row_ptr.get(), n, kh, cnt.get());
                SOB_LAUNCH("hyb_surplus");
            }
            exclusive_scan_i64(cnt.get(), off.get(), n, s);
            const int64_t zc = d2h_scalar(off.get() + n, s);
            m->ell.stored_nnz = z - zc;
            CooPart& c = m->coo;
            c.nnz = zc;
            c.row.alloc(zc, s);
            c.col.alloc(zc, s);
            c.val.alloc(zc, s);
            if (zc) {
                FillHybCoo op;
                op.rp = csr.csr.row_ptr.get();
                op.col = csr.csr.col.get();
                op.val = csr.csr.val.get();
                op.kh = kh;
                op.coo_off = off.get();
                op.crow = c.row.get();
                op.ccol = c.col.get();
                op.cval = c.val.get();
                sweep(csr, op, s);
            }
            return m.release();
        }
        case SO_HDC: {  // formats.cpp:174-205
            const int64_t thr = true_diag_threshold(cfg.true_diag_ratio, n, csr.ncols);
            std::unique_ptr<so_matrix> m(new_matrix(csr, SO_HDC));
            m->threshold = thr;
            const int64_t nbins = n + csr.ncols;
            DBuf<int32_t> bins(nbins, s);
            if (nbins) SOB_CUDA(cudaMemsetAsync(bins.get(), 0, bins.bytes(), s));
            diag_histogram(csr, bins.get(), s);
            // entries on diagonals with count >= thr go to the DIA part
            build_dia_part(csr, bins.get(), thr, m->dia, cap, s);
            CsrPart& c = m->csr;
            const int64_t z = csr.csr.nnz;
            c.row_ptr.alloc(n + 1, s);
            // banded / stencil inputs: every entry is on a true diagonal -> empty CSR part
            DBuf<unsigned long long> rest(1, s);
            SOB_CUDA(cudaMemsetAsync(rest.get(), 0, sizeof(unsigned long long), s));
            if (nbins) {
                hdc_rest_total<<<grid_for(nbins, 256), 256, 0, s>>>(bins.get(), nbins, thr, rest.get());
                SOB_LAUNCH("hdc_rest_total");
            }
            const int64_t rest_total = int64_t(d2h_scalar(rest.get(), s));
            if (rest_total == 0) {
                SOB_CUDA(cudaMemsetAsync(c.row_ptr.get(), 0, c.row_ptr.bytes(), s));
                c.nnz = 0;
                c.col.alloc(0, s);
                c.val.alloc(0, s);
                build_row_blocks(c, n, s);
                return m.release();
            }
            // scattered inputs (R-MAT): no diagonal reaches the threshold, the
            // CSR part is the whole input -- copy it, no keep flags / compaction
            if (rest_total == z) {
                SOB_CUDA(cudaMemcpyAsync(c.row_ptr.get(), csr.csr.row_ptr.get(), c.row_ptr.bytes(),
                                         cudaMemcpyDeviceToDevice, s));
                c.nnz = z;
                c.col.alloc(z, s);
                c.val.alloc(z, s);
                SOB_CUDA(cudaMemcpyAsync(c.col.get(), csr.csr.col.get(), c.col.bytes(), cudaMemcpyDeviceToDevice, s));
                SOB_CUDA(cudaMemcpyAsync(c.val.get(), csr.csr.val.get(), c.val.bytes(), cudaMemcpyDeviceToDevice, s));
                c.canonical.store(csr.csr.canonical.load());
                build_row_blocks(c, n, s);
                return m.release();
            }
            DBuf<int32_t> keep(z, s);
            DBuf<int64_t> pos(z + 1, s);
            if (z > 0) {
                KeepFlag kf;
                kf.col = csr.csr.col.get();
                kf.bins = bins.get();
                kf.nrows = n;
                kf.thr = thr;
                kf.keep = keep.get();
                sweep(csr, kf, s);
            }
            exclusive_scan_i32_to_i64(keep.get(), pos.get(), z, s);
            hdc_rest_rowptr<<<unsigned(ceil_div(n + 1, 256)), 256, 0, s>>>(csr.csr.row_ptr.get(), pos.get(), n,
                                                                          c.row_ptr.get());
            SOB_LAUNCH("hdc_rest_rowptr");
            c.nnz = d2h_scalar(pos.get() + z, s);
            c.col.alloc(c.nnz, s);
            c.val.alloc(c.nnz, s);
            if (c.nnz) {
                hdc_rest_fill<<<unsigned(ceil_div(z, 256)), 256, 0, s>>>(keep.get(), pos.get(), z,
                                                                       csr.csr.col.get(), csr.csr.val.get(),
                                                                       c.col.get(), c.val.get());
                SOB_LAUNCH("hdc_rest_fill");
            }
            build_row_blocks(c, n, s);
            return m.release();
        }
    }
    fail(SO_INVALID_INPUT, "unknown target format");
}

// to_coo semantics (formats.cpp:432-461) delivered as a canonical-order CSR.
so_matrix* any_to_csr(const so_matrix& m, cudaStream_t s) {
    const int64_t n = m.nrows;
    if (m.format == SO_COO) {
        // to_coo(COO) returns the payload unchanged; from_coo then demands
        // canonical input (formats.cpp:22-26).
        if (!coo_is_canonical(m, s)) fail(SO_INVALID_INPUT, "from_coo: source matrix is not canonical COO");
        return coo_to_csr_device(m, s);
    }
    std::unique_ptr<so_matrix> out(new_matrix(m, SO_CSR));
    CsrPart& c = out->csr;
    DBuf<int64_t> cnt(n, s);
    auto grid = unsigned(ceil_div(n, 256));
    const bool need_sort = true;  // cheap when rows are already sorted
    if (n > 0) {
        switch (m.format) {
            case SO_CSR:
                csr_row_counts<<<grid, 256, 0, s>>>(m.csr.row_ptr.get(), n, cnt.get(), false);
                break;
            case SO_DIA:
                dia_row_counts<<<grid, 256, 0, s>>>(n, m.ncols, int(m.dia.ndiags), m.dia.offsets.get(),
                                                    m.dia.values.get(), cnt.get(), false);
                break;
            case SO_ELL:
            case SO_HYB:
                ell_row_counts<<<grid, 256, 0, s>>>(n, m.ell.width, m.ell.col.get(), cnt.get());
                if (m.format == SO_HYB && m.coo.nnz) {
                    SOB_LAUNCH("ell_row_counts");
                    coo_row_counts_atomic<<<unsigned(ceil_div(m.coo.nnz, 256)), 256, 0, s>>>(
                        m.coo.row.get(), m.coo.nnz, reinterpret_cast<unsigned long long*>(cnt.get()));
                }
                break;
            case SO_HDC:
                dia_row_counts<<<grid, 256, 0, s>>>(n, m.ncols, int(m.dia.ndiags), m.dia.offsets.get(),
                                                    m.dia.values.get(), cnt.get(), false);
                SOB_LAUNCH("dia_row_counts");
                csr_row_counts<<<grid, 256, 0, s>>>(m.csr.row_ptr.get(), n, cnt.get(), true);
                break;
        }
        SOB_LAUNCH("row counts");
    }
    c.row_ptr.alloc(n + 1, s);
    exclusive_scan_i64(cnt.get(), c.row_ptr.get(), n, s);
    c.nnz = d2h_scalar(c.row_ptr.get() + n, s);
    c.col.alloc(c.nnz, s);
    c.val.alloc(c.nnz, s);
    if (c.nnz > 0) {
        DBuf<int64_t> fill(n, s);
        SOB_CUDA(cudaMemsetAsync(fill.get(), 0, fill.bytes(), s));
        switch (m.format) {
            case SO_CSR:
                csr_to_rows<<<grid, 256, 0, s>>>(n, m.csr.row_ptr.get(), m.csr.col.get(), m.csr.val.get(),
                                                 c.row_ptr.get(), fill.get(), c.col.get(), c.val.get());
                break;
            case SO_DIA:
                dia_to_rows<<<grid, 256, 0, s>>>(n, m.ncols, int(m.dia.ndiags), m.dia.offsets.get(),
                                                 m.dia.values.get(), c.row_ptr.get(), fill.get(), c.col.get(),
                                                 c.val.get());
                break;
            case SO_ELL:
            case SO_HYB:
                ell_to_rows<<<grid, 256, 0, s>>>(n, m.ell.width, m.ell.col.get(), m.ell.val.get(),
                                                 c.row_ptr.get(), fill.get(), c.col.get(), c.val.get());
                if (m.format == SO_HYB && m.coo.nnz) {
                    SOB_LAUNCH("ell_to_rows");
                    coo_to_rows<<<unsigned(ceil_div(m.coo.nnz, 256)), 256, 0, s>>>(
                        m.coo.nnz, m.coo.row.get(), m.coo.col.get(), m.coo.val.get(), c.row_ptr.get(),
                        reinterpret_cast<unsigned long long*>(fill.get()), c.col.get(), c.val.get());
                }
                break;
            case SO_HDC:
                dia_to_rows<<<grid, 256, 0, s>>>(n, m.ncols, int(m.dia.ndiags), m.dia.offsets.get(),
                                                 m.dia.values.get(), c.row_ptr.get(), fill.get(), c.col.get(),
                                                 c.val.get());
                SOB_LAUNCH("dia_to_rows");
                csr_to_rows<<<grid, 256, 0, s>>>(n, m.csr.row_ptr.get(), m.csr.col.get(), m.csr.val.get(),
                                                 c.row_ptr.get(), fill.get(), c.col.get(), c.val.get());
                break;
        }
        SOB_LAUNCH("to rows");
        if (need_sort) {
            sort_rows<<<grid, 256, 0, s>>>(c.row_ptr.get(), n, c.col.get(), c.val.get());
            SOB_LAUNCH("sort_rows");
        }
    }
    build_row_blocks(c, n, s);
    return out.release();
}

// ------------------------------------------------------------ CSR checks

namespace {
}  // namespace

struct UnsortedOp : OpBase {
    const int64_t* rp;
    const int32_t* col;
    int* bad;
    __device__ void operator()(int r, int64_t k, bool valid) const {
        if (valid && k > __ldg(rp + r) && __ldg(col + k - 1) >= __ldg(col + k)) *bad = 1;
    }
};

// strictly increasing columns in every row: the CSR already is to_coo's
// canonical order and can feed conversions without a copy (cached per matrix)
bool csr_rows_canonical(const so_matrix& m, cudaStream_t s) {
    if (m.csr.nnz <= 1) return true;
    if (m.csr.canonical >= 0) return m.csr.canonical == 1;
    DBuf<int> bad(1, s);
    SOB_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    UnsortedOp op;
    op.rp = m.csr.row_ptr.get();
    op.col = m.csr.col.get();
    op.bad = bad.get();
    row_sweep_launch(m, op, s);
    m.csr.canonical = d2h_scalar(bad.get(), s) == 0 ? 1 : 0;
    return m.csr.canonical == 1;
}

// ------------------------------------------------------------ generators

namespace {

__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// values[d * nloc + il] for the 27-point stencil slice; holes where the
// neighbour leaves the grid or the column window.
__global__ void stencil27_fill(int64_t g, int64_t row_lo, int64_t nloc, int64_t col_lo, int64_t col_hi,
                               uint64_t seed, double* __restrict__ vals, unsigned long long* __restrict__ stored) {
    int64_t cnt = 0;
    for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < 27 * nloc;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int d = int(idx / nloc);
        const int64_t il = idx - int64_t(d) * nloc;
        const int64_t i = row_lo + il;
        const int dz = d / 9 - 1, dy = (d / 3) % 3 - 1, dx = d % 3 - 1;
        const int64_t z = i / (g * g), y = (i / g) % g, x = i % g;
        const int64_t j = i + dz * g * g + dy * g + dx;
        const bool ok = z + dz >= 0 && z + dz < g && y + dy >= 0 && y + dy < g && x + dx >= 0 && x + dx < g &&
                        j >= col_lo && j < col_hi;
        double v = 0.0;
        if (ok) {
            const uint64_t h = splitmix(seed ^ splitmix(uint64_t(i) * 27 + uint64_t(d)));
            const double u = double(h >> 11) * 0x1.0p-53;
            v = 0.5 + 1.5 * u;
            if (h & 1) v = -v;
            ++cnt;
        }
        vals[idx] = v;
    }
    cnt = warp_sum(cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(stored, (unsigned long long)cnt);
}

}  // namespace

so_matrix* gen_stencil27_dia(int64_t g, int64_t row_lo, int64_t row_hi, int64_t col_lo, int64_t col_hi,
                             uint64_t seed, cudaStream_t s) {
    auto* m = new so_matrix();
    SOB_CUDA(cudaGetDevice(&m->device));
    m->format = SO_DIA;
    m->nrows = row_hi - row_lo;
    m->ncols = col_hi - col_lo;
    DiaPart& d = m->dia;
    d.ndiags = 27;
    std::vector<int64_t> off(27);
    for (int k = 0; k < 27; ++k)  // ascending: dz major, then dy, then dx
        off[size_t(k)] = (k / 9 - 1) * g * g + ((k / 3) % 3 - 1) * g + (k % 3 - 1) + (row_lo - col_lo);
    d.offsets.alloc(27, s);
    SOB_CUDA(cudaMemcpyAsync(d.offsets.get(), off.data(), 27 * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    d.values.alloc(27 * m->nrows, s);
    DBuf<unsigned long long> stored(1, s);
    SOB_CUDA(cudaMemsetAsync(stored.get(), 0, sizeof(unsigned long long), s));
    if (m->nrows > 0) {
        stencil27_fill<<<grid_for(27 * m->nrows, 256), 256, 0, s>>>(g, row_lo, m->nrows, col_lo, col_hi, seed,
                                                                     d.values.get(), stored.get());
        SOB_LAUNCH("stencil27_fill");
    }
    d.stored_nnz = int64_t(d2h_scalar(stored.get(), s));
    return m;
}

}  // namespace sob
