// The ten structural features (features.cpp:82-153) on the device.
//
// Pass 1 (one kernel per stored part, no conversion): per-row counts and the
// diagonal histogram, with shared-memory privatised bins (hist.cuh).  DIA
// parts count per diagonal directly (no dense bins).
// Pass 2: row statistics + per-chunk sums of squared deviations; N_D / N_TD
// over the bins.
// Pass 3: nnz_row_spread.  The reference sums (c_i - avg)^2 SEQUENTIALLY in
// row order (features.cpp:139-144); a parallel reduction lands closer to the
// exact value and misses the 1e-12 parity target by up to 1.7e-9.
// The "binade replay" below reproduces the sequential rounding bit-exactly:
// while the running sum S stays inside one binade [2^e, 2^(e+1)), fl(S+t)
// adds round(t / ulp) ulps, so a run of additions is an integer sum -- except
// at exact ties, where round-half-even depends on the parity of S.  Each
// element is therefore a function parity -> (ulp increment, parity); these
// compose associatively, so chunks are summarised in parallel and a single
// warp walks the chunk summaries, verifying every binade assumption exactly
// and recursing (32-way) into any chunk where S changes binade.  The result
// is the reference's double, not an approximation of it.
#include <cstdlib>
#include <cfloat>
#include <memory>
#include <mutex>

#include "features.cuh"
#include "hist.cuh"

namespace sob {

namespace {

constexpr int kB = 256;
constexpr int kMaxSpreadChunk = 8192;
constexpr int kSubs = 32;  // sub-chunks per spread chunk (one per lane of the walk)
// rows per spread chunk: a power of two in [1024, 8192] giving ~512 chunks,
// so big matrices keep the chunk walk short and small ones keep the exact
// slow path over their first chunk cheap
inline int64_t spread_chunk(int64_t n) {
    int64_t c = 1024;
    while (c < kMaxSpreadChunk && c * 512 < n) c *= 2;
    return c;
}
constexpr int kMaxSmemDiag = 1024;

// ------------------------------------------------------------ pass 1: scans

// CSR part: row counts from row_ptr, diagonal keys through the shared-memory
// hash with the row-lockstep sweep (hist.cuh): for banded rows every lane of a
// warp holds the same key at each step, so 32 updates merge into one.
template <bool ACCUM_RC>
struct FeatCsrOp {
    const int32_t* col;
    int64_t nrows;
    int32_t* rc;
    int32_t* bins;
    FeatState* st;
    SmemHash* h;
    unsigned long long visits;
    __device__ void begin() {
        __shared__ SmemHash sh;
        h = &sh;
        hash_init(sh);
        visits = 0;
        __syncthreads();
    }
    __device__ void row(int r, bool valid, int64_t len) {
        if (!valid) return;
        rc[r] = ACCUM_RC ? rc[r] + int(len) : int(len);
        visits += len;
    }
    __device__ void operator()(int r, int64_t k, bool valid) {
        hash_add(*h, bins, valid ? int32_t(int64_t(col[k]) - r + nrows - 1) : -1);
    }
    static constexpr bool kPieceDirect = true;  // piece_sweep (hist.cuh)
    __device__ void piece(int r, int64_t k, bool valid) {
        if (valid) atomicAdd(bins + (int64_t(col[k]) - r + nrows - 1), 1);
    }
    // all_direct (sweep mode 2, the tune plan's choice for matrices whose
    // keys barely repeat): every entry is a global atomic, no hash probing
    bool all_direct;
    __device__ bool scattered() const {
        return all_direct || __shfl_sync(0xffffffffu, h->used >= kHashSlots / 2, 0);
    }
    __device__ void direct(int r, int32_t c, bool valid) {
        if (!valid) return;
        const int32_t key = int32_t(int64_t(c) - r + nrows - 1);
        if (all_direct)
            atomicAdd(bins + key, 1);
        else
            hash_insert_one(*h, bins, key, 1);
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
        const unsigned long long v = warp_sum(visits);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&st->visits, v);
        cache.flush(*h, bins);
        __syncthreads();
        hash_flush(*h, bins);
    }
};

// Entry-parallel CSR sweep for small matrices (fewer than 16 row-lockstep
// warps per SM): the row blocks of the CSR partition (<= kRowsPerBlock rows,
// ~2*kWindow entries) with their row_ptr staged in shared memory, 256
// consecutive entries per step (one per thread), keys into the same shared
// hash.  The row-lockstep sweep gives such a matrix one warp per 32 rows, each
// a serial chain over its rows' entries (config-4 id 1762: 41 us for 359 K
// entries); here every thread of every block has independent work.  Covers
// long rows too, except rows longer than big_row (a block holding one such row
// would be one CTA's serial walk -- an arrow matrix's dense row is ~4K steps):
// their entries are left to piece_sweep, ~2K entries per CTA.
constexpr int64_t kBigRowPieces = 8;  // rows of more than 8 SpMV pieces (16 K entries)
template <bool ACCUM_RC>
__global__ void __launch_bounds__(kB)
    feat_csr_entries(const int32_t* __restrict__ blk, int64_t nblk, const int64_t* __restrict__ rp,
                     FeatCsrOp<ACCUM_RC> op, int64_t big_row) {
    pdl_enter();
    __shared__ int64_t srp[kRowsPerBlock + 1];
    op.begin();
    for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
        const int r0 = blk[b], nr = blk[b + 1] - r0;
        __syncthreads();
        for (int j = threadIdx.x; j <= nr; j += kB) srp[j] = rp[r0 + j];
        __syncthreads();
        for (int j = threadIdx.x; j < nr; j += kB) op.row(r0 + j, true, srp[j + 1] - srp[j]);
        // a row longer than kWindow stands alone in its block
        if (nr == 1 && srp[1] - srp[0] > big_row) continue;
        const int64_t k0 = srp[0], k1 = srp[nr];
        for (int64_t base = k0; base < k1; base += kB) {
            const int64_t k = base + threadIdx.x;
            const bool valid = k < k1;
            op(valid ? r0 + row_in_block(srp, nr, k) : -1, k, valid);
        }
    }
    op.end();
}

__global__ void __launch_bounds__(kB)
    feat_coo(int64_t z, int64_t nrows, const int32_t* __restrict__ row, const int32_t* __restrict__ col,
             int32_t* __restrict__ rc, int32_t* __restrict__ bins, FeatState* __restrict__ st) {
    pdl_enter();
    __shared__ SmemHash h;
    hash_init(h);
    __syncthreads();
    const unsigned lane = threadIdx.x & 31u;
    for (int64_t base = int64_t(blockIdx.x) * kB; base < z; base += int64_t(gridDim.x) * kB) {
        const int64_t k = base + threadIdx.x;
        const bool valid = k < z;
        const int32_t r = valid ? row[k] : -2 - int32_t(lane);
        // warp-aggregated row counts (canonical rows are sorted => long runs)
        const unsigned peers = __match_any_sync(0xffffffffu, r);
        if (valid && int(lane) == __ffs(peers) - 1) atomicAdd(rc + r, __popc(peers));
        hash_add(h, bins, valid ? int32_t(int64_t(col[k]) - r + nrows - 1) : -1);
    }
    __syncthreads();
    hash_flush(h, bins);
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&st->visits, (unsigned long long)z);
}

__global__ void __launch_bounds__(kB)
    feat_ell(int64_t nrows, int width, const int32_t* __restrict__ ecol, int32_t* __restrict__ rc,
             int32_t* __restrict__ bins, FeatState* __restrict__ st) {
    pdl_enter();
    __shared__ SmemHash h;
    hash_init(h);
    __syncthreads();
    unsigned long long visits = 0, structure = 0;
    for (int64_t base = int64_t(blockIdx.x) * kB; base < nrows; base += int64_t(gridDim.x) * kB) {
        const int64_t i = base + threadIdx.x;
        bool done = i >= nrows;
        int cnt = 0;
        for (int k = 0; k < width; ++k) {
            if (!__any_sync(0xffffffffu, !done)) break;
            int32_t key = -1;
            if (!done) {
                const int32_t c = ecol[int64_t(k) * nrows + i];
                if (c == -1) {  // features.cpp:71-74: one sentinel probe per padded row
                    done = true;
                    ++structure;
                } else {
                    ++cnt;
                    key = int32_t(int64_t(c) - i + nrows - 1);
                }
            }
            hash_add(h, bins, key);
        }
        if (i < nrows) rc[i] = cnt;
        visits += cnt;
    }
    visits = warp_sum(visits);
    structure = warp_sum(structure);
    if ((threadIdx.x & 31) == 0) {
        if (visits) atomicAdd(&st->visits, visits);
        if (structure) atomicAdd(&st->structure, structure);
    }
    __syncthreads();
    hash_flush(h, bins);
}

// DIA: one thread per row, diagonals ascending; eight diagonals' cells are
// loaded before any is classified (in-bounds for every valid row, so the
// loads are unpredicated and issue back to back); per-diagonal entry counts
// are reduced warp (ballot) -> shared -> one global atomic per diagonal per CTA.
__global__ void __launch_bounds__(kB)
    feat_dia(int64_t nrows, int64_t ncols, int nd, const int64_t* __restrict__ off,
             const double* __restrict__ vals, int32_t* __restrict__ rc,
             unsigned long long* __restrict__ dcount, FeatState* __restrict__ st) {
    pdl_enter();
    __shared__ unsigned long long sdc[kMaxSmemDiag];
    __shared__ int64_t soff[kMaxSmemDiag];
    const int nsm = nd < kMaxSmemDiag ? nd : kMaxSmemDiag;
    for (int d = threadIdx.x; d < nsm; d += kB) {
        sdc[d] = 0;
        soff[d] = off[d];
    }
    __syncthreads();
    unsigned long long visits = 0, structure = 0;
    constexpr int U = 8;
    for (int64_t base = int64_t(blockIdx.x) * kB; base < nrows; base += int64_t(gridDim.x) * kB) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < nrows;
        const int64_t iv = valid ? i : nrows - 1;
        int cnt = 0;
        for (int d0 = 0; d0 < nd; d0 += U) {
            double v[U];
            bool inr[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int d = d0 + u < nd ? d0 + u : nd - 1;
                const int64_t j = iv + (d < kMaxSmemDiag ? soff[d] : off[d]);
                inr[u] = valid && d0 + u < nd && j >= 0 && j < ncols;
                v[u] = vals[int64_t(d) * nrows + iv];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool nz = inr[u] && v[u] != 0.0;  // features.cpp:57
                cnt += nz;
                structure += inr[u] && !nz;
                const unsigned b = __ballot_sync(0xffffffffu, nz);
                if ((threadIdx.x & 31) == 0 && b) {
                    const int d = d0 + u;
                    if (d < kMaxSmemDiag)
                        atomicAdd(&sdc[d], (unsigned long long)__popc(b));
                    else
                        atomicAdd(&dcount[d], (unsigned long long)__popc(b));
                }
            }
        }
        if (valid) rc[i] = cnt;
        visits += cnt;
    }
    visits = warp_sum(visits);
    structure = warp_sum(structure);
    if ((threadIdx.x & 31) == 0) {
        if (visits) atomicAdd(&st->visits, visits);
        if (structure) atomicAdd(&st->structure, structure);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < nsm; d += kB)
        if (sdc[d]) atomicAdd(&dcount[d], sdc[d]);
}

// HDC: fold the DIA part's per-diagonal counts into the dense bins.
__global__ void dcount_to_bins(const unsigned long long* __restrict__ dcount, const int64_t* __restrict__ off,
                               int nd, int64_t nrows, int32_t* __restrict__ bins) {
    pdl_enter();
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d < nd && dcount[d]) atomicAdd(bins + (off[d] + nrows - 1), int32_t(dcount[d]));
}

// ------------------------------------------------------ pass 2: statistics

__device__ __forceinline__ double sq_dev(int32_t c, double avg) {
    const double dev = __dsub_rn(double(c), avg);  // features.cpp:140
    return __dmul_rn(dev, dev);
}

__global__ void __launch_bounds__(kB)
    feat_rows(const int32_t* __restrict__ rc, int64_t nrows, int64_t chunk, FeatState* __restrict__ st,
              double* __restrict__ csum) {
    pdl_enter();
    const double avg = double(st->visits) / double(nrows);
    const int64_t base = int64_t(blockIdx.x) * chunk;
    int mx = 0, mn = INT32_MAX;
    double s = 0.0;
#pragma unroll 4
    for (int j = 0; j < chunk / kB; ++j) {
        const int64_t i = base + j * kB + threadIdx.x;
        if (i < nrows) {
            const int32_t c = rc[i];
            mx = c > mx ? c : mx;
            mn = c < mn ? c : mn;
            s += sq_dev(c, avg);
        }
    }
    mx = warp_max(mx);
    mn = warp_min(mn);
    s = warp_sum(s);
    __shared__ double ss[kB / 32];
    __shared__ int smx[kB / 32], smn[kB / 32];
    if ((threadIdx.x & 31) == 0) {
        ss[threadIdx.x >> 5] = s;
        smx[threadIdx.x >> 5] = mx;
        smn[threadIdx.x >> 5] = mn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kB / 32; ++w) {
            t += ss[w];
            mx = smx[w] > mx ? smx[w] : mx;
            mn = smn[w] < mn ? smn[w] : mn;
        }
        csum[blockIdx.x] = t;
        atomicMax(&st->max_row, mx);
        atomicMin(&st->min_row, mn);
    }
}

// counts >= 1 -> N_D, counts >= thr -> N_TD (features.cpp:146-151)
template <typename T>
__global__ void feat_bins(const T* __restrict__ bins, int64_t nbins, int64_t thr, FeatState* __restrict__ st) {
    pdl_enter();
    unsigned long long nd = 0, ntd = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nbins; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t c = int64_t(bins[i]);
        nd += c >= 1;
        ntd += c >= thr;
    }
    nd = warp_sum(nd);
    ntd = warp_sum(ntd);
    if ((threadIdx.x & 31) == 0) {
        if (nd) atomicAdd(&st->nd, nd);
        if (ntd) atomicAdd(&st->ntd, ntd);
    }
}

// ------------------------------------------------ pass 3: binade replay

// f: parity -> (ulp increment, parity).  p bit0 = out parity for in 0,
// bit1 = out parity for in 1.
struct Mono {
    long long a0, a1;
    int p;
};

__device__ __forceinline__ Mono mono_id() { return Mono{0, 0, 2}; }

__device__ __forceinline__ Mono mono_cat(const Mono& m, const Mono& n) {  // m first, then n
    const int r0 = m.p & 1, r1 = (m.p >> 1) & 1;
    Mono o;
    o.a0 = m.a0 + (r0 ? n.a1 : n.a0);
    o.a1 = m.a1 + (r1 ? n.a1 : n.a0);
    const int q0 = r0 ? (n.p >> 1) & 1 : n.p & 1;
    const int q1 = r1 ? (n.p >> 1) & 1 : n.p & 1;
    o.p = q0 | (q1 << 1);
    return o;
}

constexpr double kTwo53 = 9007199254740992.0;

// Exact power-of-two scaling and binade of a positive double without the
// library ldexp/ilogb call sequences (the binade walk is a serial chain of
// these); out-of-range cases fall back to the library.
__device__ __forceinline__ double scale2(double x, int k) {  // x * 2^k, exact
    if (k >= -1022 && k <= 1023) {
        const double p = __longlong_as_double((long long)(k + 1023) << 52);
        const double r = x * p;
        if (r == 0.0 || fabs(r) >= 2.2250738585072014e-308) return r;  // normal result: exact
    }
    return ldexp(x, k);
}
__device__ __forceinline__ int binade(double x) {  // ilogb for x > 0
    const int be = int((__double_as_longlong(x) >> 52) & 0x7ff);
    return be ? be - 1023 : ilogb(x);
}

// Element t added at binade e (ulp 2^(e-52)).  Returns false when t alone
// reaches the next binade (q >= 2^53).
__device__ __forceinline__ bool mono_elem(double t, int e, Mono& out) {
    if (t == 0.0) {
        out = mono_id();
        return true;
    }
    const double q = scale2(t, 52 - e);  // exact (power-of-two scaling)
    if (!(q < kTwo53)) return false;
    const double fl = floor(q);
    const double fr = q - fl;  // exact
    const long long k = (long long)fl;
    if (fr < 0.5) {
        out = Mono{k, k, int(k & 1) | (int((k + 1) & 1) << 1)};
    } else if (fr > 0.5) {
        const long long k1 = k + 1;
        out = Mono{k1, k1, int(k1 & 1) | (int((k1 + 1) & 1) << 1)};
    } else {  // tie: round half to even, depends on the parity of S
        out = Mono{k + (k & 1), k + ((k + 1) & 1), 0};
    }
    return true;
}

__device__ __forceinline__ Mono shfl_mono_down(const Mono& m, int o) {
    return Mono{__shfl_down_sync(0xffffffffu, m.a0, o), __shfl_down_sync(0xffffffffu, m.a1, o),
                __shfl_down_sync(0xffffffffu, m.p, o)};
}
__device__ __forceinline__ Mono shfl_mono_up(const Mono& m, int o) {
    return Mono{__shfl_up_sync(0xffffffffu, m.a0, o), __shfl_up_sync(0xffffffffu, m.a1, o),
                __shfl_up_sync(0xffffffffu, m.p, o)};
}
// No tie anywhere: the summary is "add k ulps" (a0 == a1) and the out parity
// is the in parity flipped by k's parity -- composition is integer addition.
__device__ __forceinline__ bool mono_canonical(const Mono& m) {
    return m.a0 == m.a1 && m.p == (int(m.a0 & 1) | (int((m.a0 + 1) & 1) << 1));
}

// ordered inclusive scan across the warp (ok: AND over lanes <= this one).
// When every lane is canonical (no exact ties: the usual case) it is a
// plain 64-bit add-scan, a tenth of the instructions of the general
// composition -- the walk is one warp's dependent chain, so instruction
// count is its time.
__device__ __forceinline__ Mono warp_scan_mono(Mono m, bool& ok) {
    const unsigned lane = threadIdx.x & 31u;
    if (__all_sync(0xffffffffu, mono_canonical(m))) {
        long long a = m.a0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, a, o);
            if (lane >= unsigned(o)) a += t;
        }
        const unsigned bad = __ballot_sync(0xffffffffu, !ok);
        const unsigned le = lane == 31u ? 0xffffffffu : ((2u << lane) - 1u);
        ok = (bad & le) == 0u;
        return Mono{a, a, int(a & 1) | (int((a + 1) & 1) << 1)};
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const Mono up = shfl_mono_up(m, o);
        const bool uok = __shfl_up_sync(0xffffffffu, ok, o);
        if (lane >= unsigned(o)) {
            m = mono_cat(up, m);
            ok = ok && uok;
        }
    }
    return m;
}

enum : int { kMonoSafe = 1, kMonoIdent = 2 };

struct MonoRec {
    long long a0, a1;
    int p;
    int e;
    int flags;
    int pad;
};

// exclusive prefix of the chunk sums (approximate S at chunk starts)
__global__ void __launch_bounds__(512) spread_prefix(const double* __restrict__ csum, int64_t nch,
                                                       double* __restrict__ P) {
    pdl_enter();
    __shared__ double wt[33];
    double carry = 0.0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t base = 0; base < nch; base += 512) {
        const int64_t i = base + threadIdx.x;
        const double v = i < nch ? csum[i] : 0.0;
        double inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double w = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += w;
        }
        if (lane == 31) wt[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            const double w = lane < 16 ? wt[lane] : 0.0;
            double wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double u = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += u;
            }
            if (lane < 16) wt[lane] = wi - w;
            if (lane == 15) wt[32] = wi;
        }
        __syncthreads();
        if (i < nch) P[i] = carry + wt[warp] + inc - v;
        carry += wt[32];
        __syncthreads();
    }
    if (threadIdx.x == 0) P[nch] = carry;
}

__device__ __forceinline__ MonoRec ident_rec() { return MonoRec{0, 0, 2, 0, kMonoIdent, 0}; }

// Two-level summaries.  Every chunk is cut into 32 sub-chunks of chunk/32
// rows (8 threads each); a sub-chunk is summarised at the binade its
// approximate prefix (P[c] + sums of the earlier sub-chunks) puts it in, the
// chunk record is the ordered product of its sub-chunk records when they all
// share one binade.  spread_walk descends to the sub-chunk records of a
// chunk it cannot take whole, so the exact row-by-row path only ever runs
// over the one sub-chunk where the running sum changes binade.
__device__ __forceinline__ void mono_chunk(int64_t c, const int32_t* __restrict__ rc, int64_t nrows, int64_t chunk,
                                           double avg, double csum_c, double P_c, MonoRec* __restrict__ rec,
                                           MonoRec* __restrict__ fine) {
    const int t = threadIdx.x, lane = t & 31;
    if (csum_c == 0.0) {  // every t == 0: identity at any binade
        if (t < kSubs) fine[c * kSubs + t] = ident_rec();
        if (t == 0) rec[c] = ident_rec();
        return;
    }
    __shared__ double sub_sum[kSubs];
    __shared__ double psub[kSubs + 1];
    __shared__ MonoRec fr[kSubs];
    const int rpt = int(chunk / kB);  // rows per thread; 8 threads per sub-chunk
    const int64_t base = c * chunk + int64_t(t) * rpt;
    double ps = 0.0;  // approximate (order is irrelevant for the guess)
    for (int j = 0; j < rpt; ++j)
        if (base + j < nrows) ps += sq_dev(rc[base + j], avg);
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
    if ((lane & 7) == 0) sub_sum[t >> 3] = ps;
    __syncthreads();
    if (t < 32) {
        const double v = sub_sum[lane];
        double inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double w = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += w;
        }
        psub[lane] = P_c + (inc - v);
        if (lane == 31) psub[kSubs] = P_c + inc;
    }
    __syncthreads();
    const int sj = t >> 3;
    const double lo = psub[sj], hi = psub[sj + 1];
    const bool zero = sub_sum[sj] == 0.0;  // sum of non-negative terms: all zero
    const bool safe = !zero && lo > 0.0 && binade(lo) == binade(hi);
    const int e = safe ? binade(lo) : 0;
    Mono m = mono_id();
    bool ok = safe;
    if (safe) {
        for (int j = 0; j < rpt && ok; ++j) {
            if (base + j < nrows) {
                Mono el;
                ok = mono_elem(sq_dev(rc[base + j], avg), e, el);
                if (ok) m = mono_cat(m, el);
            }
        }
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {  // ordered product over the 8 threads of the sub-chunk
        const Mono other = shfl_mono_down(m, o);
        const bool ook = __shfl_down_sync(0xffffffffu, ok, o);
        if ((lane & (2 * o - 1)) == 0) {
            m = mono_cat(m, other);
            ok = ok && ook;
        }
    }
    if ((lane & 7) == 0) {
        const MonoRec r = zero ? ident_rec() : MonoRec{m.a0, m.a1, m.p, e, ok ? kMonoSafe : 0, 0};
        fine[c * kSubs + sj] = r;
        fr[sj] = r;
    }
    __syncthreads();
    if (t == 0) {
        Mono acc = mono_id();
        int ce = INT32_MIN;
        bool cok = true;
        for (int j = 0; j < kSubs && cok; ++j) {
            const MonoRec& r = fr[j];
            if (r.flags & kMonoIdent) continue;
            if (!(r.flags & kMonoSafe) || (ce != INT32_MIN && r.e != ce)) cok = false;
            ce = r.e;
            acc = mono_cat(acc, Mono{r.a0, r.a1, r.p});
        }
        rec[c] = cok ? MonoRec{acc.a0, acc.a1, acc.p, ce, kMonoSafe, 0} : MonoRec{0, 0, 2, 0, 0, 0};
    }
    __syncthreads();  // fr / sub_sum are reused by the next call
}

__global__ void __launch_bounds__(kB)
    spread_mono(const int32_t* __restrict__ rc, int64_t nrows, int64_t chunk, const FeatState* __restrict__ st,
                const double* __restrict__ csum, const double* __restrict__ P, MonoRec* __restrict__ rec,
                MonoRec* __restrict__ fine) {
    pdl_enter();
    const int64_t c = blockIdx.x;
    const double avg = double(st->visits) / double(nrows);
    mono_chunk(c, rc, nrows, chunk, avg, csum[c], P[c], rec, fine);
}


// Plain sequential IEEE additions over rows [lo, hi), 32 rows per step: the
// lanes compute the terms, one lane runs the dependent add chain, and S is
// broadcast back (warp-uniform).
__device__ double seq_rows(double S, int64_t lo, int64_t hi, const int32_t* __restrict__ rc, double avg) {
    // lanes compute 32 terms into shared memory; lane 0 runs the dependent
    // add chain from there (loads issue ahead of the adds), then broadcasts
    __shared__ double tbuf[32];
    const unsigned lane = threadIdx.x & 31u;
    for (int64_t b = lo; b < hi; b += 32) {
        const int64_t i = b + lane;
        tbuf[lane] = i < hi ? sq_dev(rc[i], avg) : 0.0;
        __syncwarp();
        const int cnt = int(hi - b < 32 ? hi - b : 32);
        if (lane == 0) {
            double t[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) t[j] = tbuf[j];
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (j < cnt) S = __dadd_rn(S, t[j]);
        }
        S = __shfl_sync(0xffffffffu, S, 0);
        __syncwarp();
    }
    return S;
}

// The exact path over one sub-chunk (<= kMaxSpreadChunk / kSubs = 256 rows):
// plain sequential additions by one lane (~8 cycles each) -- cheaper than
// binade-replay rounds over so few rows.  Warp-cooperative call (all 32
// lanes, same arguments; the same S comes back in every lane).
static_assert(kMaxSpreadChunk / kSubs <= 256, "sub-chunks stay short enough for the sequential path");
__device__ double advance_exact(double S, int64_t lo, int64_t hi, const int32_t* __restrict__ rc, double avg) {
    return seq_rows(S, lo, hi, rc, avg);
}

// Apply records rec[0..nrec) in order to S, 32 at a time (one per lane):
// every record whose binade matches the exact running sum is folded in with
// one warp scan, verified to stay inside the binade; a record that cannot be
// taken whole goes to fallback(S, index).
template <class Fallback>
__device__ double walk_records(double S, const MonoRec* __restrict__ rec, int64_t nrec, Fallback fallback) {
    const unsigned lane = threadIdx.x & 31u;
    int64_t c = 0;
    int64_t pre_c = 0;  // group whose records sit in `nxt`
    MonoRec nxt = lane < nrec ? rec[lane] : ident_rec();
    while (c < nrec) {
        const int64_t ci = c + lane;
        MonoRec r = (pre_c == c) ? nxt : (ci < nrec ? rec[ci] : ident_rec());
        // prefetch the most likely next group (all 32 consumed) while this one is applied
        pre_c = c + 32;
        nxt = pre_c + lane < nrec ? rec[pre_c + lane] : ident_rec();
        const int eS = S > 0.0 ? binade(S) : INT32_MIN;
        const bool usable = ci < nrec && ((r.flags & kMonoIdent) || ((r.flags & kMonoSafe) && r.e == eS));
        const unsigned badm = __ballot_sync(0xffffffffu, !usable);
        int j = badm ? __ffs(badm) - 1 : 32;
        const int64_t remaining = nrec - c;
        if (j > remaining) j = int(remaining);
        if (j > 0) {
            Mono mm = (int(lane) < j) ? Mono{r.a0, r.a1, r.p} : mono_id();
            bool ok = true;
            Mono pre = warp_scan_mono(mm, ok);
            if (S == 0.0) {  // only identity records can be usable at S == 0
                c += j;
                continue;
            }
            const long long m = (long long)scale2(S, 52 - eS);
            const long long mi = m + ((m & 1) ? pre.a1 : pre.a0);
            const bool good = double(mi) < kTwo53 || int(lane) >= j;
            const unsigned bad = __ballot_sync(0xffffffffu, !good);
            const int f = bad ? __ffs(bad) - 1 : j;  // first record whose prefix leaves the binade
            if (f > 0) {
                const long long mf = __shfl_sync(0xffffffffu, mi, f - 1);
                S = scale2(double(mf), eS - 52);
            }
            c += f;
            if (f == j) continue;
        }
        S = fallback(S, c);
        c += 1;
    }
    return S;
}

// One warp walks the chunk records, descending into the sub-chunk records of
// a chunk it cannot take whole and to the exact row-by-row path only for the
// sub-chunk where S changes binade; then finalizes the FeatureVector
// (features.cpp:121-152).
__device__ __forceinline__ void walk_and_finalize(const int32_t* __restrict__ rc, int64_t nrows, int64_t ncols,
                                                  int64_t nch, int64_t chunk, const MonoRec* __restrict__ rec,
                                                  const MonoRec* __restrict__ fine, FeatState* __restrict__ st) {
    const unsigned lane = threadIdx.x & 31u;
#ifdef SOB_SPREAD_DEBUG
    unsigned long long dbg_t0;
    {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        dbg_t0 = gt;
    }
    unsigned long long dbg_exact_ns = 0, dbg_exact_n = 0;
#endif
    const double avg = double(st->visits) / double(nrows);
    const int64_t sub = chunk / kSubs;
    const double S = walk_records(0.0, rec, nch, [&](double S, int64_t c) {
        const int64_t r0 = c * chunk;
        const int64_t nsub = ceil_div(((r0 + chunk < nrows) ? r0 + chunk : nrows) - r0, sub);
        return walk_records(S, fine + c * kSubs, nsub, [&](double S, int64_t j) {
#ifdef SOB_SPREAD_DEBUG
            unsigned long long g0, g1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
            const int64_t lo = r0 + j * sub;
            const double S2 = advance_exact(S, lo, lo + sub < nrows ? lo + sub : nrows, rc, avg);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
            dbg_exact_ns += g1 - g0;
            ++dbg_exact_n;
            return S2;
#else
            const int64_t lo = r0 + j * sub;
            return advance_exact(S, lo, lo + sub < nrows ? lo + sub : nrows, rc, avg);
#endif
        });
    });
#ifdef SOB_SPREAD_DEBUG
    {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        if (lane == 0)
            printf("spread walk total %llu ns, %llu exact fallbacks %llu ns\n", gt - dbg_t0, dbg_exact_n, dbg_exact_ns);
    }
#endif
    if (lane == 0) {
        st->S = S;
        so_feature_vector& f = st->out;
        const int64_t z = int64_t(st->visits);
        f.nrows = nrows;
        f.ncols = ncols;
        f.nnz = z;
        f.avg_nnz_per_row = avg;
        f.density = double(z) / (double(nrows) * double(ncols));
        f.max_nnz_per_row = st->max_row;
        f.min_nnz_per_row = st->min_row;
        f.nnz_row_spread = S / double(nrows);
        f.ndiags = int64_t(st->nd);
        f.ntrue_diags = int64_t(st->ntd);
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        st->t_end = t;
    }
}

// The walk is one warp and a chain of dependent loads (records, then rows of
// the sub-chunks where S changes binade), ~5 L2 round trips per binade
// change.  When the row counts and both record levels fit in shared memory
// (matrices up to ~32K rows: the config-4 corpus starts at 10^4) the CTA
// first stages them there and warp 0 walks the staged copy -- same
// arithmetic, same order; larger matrices walk global memory.
constexpr int kWalkThreads = 512;
constexpr size_t kWalkSmem = 200 * 1024;

inline size_t walk_smem_bytes(int64_t nrows, int64_t nch) {
    return size_t(nch) * (kSubs + 1) * sizeof(MonoRec) + size_t(nrows) * sizeof(int32_t);
}
// STAGE: 0 = walk global memory, 2 = records and row counts staged in
// shared memory (1 = records only was measured: no gain, r02l)
template <int STAGE>
__global__ void spread_walk(const int32_t* __restrict__ rc, int64_t nrows, int64_t ncols, int64_t nch,
                            int64_t chunk, const MonoRec* __restrict__ rec, const MonoRec* __restrict__ fine,
                            FeatState* __restrict__ st);

// The staged walk's dynamic shared memory limit, once per device (a function
// attribute is per device; set outside stream capture).
void ensure_walk_smem_attr() {
    static std::mutex mu;
    static uint64_t done = 0;
    int dev = 0;
    SOB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (dev < 64 && (done >> dev) & 1) return;
    SOB_CUDA(cudaFuncSetAttribute(spread_walk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kWalkSmem)));
    if (dev < 64) done |= uint64_t(1) << dev;
}

template <int STAGE>
__global__ void __launch_bounds__(kWalkThreads)
    spread_walk(const int32_t* __restrict__ rc, int64_t nrows, int64_t ncols, int64_t nch, int64_t chunk,
                const MonoRec* __restrict__ rec, const MonoRec* __restrict__ fine, FeatState* __restrict__ st) {
    pdl_enter();
    if (STAGE > 0) {
        extern __shared__ __align__(16) unsigned char wsm[];
        MonoRec* srec = reinterpret_cast<MonoRec*>(wsm);
        MonoRec* sfine = srec + nch;
        for (int64_t i = threadIdx.x; i < nch; i += kWalkThreads) srec[i] = rec[i];
        for (int64_t i = threadIdx.x; i < nch * kSubs; i += kWalkThreads) sfine[i] = fine[i];
        const int32_t* walk_rc = rc;
        if (STAGE == 2) {
            int32_t* src = reinterpret_cast<int32_t*>(sfine + nch * kSubs);
            const int4* rc4 = reinterpret_cast<const int4*>(rc);
            int4* src4 = reinterpret_cast<int4*>(src);
            for (int64_t i = threadIdx.x; i < nrows / 4; i += kWalkThreads) src4[i] = rc4[i];
            for (int64_t i = (nrows / 4) * 4 + threadIdx.x; i < nrows; i += kWalkThreads) src[i] = rc[i];
            walk_rc = src;
        }
        __syncthreads();
        if (threadIdx.x < 32) walk_and_finalize(walk_rc, nrows, ncols, nch, chunk, srec, sfine, st);
    } else {
        if (threadIdx.x < 32) walk_and_finalize(rc, nrows, ncols, nch, chunk, rec, fine, st);
    }
}

// The state, and the scratch every sweep accumulates into (dense diagonal
// bins, DIA diagonal counts, COO row counts), zeroed in one launch (the
// chain stays kernel -> kernel for programmatic dependent launch).
__global__ void feat_init(FeatState* st, int32_t* bins, int64_t nbins, unsigned long long* dcount, int64_t nd,
                          int32_t* rc, int64_t nrc) {
    pdl_enter();
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nbins; i += stride) bins[i] = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nd; i += stride) dcount[i] = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nrc; i += stride) rc[i] = 0;
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    st->t_begin = t;
    st->visits = 0;
    st->structure = 0;
    st->max_row = 0;
    st->min_row = INT32_MAX;
    st->nd = 0;
    st->ntd = 0;
    st->S = 0.0;
    st->ticket = 0;
}

}  // namespace

FeatWorkspace::FeatWorkspace(const so_matrix& m, cudaStream_t s) {
    ensure_walk_smem_attr();
    const int64_t n = m.nrows;
    const int64_t nch = ceil_div(n, spread_chunk(n));
    rc.alloc(n, s);
    if (m.format != SO_DIA) bins.alloc(n + m.ncols, s);
    if (m.format == SO_DIA || m.format == SO_HDC) dcount.alloc(m.dia.ndiags, s);
    csum.alloc(nch, s);
    P.alloc(nch + 1, s);
    rec.alloc(nch * (1 + kSubs) * int64_t(sizeof(MonoRec)), s);  // chunk + sub-chunk records
}

FeatWorkspace::~FeatWorkspace() {
    if (aux) cudaStreamDestroy(aux);
    if (fork_ev) cudaEventDestroy(fork_ev);
    if (join_ev) cudaEventDestroy(join_ev);
}

void FeatWorkspace::enable_fork() {
    if (aux) return;
    SOB_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
    SOB_CUDA(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    SOB_CUDA(cudaEventCreateWithFlags(&join_ev, cudaEventDisableTiming));
}

void enqueue_features(const so_matrix& m, double ratio, FeatState* st, cudaStream_t s, FeatWorkspace* ws_in) {
    const int64_t n = m.nrows, nc = m.ncols;
    const int64_t thr = true_diag_threshold(ratio, n, nc);  // features.cpp:146-147
    std::unique_ptr<FeatWorkspace> own;
    if (!ws_in) own.reset(new FeatWorkspace(m, s));
    FeatWorkspace& ws = ws_in ? *ws_in : *own;
    DBuf<int32_t>& rc = ws.rc;
    const bool dense_bins = m.format != SO_DIA;
    const int64_t nbins = n + nc;
    DBuf<int32_t>& bins = ws.bins;
    DBuf<unsigned long long>& dcount = ws.dcount;
    {
        const int64_t zb = dense_bins ? bins.n : 0, zr = m.format == SO_COO ? rc.n : 0;
        const int64_t most = std::max<int64_t>({zb, dcount.n, zr, 1});
        launch_pdl(feat_init, dim3(unsigned(grid_for(most, 256, 4))), dim3(256), 0, s, st, bins.get(), zb,
                   dcount.get(), dcount.n, rc.get(), zr);
        SOB_LAUNCH("feat_init");
    }
    const int grid_rows = grid_for(n, kB, 4);

    auto scan_csr = [&](bool accum) {
        if (n == 0) return;
        const CsrPart& c = m.csr;
        // entry-parallel for small matrices and for skewed ones up to 2M rows
        // (rows longer than the SpMV group cap: power-law corpus matrices
        // 126 -> 43 us, 302 -> 239 us); the row-lockstep sweep for the rest
        // (banded/stencil keys repeat across rows and its slot cache wins;
        // config 3's 4M-row R-MAT: 0.87 vs 0.93 ms entry-parallel)
        static const int force_entry = [] {  // diagnostic knob (A/B): SOB_FEAT_ENTRY=0/1/2 forces a sweep
            const char* e = std::getenv("SOB_FEAT_ENTRY");
            return e ? std::atoi(e) : -1;
        }();
        const bool entry = force_entry >= 0 ? force_entry == 1
                           : ws.sweep >= 0  ? ws.sweep == 1
                                            : (ceil_div(n, 32) < int64_t(current_ctx().num_sms) * 16 ||
                                               (c.nlong > 0 && n < (1 << 21)));
        if (entry && c.nblk > 0) {
            const int gb = grid_for(c.nblk * kB, kB, 4);
            // a row of more than kBigRowPieces pieces exists only if the pieces
            // outnumber the long rows by at least that much
            static const bool no_big = std::getenv("SOB_NO_BIGROW_PIECES") != nullptr;  // diagnostic knob (A/B)
            const bool big = !no_big && c.nlong > 0 && c.npieces - c.nlong >= kBigRowPieces;
            const int64_t big_row = big ? kBigRowPieces * kPiece : INT64_MAX;
            if (accum) {
                FeatCsrOp<true> op{c.col.get(), n, rc.get(), bins.get(), st, nullptr, 0, false};
                launch_pdl(feat_csr_entries<true>, dim3(gb), dim3(kB), 0, s, c.blk.get(), c.nblk, c.row_ptr.get(), op, big_row);
            } else {
                FeatCsrOp<false> op{c.col.get(), n, rc.get(), bins.get(), st, nullptr, 0, false};
                launch_pdl(feat_csr_entries<false>, dim3(gb), dim3(kB), 0, s, c.blk.get(), c.nblk, c.row_ptr.get(), op, big_row);
            }
            SOB_LAUNCH("feat_csr_entries");
            if (big) {
                FeatCsrOp<false> op{c.col.get(), n, rc.get(), bins.get(), st, nullptr, 0, false};
                launch_pdl(piece_sweep<FeatCsrOp<false>>, dim3(unsigned(c.npieces)), dim3(256), 0, s, c.piece_k.get(),
                           c.long_row.get(), c.long_piece.get(), c.nlong, op, kBigRowPieces);
                SOB_LAUNCH("feat_csr_pieces");
            }
            return;
        }
        const int g = grid_for(ceil_div(n, 32) * 256 / 8, 256, 8);
        // long rows (SpMV pieces) are swept piece-parallel instead of by one warp
        const int64_t skip = c.nlong > 0 ? int64_t(c.grp_cap) : INT64_MAX;
        unsigned* ticket = c.nlong > 0 ? &st->ticket : nullptr;  // skewed rows: dynamic groups
        // sweep mode 2: every entry straight to the global bins (no hash)
        const bool all_direct = force_entry == 2 || (force_entry < 0 && ws.sweep == 2);
        if (accum) {
            FeatCsrOp<true> op{c.col.get(), n, rc.get(), bins.get(), st, nullptr, 0, all_direct};
            launch_pdl(row_sweep_cols<FeatCsrOp<true>>, dim3(g), dim3(256), 0, s, c.row_ptr.get(), c.col.get(), n, op, skip,
                       ticket);
        } else {
            FeatCsrOp<false> op{c.col.get(), n, rc.get(), bins.get(), st, nullptr, 0, all_direct};
            launch_pdl(row_sweep_cols<FeatCsrOp<false>>, dim3(g), dim3(256), 0, s, c.row_ptr.get(), c.col.get(), n, op, skip,
                       ticket);
        }
        SOB_LAUNCH("feat_csr");
        if (c.nlong > 0) {
            FeatCsrOp<false> op{c.col.get(), n, rc.get(), bins.get(), st, nullptr, 0, false};
            launch_pdl(piece_sweep<FeatCsrOp<false>>, dim3(unsigned(c.npieces)), dim3(256), 0, s, c.piece_k.get(),
                       c.long_row.get(), c.long_piece.get(), c.nlong, op, int64_t(0));
            SOB_LAUNCH("feat_csr_pieces");
        }
    };
    auto scan_dia = [&]() {
        launch_pdl(feat_dia, dim3(grid_rows), dim3(kB), 0, s, n, nc, int(m.dia.ndiags), m.dia.offsets.get(),
                   m.dia.values.get(), rc.get(), dcount.get(), st);
        SOB_LAUNCH("feat_dia");
    };
    auto scan_ell = [&]() {
        launch_pdl(feat_ell, dim3(grid_rows), dim3(kB), 0, s, n, int(m.ell.width), m.ell.col.get(), rc.get(),
                   bins.get(), st);
        SOB_LAUNCH("feat_ell");
    };
    auto scan_coo = [&]() {
        if (m.coo.nnz == 0) return;
        launch_pdl(feat_coo, dim3(grid_for(m.coo.nnz, kB, 4)), dim3(kB), 0, s, m.coo.nnz, n, m.coo.row.get(),
                   m.coo.col.get(), rc.get(), bins.get(), st);
        SOB_LAUNCH("feat_coo");
    };

    switch (m.format) {
        case SO_COO:  // rc zeroed by feat_init
            scan_coo();
            break;
        case SO_CSR:
            scan_csr(false);
            break;
        case SO_DIA:
            scan_dia();
            break;
        case SO_ELL:
            scan_ell();
            break;
        case SO_HYB:
            scan_ell();
            scan_coo();
            break;
        case SO_HDC:
            scan_dia();
            if (m.dia.ndiags) {
                launch_pdl(dcount_to_bins, dim3(unsigned(ceil_div(m.dia.ndiags, 256))), dim3(256), 0, s,
                           dcount.get(), m.dia.offsets.get(), int(m.dia.ndiags), n, bins.get());
                SOB_LAUNCH("dcount_to_bins");
            }
            scan_csr(true);
            break;
    }

    const int64_t chunk = spread_chunk(n);
    const int64_t nch = ceil_div(n, chunk);
    DBuf<double>& csum = ws.csum;
    DBuf<double>& P = ws.P;
    MonoRec* rec = reinterpret_cast<MonoRec*>(ws.rec.get());
    // N_D / N_TD over the bins only feed the finalize at the end of the
    // spread walk: with a forked workspace (the tune graph) they run on a
    // second branch beside feat_rows -> spread_prefix -> spread_mono
    const bool fork = ws.aux != nullptr;
    cudaStream_t sb = fork ? ws.aux : s;
    if (fork) {
        SOB_CUDA(cudaEventRecord(ws.fork_ev, s));
        SOB_CUDA(cudaStreamWaitEvent(sb, ws.fork_ev, 0));
    }
    if (dense_bins) {
        launch_pdl(feat_bins<int32_t>, dim3(grid_for(nbins, 256)), dim3(256), 0, sb, bins.get(), nbins, thr, st);
        SOB_LAUNCH("feat_bins");
    } else if (m.dia.ndiags) {
        launch_pdl(feat_bins<unsigned long long>, dim3(grid_for(m.dia.ndiags, 256)), dim3(256), 0, sb, dcount.get(),
                   m.dia.ndiags, thr, st);
        SOB_LAUNCH("feat_bins");
    }
    if (fork) SOB_CUDA(cudaEventRecord(ws.join_ev, sb));
    launch_pdl(feat_rows, dim3(unsigned(nch)), dim3(kB), 0, s, rc.get(), n, chunk, st, csum.get());
    SOB_LAUNCH("feat_rows");
    launch_pdl(spread_prefix, dim3(1), dim3(512), 0, s, csum.get(), nch, P.get());
    SOB_LAUNCH("spread_prefix");
    MonoRec* fine = rec + nch;
    launch_pdl(spread_mono, dim3(unsigned(nch)), dim3(kB), 0, s, rc.get(), n, chunk, st, csum.get(), P.get(), rec,
               fine);
    SOB_LAUNCH("spread_mono");
    if (fork) SOB_CUDA(cudaStreamWaitEvent(s, ws.join_ev, 0));  // the walk's finalize reads N_D / N_TD
    const size_t wsm = walk_smem_bytes(n, nch);
    if (wsm <= kWalkSmem) {
        ensure_walk_smem_attr();  // normally done by the workspace, before any capture
        launch_pdl(spread_walk<2>, dim3(1), dim3(kWalkThreads), wsm, s, rc.get(), n, nc, nch, chunk, rec, fine, st);
    } else {
        launch_pdl(spread_walk<0>, dim3(1), dim3(32), 0, s, rc.get(), n, nc, nch, chunk, rec, fine, st);
    }
    SOB_LAUNCH("spread_walk");
}

}  // namespace sob
