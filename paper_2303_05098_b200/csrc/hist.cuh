// Diagonal histogram with shared-memory privatisation.
//
// Banded/stencil matrices send every entry into a handful of diagonal bins
// (27 for configs 2 and 5), so direct global atomics would serialise on the
// L2 atomic units.  Each persistent CTA keeps an open-addressing hash of
// (key -> count) in shared memory; lanes holding the same key are first
// merged with __match_any_sync, leaders insert into the hash, and the hash is
// flushed with one global atomic per distinct key per CTA.  Keys that do not
// find a slot within kProbe probes (scattered matrices) go straight to the
// global bins, where they are spread over many addresses anyway.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace sob {

constexpr int kHashSlots = 2048;  // power of two
constexpr int kProbe = 8;
constexpr int32_t kEmptyKey = -1;

struct SmemHash {
    int32_t keys[kHashSlots];
    int32_t cnts[kHashSlots];
    int32_t used;  // distinct keys inserted; past half full, new keys go straight to global
};

__device__ __forceinline__ void hash_init(SmemHash& h) {
    for (int i = threadIdx.x; i < kHashSlots; i += blockDim.x) {
        h.keys[i] = kEmptyKey;
        h.cnts[i] = 0;
    }
    if (threadIdx.x == 0) h.used = 0;
}

__device__ __forceinline__ void hash_insert_one(SmemHash& h, int32_t* __restrict__ gbins, int32_t key, int32_t add);

// Per-warp cache of the key seen at each lockstep slot (banded rows present
// the same key at slot j in every row: offset_j + n - 1).  Slot j lives in
// lane j % 32, register j / 32.  A uniform step costs one vote and one
// register add instead of a hash update; a slot whose key changes spills its
// count to the hash.  Call flush() (every lane) before the hash is flushed.
struct SlotCache {
    int32_t key[2] = {-1, -1};
    int32_t cnt[2] = {0, 0};
    // all 32 lanes call; returns true when the step was absorbed
    __device__ __forceinline__ bool add(SmemHash& h, int32_t* gbins, int32_t k, int slot) {
        if (slot < 0) return false;
        const unsigned valid = __ballot_sync(0xffffffffu, k >= 0);
        if (!valid) return true;
        const int32_t k0 = __shfl_sync(0xffffffffu, k, __ffs(valid) - 1);
        if (!__all_sync(0xffffffffu, k < 0 || k == k0)) return false;
        if (int(threadIdx.x & 31u) == (slot & 31)) {
            const int w = slot >> 5;
            const int32_t ck = w ? key[1] : key[0];
            const int32_t cc = w ? cnt[1] : cnt[0];
            int32_t nk = k0, nc = __popc(valid);
            if (ck == k0) {
                nc += cc;
            } else if (ck >= 0) {
                hash_insert_one(h, gbins, ck, cc);
            }
            if (w) {
                key[1] = nk;
                cnt[1] = nc;
            } else {
                key[0] = nk;
                cnt[0] = nc;
            }
        }
        return true;
    }
    // Eight consecutive slots j0..j0+7 at once, when every lane holds a valid
    // entry in each and all lanes agree slot by slot (the interior of banded
    // matrices): one vote for the batch, lane (j0+d)%32 absorbs slot j0+d.
    // All 32 lanes call; returns false (nothing done) otherwise.
    __device__ __forceinline__ bool add8(SmemHash& h, int32_t* gbins, const int32_t (&k)[8], int j0, bool all_valid) {
        if (!__all_sync(0xffffffffu, all_valid)) return false;
        int32_t k0[8];
        bool same = true;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            k0[u] = __shfl_sync(0xffffffffu, k[u], 0);
            same = same && k[u] == k0[u];
        }
        if (!__all_sync(0xffffffffu, same)) return false;
        const int d = int(threadIdx.x & 31u) - (j0 & 31);
        if (d >= 0 && d < 8) {
            int32_t kk = k0[0];
#pragma unroll
            for (int u = 1; u < 8; ++u) kk = d == u ? k0[u] : kk;
            const int w = (j0 + d) >> 5;
            const int32_t ck = w ? key[1] : key[0];
            const int32_t cc = w ? cnt[1] : cnt[0];
            int32_t nc = 32;
            if (ck == kk)
                nc += cc;
            else if (ck >= 0)
                hash_insert_one(h, gbins, ck, cc);
            if (w) {
                key[1] = kk;
                cnt[1] = nc;
            } else {
                key[0] = kk;
                cnt[0] = nc;
            }
        }
        return true;
    }
    __device__ __forceinline__ void flush(SmemHash& h, int32_t* gbins) {
        for (int w = 0; w < 2; ++w)
            if (key[w] >= 0 && cnt[w] > 0) hash_insert_one(h, gbins, key[w], cnt[w]);
        key[0] = key[1] = -1;
        cnt[0] = cnt[1] = 0;
    }
};

// One lane adds `add` to `key`: shared-memory hash, or the global bins when
// the key finds no slot.  Not warp-synchronous.
__device__ __forceinline__ void hash_insert_one(SmemHash& h, int32_t* __restrict__ gbins, int32_t key, int32_t add) {
    unsigned slot = unsigned(key) & (kHashSlots - 1);
    // scattered keys (hash half full): only the home slot is checked, so keys
    // that were hot early still merge in shared memory and the rest go
    // straight to the global bins without a probe chain
    const bool full = h.used >= kHashSlots / 2;
    const int probes = full ? 1 : kProbe;
#pragma unroll 1
    for (int p = 0; p < probes; ++p) {
        int32_t old = h.keys[slot];
        if (old == key) {
            atomicAdd(&h.cnts[slot], add);
            return;
        }
        if (old == kEmptyKey) {
            if (full) break;
            old = atomicCAS(&h.keys[slot], kEmptyKey, key);
            if (old == kEmptyKey) {
                atomicAdd(&h.used, 1);
                atomicAdd(&h.cnts[slot], add);
                return;
            }
            if (old == key) {
                atomicAdd(&h.cnts[slot], add);
                return;
            }
        }
        slot = (slot + 1) & (kHashSlots - 1);
    }
    atomicAdd(gbins + key, add);
}

// key >= 0 valid; key < 0 means "no entry for this lane".  Every lane of the
// warp must call this (warp-synchronous).
__device__ __forceinline__ void hash_add(SmemHash& h, int32_t* __restrict__ gbins, int32_t key) {
    const unsigned lane = threadIdx.x & 31u;
    // fast path: every valid lane holds the same key (banded rows swept in
    // lockstep) -- a vote instead of __match_any_sync
    const unsigned valid = __ballot_sync(0xffffffffu, key >= 0);
    if (!valid) return;
    const int first = __ffs(valid) - 1;
    const int32_t k0 = __shfl_sync(0xffffffffu, key, first);
    unsigned peers;
    if (__all_sync(0xffffffffu, key < 0 || key == k0)) {
        peers = valid;
    } else if (__shfl_sync(0xffffffffu, h.used >= kHashSlots / 2, 0)) {
        // scattered keys (the CTA's hash is already half full): warp
        // merging rarely pays for its __match_any_sync -- each lane goes on
        // alone (home-slot check, else a global atomic)
        if (key >= 0) hash_insert_one(h, gbins, key, 1);
        return;
    } else {
        // distinct dummy keys for idle lanes so they never merge with real ones
        const int32_t k = key >= 0 ? key : -2 - int32_t(lane);
        peers = __match_any_sync(0xffffffffu, k);
    }
    if (key < 0) return;
    const int leader = __ffs(peers) - 1;
    if (int(lane) != leader) return;
    hash_insert_one(h, gbins, key, __popc(peers));
}

__device__ __forceinline__ void hash_flush(SmemHash& h, int32_t* __restrict__ gbins) {
    for (int i = threadIdx.x; i < kHashSlots; i += blockDim.x) {
        const int32_t k = h.keys[i];
        if (k != kEmptyKey && h.cnts[i] != 0) atomicAdd(gbins + k, h.cnts[i]);
    }
}

// Row of entry k inside a row-block whose row_ptr slice [r0, r0+nr] is staged
// in shared memory: the last row whose start is <= k.
__device__ __forceinline__ int row_in_block(const int64_t* srp, int nr, int64_t k) {
    int lo = 0, hi = nr;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (srp[mid] <= k)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// Histogram ops with a direct path (kPieceDirect): piece(r, k, valid) for
// long-row pieces (the entries of one row have distinct columns, so their
// diagonal keys never repeat inside a piece: a global atomic each), and
// scattered() / direct(r, c, valid) for row sweeps once the CTA's hash is
// half full.
template <class Op, class = void>
struct piece_direct : std::false_type {};
template <class Op>
struct piece_direct<Op, std::void_t<decltype(Op::kPieceDirect)>> : std::bool_constant<Op::kPieceDirect> {};

// ------------------------------------------------------------ row sweep
// Row-lockstep traversal of a CSR: lane = row, slot j in lockstep across the
// warp, so banded / stencil rows present the SAME diagonal key in every lane
// at every step and warp aggregation (hash_add's __match_any_sync) collapses
// 32 updates into one.  Rows longer than kLockstepMax finish cooperatively:
// the whole warp strides over the rest of the row.  Every op call is made by
// all 32 lanes (valid=false for idle lanes), so ops may be warp-synchronous.
// Op interface: begin(), row(r, valid, len) once per row, (r, k, valid) per
// entry slot, end().  Entries of rows longer than skip_above are not visited
// (CSR long rows are split into kPiece pieces and swept by piece_sweep).
constexpr int kLockstepMax = 64;

// With a ticket (a zeroed counter), warps claim 32-row groups dynamically --
// skewed row lengths (power-law) otherwise leave most warps of a CTA waiting
// at op.end()'s barrier for the one that drew the heavy rows.
__device__ __forceinline__ int64_t next_group(unsigned* ticket) {
    unsigned t = 0;
    if ((threadIdx.x & 31u) == 0) t = atomicAdd(ticket, 1u);
    return int64_t(__shfl_sync(0xffffffffu, t, 0)) * 32;
}

template <class Op>
__global__ void __launch_bounds__(256) row_sweep(const int64_t* __restrict__ rp, int64_t nrows, Op op,
                                                 int64_t skip_above = INT64_MAX, unsigned* ticket = nullptr) {
    pdl_enter();
    op.begin();
    const int lane = int(threadIdx.x & 31u);
    const int64_t nwarps = int64_t(gridDim.x) * (blockDim.x / 32);
    for (int64_t wb = ticket ? next_group(ticket) : (int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5)) * 32;
         wb < nrows; wb = ticket ? next_group(ticket) : wb + nwarps * 32) {
        const int64_t r = wb + lane;
        const bool has = r < nrows;
        const int64_t a = has ? rp[r] : 0;
        const int64_t len = has ? rp[r + 1] - a : 0;
        op.row(int(r), has, len);
        // rows above skip_above are left entirely to a piece-parallel kernel
        const int64_t elen = len > skip_above ? 0 : len;
        const int64_t maxlen = warp_max(elen < kLockstepMax ? elen : int64_t(kLockstepMax));
        for (int64_t j = 0; j < maxlen; ++j) op(int(r), a + j, has && j < elen);
        unsigned longm = __ballot_sync(0xffffffffu, elen > kLockstepMax);
        while (longm) {
            const int src = __ffs(longm) - 1;
            longm &= longm - 1;
            const int64_t la = __shfl_sync(0xffffffffu, a, src);
            const int64_t ll = __shfl_sync(0xffffffffu, elen, src);
            const int lr = __shfl_sync(0xffffffffu, int(r), src);
            for (int64_t j0 = kLockstepMax; j0 < ll; j0 += 32) op(lr, la + j0 + lane, j0 + lane < ll);
        }
    }
    op.end();
}

// row_sweep for ops that only need the column of an entry (op.entry(r, col,
// valid, slot)): the columns of 8 lockstep slots are loaded before any is
// handed to the op, so each lane keeps 8 independent loads in flight instead
// of one load per (synchronising) hash update.  slot = the lockstep slot j
// (< kLockstepMax), or -1 in the cooperative tail of a long row.
template <class Op>
__global__ void __launch_bounds__(256) row_sweep_cols(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                      int64_t nrows, Op op, int64_t skip_above = INT64_MAX,
                                                      unsigned* ticket = nullptr) {
    pdl_enter();
    constexpr int U = 8;
    op.begin();
    const int lane = int(threadIdx.x & 31u);
    const int64_t nwarps = int64_t(gridDim.x) * (blockDim.x / 32);
    for (int64_t wb = ticket ? next_group(ticket) : (int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5)) * 32;
         wb < nrows; wb = ticket ? next_group(ticket) : wb + nwarps * 32) {
        const int64_t r = wb + lane;
        const bool has = r < nrows;
        const int64_t a = has ? rp[r] : 0;
        const int64_t len = has ? rp[r + 1] - a : 0;
        op.row(int(r), has, len);
        const int64_t elen = len > skip_above ? 0 : len;
        if constexpr (piece_direct<Op>::value) {
            // scattered keys (the CTA's hash is half full): no lockstep
            // votes, every lane inserts its own entries (hash home slot,
            // else a global atomic)
            if (op.scattered()) {
                for (int64_t j0 = 0; j0 < elen; j0 += U) {
                    int32_t cv[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) cv[u] = j0 + u < elen ? __ldg(col + a + j0 + u) : 0;
#pragma unroll
                    for (int u = 0; u < U; ++u) op.direct(int(r), cv[u], j0 + u < elen);
                }
                continue;
            }
        }
        const int64_t maxlen = warp_max(elen < kLockstepMax ? elen : int64_t(kLockstepMax));
        for (int64_t j0 = 0; j0 < maxlen; j0 += U) {
            int32_t cv[U];
#pragma unroll
            // L1-allocating: a lane's 8 consecutive columns share one or two sectors
            for (int u = 0; u < U; ++u) cv[u] = (has && j0 + u < elen) ? __ldg(col + a + j0 + u) : 0;
            if constexpr (Op::kHasEntry8) {
                if (op.entry8(int(r), cv, int(j0), has && j0 + U <= elen)) continue;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (j0 + u < maxlen) op.entry(int(r), cv[u], has && j0 + u < elen, int(j0 + u));
        }
        unsigned longm = __ballot_sync(0xffffffffu, elen > kLockstepMax);
        while (longm) {
            const int src = __ffs(longm) - 1;
            longm &= longm - 1;
            const int64_t la = __shfl_sync(0xffffffffu, a, src);
            const int64_t ll = __shfl_sync(0xffffffffu, elen, src);
            const int lr = __shfl_sync(0xffffffffu, int(r), src);
            for (int64_t j0 = kLockstepMax; j0 < ll; j0 += 32 * U) {
                int32_t cv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t j = j0 + u * 32 + lane;
                    cv[u] = j < ll ? ld_stream(col + la + j) : 0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) op.entry(lr, cv[u], j0 + u * 32 + lane < ll, -1);
            }
        }
    }
    op.end();
}

// One CTA per long-row piece (CsrPart::piece_k): coalesced entries of a
// single row, so no row search.  Same op interface (row() is not called).
// Pieces of rows with at most min_pieces pieces exit at once.
template <class Op>
__global__ void __launch_bounds__(256) piece_sweep(const int64_t* __restrict__ pk, const int32_t* __restrict__ lrow,
                                                   const int64_t* __restrict__ lpiece, int64_t nlong, Op op,
                                                   int64_t min_pieces = 0) {
    pdl_enter();
    const int64_t k0 = pk[2 * blockIdx.x], k1 = pk[2 * blockIdx.x + 1];
    // row of this piece: the long row whose piece range holds blockIdx.x
    int64_t lo = 0, hi = nlong;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (lpiece[mid] <= int64_t(blockIdx.x))
            lo = mid;
        else
            hi = mid;
    }
    // rows of at most min_pieces pieces were swept by the caller's other kernel
    if (lpiece[lo + 1] - lpiece[lo] <= min_pieces) return;
    op.begin();
    const int r = lrow[lo];
    for (int64_t b = k0; b < k1; b += blockDim.x) {
        if constexpr (piece_direct<Op>::value)
            op.piece(r, b + threadIdx.x, b + threadIdx.x < k1);
        else
            op(r, b + threadIdx.x, b + threadIdx.x < k1);
    }
    op.end();
}

}  // namespace sob
