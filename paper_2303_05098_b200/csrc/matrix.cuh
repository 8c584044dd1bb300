// Device-resident sparse containers (the HBM layout of DESIGN.md §3) and the
// internal entry points shared by the .cu translation units.
#pragma once
#include <atomic>
#include <functional>

#include <memory>
#include <mutex>
#include <string>

#include "common.cuh"

namespace sob {

// CSR row-block partition (the "analysis" done once per matrix):
// CTA b of the streaming CSR kernel owns rows [blk[b], blk[b+1]).  A block
// holds the rows whose first entry falls into one kWindow-wide nnz window
// (<= 2*kWindow entries, staged in shared memory), at most kRowsPerBlock rows,
// or exactly one row longer than kWindow ("long row" block).
constexpr int kWindow = 1024;
constexpr int kGrpPadBit = 62;
constexpr int64_t kGrpPad = int64_t(1) << kGrpPadBit;
constexpr int64_t kGrpPadShare = 64;  // padded kernel when >= 1/64 of the groups prefer it
constexpr int kPiece = 2048;  // entries per CTA for rows longer than grp_cap
// SpMV warp groups: <= kGroupRowsMax consecutive rows holding <= grp_cap = 32*items
// entries (greedy); short-row matrices (mean <= 8) load 8 entries per lane,
// others 12 (scripts/spmv_lab.cu measurements).
constexpr int kGroupItemsShort = 8;
constexpr int kGroupItemsLong = 12;
constexpr int kRowsPerBlock = 1024;
// a warp group holds at most kGroupRowsMax rows (lane i walks rows i, i+32,
// ...): tiny rows (R-MAT's tail, sparse corpus matrices) fill a group's
// entries instead of leaving most of its 32*IT slots empty
constexpr int kGroupRowsMax = 128;
// CSR rows longer than this (and <= grp_cap) are summed by the whole warp
// (strided partial sums + fixed butterfly) instead of one lane's serial walk
constexpr int kCoopLen = 64;
constexpr int kStreamBlock = 256;

struct CooPart {
    int64_t nnz = 0;
    DBuf<int32_t> row, col;
    DBuf<double> val;
    // Lazily profiled on the first multiply (spmv.cu coo_profile); atomics
    // because concurrent readers of one const matrix may race to fill them
    // (each value is meaningful on its own: -1 = unknown = the safe path).
    mutable std::atomic<int64_t> max_gap{-1};  // longest empty-row run
    mutable std::atomic<int> long_runs{-1};    // some row covers > kFixupInline chunks
    mutable std::atomic<int> short_rows{-1};   // every row <= 32 entries (COO CONT: no records)
};
struct CsrPart {
    int64_t nnz = 0;
    DBuf<int64_t> row_ptr;
    DBuf<int32_t> col;
    DBuf<double> val;
    DBuf<int32_t> blk;    // row-block partition, nblk+1 entries
    DBuf<int64_t> blk_k;  // first entry of each row block (= row_ptr[blk[b]])
    int64_t nblk = 0;
    mutable std::atomic<int> canonical{-1};  // rows strictly increasing: -1 unknown, 0 no, 1 yes (cached)
    // SpMV warp-group partition
    int64_t ngrp = 0;
    int grp_cap = 32 * kGroupItemsLong;
    DBuf<int32_t> grp;     // [ngrp+1]
    DBuf<int64_t> grp_k;   // [ngrp+1]; bit kGrpPadBit of grp_k[g]: group g's padded product layout
    int64_t npad = 0;      // groups flagged padded (0: no flags set, the SpMV runs the plain-layout kernel)
    int64_t ncoop = 0;     // rows of kCoopLen < length <= grp_cap (summed by the whole warp, spmv.cu)
    int grp_rpl = 1;       // rows per lane of the widest group (1: every group <= 32 rows; else kGroupRowsMax / 32)
    // rows longer than grp_cap, split into kPiece-entry pieces for SpMV
    int64_t nlong = 0, npieces = 0;
    DBuf<int32_t> long_row;     // [nlong]
    DBuf<int64_t> long_piece;   // [nlong+1] first piece of each long row
    DBuf<int64_t> piece_k;      // [2*npieces] entry range [start, end) of each piece
};
struct DiaPart {
    int64_t ndiags = 0;
    DBuf<int64_t> offsets;
    DBuf<double> values;  // [d * nrows + i]
    int64_t stored_nnz = 0;
};
struct EllPart {
    int64_t width = 0;
    DBuf<int32_t> col;  // column-major [k * nrows + i], sentinel -1
    DBuf<double> val;
    int64_t stored_nnz = 0;
};

}  // namespace sob

namespace sob {
struct TunePlan;  // cached CUDA graph of tune_ml (capi.cu)
void destroy_tune_plan(TunePlan* p);
struct TunePlanDeleter {
    void operator()(TunePlan* p) const { destroy_tune_plan(p); }
};
}  // namespace sob

struct so_matrix {
    mutable std::unique_ptr<sob::TunePlan, sob::TunePlanDeleter> tune_plan;
    mutable std::mutex tune_mu;  // guards tune_plan (one tune_ml at a time per matrix)
    int device = 0;
    int32_t format = SO_COO;
    int64_t nrows = 0, ncols = 0;
    sob::CooPart coo;  // COO, HYB coo part
    sob::CsrPart csr;  // CSR, HDC csr part
    sob::DiaPart dia;  // DIA, HDC dia part
    sob::EllPart ell;  // ELL, HYB ell part
    int64_t kh = 0;
    int64_t threshold = 0;
    // cached min/max DIA offset (pipelined host spmv), filled on first use
    // (published with release on dia_window_known; concurrent fillers write the same values)
    mutable std::atomic<bool> dia_window_known{false};
    mutable std::atomic<int64_t> dia_omin{0}, dia_omax{0};
    // CSR row-group chunks of the pinned follow path (spmv.cu): group and row
    // at each chunk boundary, filled on first use (published like the window)
    static constexpr int kFollowChunks = 8;
    mutable std::atomic<bool> csr_chunks_known{false};
    mutable std::atomic<int64_t> csr_chunk_grp[kFollowChunks + 1] = {};
    mutable std::atomic<int64_t> csr_chunk_row[kFollowChunks + 1] = {};
    // COO entry-chunk ranges of the same pipeline: first chunk of each range
    // and the first row a later range may write
    mutable std::atomic<bool> coo_chunks_known{false};
    mutable std::atomic<int64_t> coo_chunk_c[kFollowChunks + 1] = {};
    mutable std::atomic<int64_t> coo_chunk_row[kFollowChunks + 1] = {};

    int64_t nnz() const {
        switch (format) {
            case SO_COO: return coo.nnz;
            case SO_CSR: return csr.nnz;
            case SO_DIA: return dia.stored_nnz;
            case SO_ELL: return ell.stored_nnz;
            case SO_HYB: return ell.stored_nnz + coo.nnz;
            case SO_HDC: return dia.stored_nnz + csr.nnz;
        }
        return 0;
    }
};

namespace sob {

// --- conversions (convert.cu) ---
void build_row_blocks(CsrPart& csr, int64_t nrows, cudaStream_t s);
so_matrix* coo_to_csr_device(const so_matrix& coo, cudaStream_t s);  // canonical input
so_matrix* csr_to_format(const so_matrix& csr, int32_t target, const so_conversion_config& cfg,
                         cudaStream_t s);
so_matrix* any_to_csr(const so_matrix& m, cudaStream_t s);  // to_coo semantics, CSR layout
so_matrix* csr_to_coo(const so_matrix& csr, cudaStream_t s);
so_matrix* clone_matrix(const so_matrix& m, cudaStream_t s);
bool coo_is_canonical(const so_matrix& coo, cudaStream_t s);
so_matrix* coo_from_triplets_device(int64_t nrows, int64_t ncols, int64_t n, const int64_t* row_h,
                                    const int64_t* col_h, const double* val_h, cudaStream_t s);
// the same over consecutive host segments (concatenated in order on the
// device: Matrix Market slices parsed by different threads)
struct TripletSegment {
    const int64_t* row;
    const int64_t* col;
    const double* val;
    int64_t n;
};
so_matrix* coo_from_triplet_segments(int64_t nrows, int64_t ncols, const TripletSegment* segs, int nseg,
                                     cudaStream_t s);
bool csr_rows_canonical(const so_matrix& csr, cudaStream_t s);

// --- Matrix Market I/O (ingest.cu) ---
so_matrix* read_matrix_market(const std::string& path, cudaStream_t s);
void write_matrix_market(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* row, const int64_t* col,
                         const double* val, const std::string& path);

// --- spmv (spmv.cu) ---
void spmv_device(const so_matrix& m, const double* x, double* y, cudaStream_t s);
void spmv_device_rows(const so_matrix& m, const double* x, double* y, int64_t lo, int64_t hi, cudaStream_t s);
// DIA-window matrix with x/y in mapped pinned host memory (device-visible
// pointers): one kernel reads x and writes y over the host link; false when
// the window is too wide or unknown (spmv.cu)
// (row blocks [blk_lo, blk_hi) of zero_copy_rows_per_block() rows; -1 = all)
bool spmv_dia_zero_copy(const so_matrix& m, const double* x_mapped, double* y_mapped, cudaStream_t s,
                        int64_t blk_lo = 0, int64_t blk_hi = -1);
int64_t zero_copy_rows_per_block();
// pinned host x (copied up by ONE copy-engine H2D on `copy`) and mapped host
// y on a narrow-window DIA matrix: a persistent kernel follows the copy front
// (spmv.cu dia_follow_kernel); synchronous; false = not eligible (or the copy
// never arrived: y must be recomputed)
bool spmv_dia_follow(const so_matrix& m, const double* x_host, double* y_mapped, cudaStream_t s,
                     cudaStream_t copy);
// pinned host x (one upload on `copy`) and mapped host y on a CSR matrix (or
// HDC without a DIA part): the CSR kernels follow the upload (spmv.cu);
// synchronous; false = not eligible or the copy never arrived
bool spmv_csr_follow(const so_matrix& m, const double* x_host, double* y_mapped, cudaStream_t s,
                     cudaStream_t copy);
// The same, in two halves (pageable staging, stage.cu): follow_launch locks
// the device's follow stage, launches the kernel -- one launch per y chunk of
// rows_per_chunk rows (a multiple of zero_copy_rows_per_block(); 0 = one
// launch), calling after_chunk(j) after launch j (e.g. to record an event) --
// then calls upload(dx) to enqueue the caller's H2D copies of x into dx on
// `copy`, then the copy-complete flag and the sentinel refill.  After s is
// synchronised (on any thread), follow_finish returns false when the copy
// never arrived (y invalid).
struct FollowToken {
    unsigned* timed_out = nullptr;  // this call's timeout word (mapped)
    cudaEvent_t done = nullptr;     // recorded after the call's kernels (before the sentinel refill)
    bool upload_first = false;      // in: the upload does not block the host (pinned x): queue it first
};
bool follow_launch(const so_matrix& m, double* y_mapped, cudaStream_t s, cudaStream_t copy, int64_t rows_per_chunk,
                   const std::function<void(int64_t)>* after_chunk, const std::function<void(double*)>& upload,
                   FollowToken& tok);
// the same for CSR / ELL / COO / HYB (one launch of the FOLLOW kernels, then
// after_kernels(y_dev), e.g. an event gating every y chunk's copy-out).
// y_dev == nullptr: the kernels stored y into y_mapped; otherwise y is in
// device memory (COO parts) and after_kernels queues its copy into y_mapped
// on `s` (without a callback: one copy of all of y)
bool follow_launch_rows(const so_matrix& m, double* y_mapped, cudaStream_t s, cudaStream_t copy,
                        const std::function<void(const double* y_dev)>* after_kernels,
                        const std::function<void(double*)>& upload, FollowToken& tok);
bool follow_finish(FollowToken& tok);
// min/max DIA offset of a DIA-window matrix (read once, cached on the matrix)
void ensure_dia_window(const so_matrix& m, cudaStream_t s);
// spmv(m, x) with PAGEABLE host x/y (stage.cu): host threads copy through a
// cached pinned staging ring while the device multiplies chunk by chunk;
// false when the call is too small to gain (the caller's one-shot path).
// make_y (y == nullptr): y is created by make_y() on the calling thread while
// the device works (so_spmv_new)
bool spmv_pageable(const so_matrix& m, const double* x, double* y, cudaStream_t s,
                   const std::function<double*()>* make_y = nullptr);
void spmv_rows_push(const so_matrix& m, const double* x, double* y, int64_t lo, int64_t hi, double* remote,
                    unsigned* ticket, unsigned long long* remote_flag, unsigned long long flag_value,
                    cudaStream_t s);
void wait_flag(const unsigned long long* flag, unsigned long long value, cudaStream_t s);
unsigned long long wait_flag_timeouts();
so_matrix* gen_stencil27_dia(int64_t g, int64_t row_lo, int64_t row_hi, int64_t col_lo, int64_t col_hi,
                             uint64_t seed, cudaStream_t s);
int64_t spmv_bytes(const so_matrix& m);

// --- host-side cap rules (formats.cpp:348-367), shared by convert + tune ---
int64_t padded_entry_cap(const so_conversion_config& c, int64_t nnz);
int64_t effective_kh(const so_conversion_config& c, int64_t nnz, int64_t nrows);
int64_t true_diag_threshold(double ratio, int64_t nrows, int64_t ncols);
int64_t checked_mul(int64_t a, int64_t b);

}  // namespace sob
