/* sparseoracle_b200.h -- C-ABI of the B200 (sm_100a) hot path.
 *
 * This is the boundary the reference's C++ API (proj/include/sparseoracle/
 * *.hpp) is re-implemented on top of: the C++ drop-in in
 * paper_2303_05098_b200/cpp/ calls only these entry points, and so do the
 * Python parity tests (ctypes) and bench.py.  Plain pointers and sizes, no
 * torch types, no C++ exceptions across the boundary: every call returns an
 * so_status and leaves a thread-local message in so_last_error().
 *
 * Each entry point names the reference interface it replaces
 * (file:line under /root/reference/proj).
 *
 * Device layout (HBM), see DESIGN.md §3:
 *   COO  row int32[z], col int32[z], val f64[z]          (canonical: row-major sorted)
 *   CSR  row_ptr int64[n+1], col int32[z], val f64[z]     (+ row-block partition int32)
 *   DIA  offsets int64[D], values f64[D*n] diagonal-major (same as host)
 *   ELL  col int32[K*n], val f64[K*n] COLUMN-major (host view is row-major i*K+k)
 *   HYB  ELL part + COO part;   HDC  DIA part + CSR part
 * Row/column counts must be < 2^31 (int32 device indices); nnz is 64-bit.
 */
#ifndef SPARSEORACLE_B200_H
#define SPARSEORACLE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The C++ shim rethrows each as the matching
 * sparseoracle::Error subclass (errors.hpp:8-71). */
typedef enum so_status {
    SO_OK = 0,
    SO_INVALID_INPUT = 1,          /* errors.hpp:13  InvalidInput        */
    SO_PADDING_OVERFLOW = 2,       /* errors.hpp:19  PaddingOverflow     */
    SO_DIMENSION_MISMATCH = 3,     /* errors.hpp:23  DimensionMismatch   */
    SO_EMPTY_MATRIX = 4,           /* errors.hpp:27  EmptyMatrix         */
    SO_MALFORMED_MODEL = 5,        /* errors.hpp:32  MalformedModel      */
    SO_INDEX_OUT_OF_RANGE = 6,     /* errors.hpp:53  IndexOutOfRange     */
    SO_ALL_FORMATS_INFEASIBLE = 7, /* errors.hpp:69  AllFormatsInfeasible*/
    SO_CUDA_ERROR = 8,
    SO_OUT_OF_MEMORY = 9,
    SO_ERROR = 10,
    SO_PARSE_ERROR = 11,           /* errors.hpp:49  ParseError          */
    SO_UNSUPPORTED_FORMAT = 12     /* errors.hpp:44  UnsupportedFormat   */
} so_status;

/* formats.hpp:17-24 -- stable ids (model files, CSVs) */
typedef enum so_format {
    SO_COO = 0,
    SO_CSR = 1,
    SO_DIA = 2,
    SO_ELL = 3,
    SO_HYB = 4,
    SO_HDC = 5
} so_format;

/* formats.hpp:124-139 ConversionConfig */
typedef struct so_conversion_config {
    int64_t kh_override;       /* 0 selects ceil(nnz / nrows)            */
    double true_diag_ratio;    /* default 0.2                            */
    double max_padding_factor; /* default 10.0                           */
    int64_t max_padded_entries;/* >0 overrides the factor                */
} so_conversion_config;

/* features.hpp:12-23 FeatureVector (field order = struct order) */
typedef struct so_feature_vector {
    int64_t nrows, ncols, nnz;
    double avg_nnz_per_row, density;
    int64_t max_nnz_per_row, min_nnz_per_row;
    double nnz_row_spread;
    int64_t ndiags, ntrue_diags;
} so_feature_vector;

/* features.hpp:27-32 FeatureScanStats */
typedef struct so_scan_stats {
    int64_t entry_visits, structure_reads;
} so_scan_stats;

/* Shape of a device matrix (every field the host containers expose). */
typedef struct so_matrix_info {
    int32_t format;
    int32_t device;
    int64_t nrows, ncols, nnz;     /* nnz = DynamicMatrix::nnz() (formats.cpp:397-409) */
    int64_t coo_nnz;               /* COO, HYB coo part                       */
    int64_t csr_nnz;               /* CSR, HDC csr part                       */
    int64_t ndiags;                /* DIA, HDC dia part                       */
    int64_t dia_stored_nnz;
    int64_t ell_width;             /* ELL, HYB ell part (entries_per_row)     */
    int64_t ell_stored_nnz;
    int64_t kh;                    /* HYB configured K_H                      */
    int64_t true_diag_threshold;   /* HDC                                     */
} so_matrix_info;

/* Host arrays in the REFERENCE host layout (int64 indices, ELL row-major).
 * Unused slots may be NULL.  Sizes follow so_matrix_info. */
typedef struct so_host_arrays {
    int64_t* coo_row; int64_t* coo_col; double* coo_val;
    int64_t* csr_row_ptr; int64_t* csr_col; double* csr_val;
    int64_t* dia_offsets; double* dia_values;
    int64_t* ell_col; double* ell_val;
} so_host_arrays;

/* formats.hpp:55, model.hpp:40-53 TuneOutcome subset */
typedef struct so_tune_outcome {
    int32_t chosen;        /* FormatId                                 */
    int32_t source;        /* TunerKind: 1 decision_tree, 2 random_forest */
    int32_t switched;      /* chosen != active format                  */
    int32_t fallback_csr;  /* predicted format infeasible              */
    double feature_time_seconds; /* T_FE  (device time: %globaltimer at
                                    the first feature kernel's start ->
                                    after the finalize)                  */
    double predict_time_seconds; /* T_PRED (device time: finalize -> vote) */
    so_feature_vector features;  /* what the model saw                 */
    double wall_time_seconds;    /* host wall clock of the whole call
                                    (graph launch -> outcome on the host) */
} so_tune_outcome;

typedef struct so_matrix so_matrix; /* opaque, device-resident */
typedef struct so_forest so_forest; /* opaque, device-resident */

/* ---- context ----------------------------------------------------------- */
const char* so_last_error(void);
const char* so_version(void);
/* Number of kernels this library has launched in the process (monotone). */
int64_t so_kernel_launches(void);
so_status so_set_device(int device);          /* device for new objects */
so_status so_get_device(int* device);         /* the calling thread's current device */
so_status so_device_sync(void);
/* Opaque cudaStream_t used by every host-facing call on the current device. */
void* so_default_stream(void);

/* ---- containers: upload / download / info  (formats.hpp:37-122) --------- */
/* Host arrays are copied H2D; int64 indices are range-checked and narrowed on
 * the device.  No canonical check here (from_coo does it). */
so_status so_matrix_upload_coo(int64_t nrows, int64_t ncols, int64_t nnz,
                               const int64_t* row, const int64_t* col,
                               const double* val, so_matrix** out);
so_status so_matrix_upload_csr(int64_t nrows, int64_t ncols, int64_t nnz,
                               const int64_t* row_ptr, const int64_t* col,
                               const double* val, so_matrix** out);
so_status so_matrix_upload_dia(int64_t nrows, int64_t ncols, int64_t ndiags,
                               const int64_t* offsets, const double* values,
                               int64_t stored_nnz, so_matrix** out);
so_status so_matrix_upload_ell(int64_t nrows, int64_t ncols, int64_t width,
                               const int64_t* col_rowmajor,
                               const double* val_rowmajor, int64_t stored_nnz,
                               so_matrix** out);
so_status so_matrix_upload_hyb(int64_t nrows, int64_t ncols, int64_t width,
                               const int64_t* ell_col, const double* ell_val,
                               int64_t ell_stored_nnz, int64_t coo_nnz,
                               const int64_t* coo_row, const int64_t* coo_col,
                               const double* coo_val, int64_t kh,
                               so_matrix** out);
so_status so_matrix_upload_hdc(int64_t nrows, int64_t ncols, int64_t ndiags,
                               const int64_t* offsets, const double* values,
                               int64_t dia_stored_nnz, int64_t csr_nnz,
                               const int64_t* row_ptr, const int64_t* col,
                               const double* val, int64_t threshold,
                               so_matrix** out);
/* CooMatrix::from_triplets (formats.cpp:293-322) on the device: range check
 * (SO_INDEX_OUT_OF_RANGE), stable radix sort by (row, col), duplicates summed
 * in input order.  Result: canonical device COO. */
so_status so_coo_from_triplets(int64_t nrows, int64_t ncols, int64_t n,
                               const int64_t* row, const int64_t* col,
                               const double* val, so_matrix** out);
/* read_matrix_market (ingest.hpp:25, ingest.cpp:135-208): the reference's
 * accepted subset (matrix coordinate {real, integer, pattern} x {general,
 * symmetric}), 1-based -> 0-based, symmetric off-diagonals mirrored, pattern
 * values 1.0; same error types (SO_PARSE_ERROR "path:line: ...",
 * SO_UNSUPPORTED_FORMAT, SO_INDEX_OUT_OF_RANGE) and the same first error in
 * file order.  Parsed by all host threads, canonicalized on the device as
 * so_coo_from_triplets.  Result: canonical device COO. */
so_status so_read_matrix_market(const char* path, so_matrix** out);
/* write_matrix_market (ingest.hpp:29, ingest.cpp:210-224) of a canonical
 * COO matrix: 'real general', 1-based, shortest round-trip decimals. */
so_status so_write_matrix_market(const so_matrix* coo, const char* path);
/* CSR already in device memory (e.g. produced by a device generator or another
 * library): row_ptr int64[n+1], col int32[nnz], val f64[nnz], all device
 * pointers on the current device, fully written before the call (the copy
 * is ordered on the library stream, not the producer's).  Copied (D2D) and
 * validated; the caller keeps ownership of its buffers. */
so_status so_matrix_import_csr_device(int64_t nrows, int64_t ncols, int64_t nnz,
                                      const int64_t* row_ptr_dev,
                                      const int32_t* col_dev,
                                      const double* val_dev, so_matrix** out);
void so_matrix_free(so_matrix* m);
so_status so_matrix_info_get(const so_matrix* m, so_matrix_info* out);
/* D2H into caller buffers sized per so_matrix_info (ELL transposed back to
 * row-major, indices widened to int64). */
so_status so_matrix_download(const so_matrix* m, const so_host_arrays* out);

/* ---- conversions  (formats.cpp:411-467) ---------------------------------- */
/* from_coo: canonical check (InvalidInput), then the target's size phase,
 * the PaddingOverflow cap check BEFORE any dense allocation, then fill. */
so_status so_from_coo(const so_matrix* coo, int32_t target,
                      const so_conversion_config* cfg, so_matrix** out);
/* switch_format semantics: from_coo(to_coo(src), target) (formats.cpp:463-467),
 * done entirely on the device.  Same-format returns a deep copy. */
so_status so_convert(const so_matrix* src, int32_t target,
                     const so_conversion_config* cfg, so_matrix** out);
/* to_coo (formats.cpp:432-461): drop DIA zero cells / ELL sentinels, sort. */
so_status so_to_coo(const so_matrix* src, so_matrix** out);
/* format_feasible (tuners.cpp:26-45), host arithmetic on a feature vector. */
int32_t so_format_feasible(int32_t target, const so_feature_vector* f,
                           const so_conversion_config* cfg);

/* ---- SpMV  (spmv.hpp:20-32, spmv.cpp:191-246) ------------------------------ */
/* Device pointers, stream-ordered, no sync.  x has ncols, y has nrows slots;
 * x and y must not overlap (the kernels read x while y is written; the
 * reference API returns a fresh vector, so it never aliases). */
so_status so_spmv_device(const so_matrix* m, const double* x_dev, double* y_dev,
                         void* stream);
/* Row range [row_lo, row_hi) of y = A x only (DIA; the row-partitioned
 * halo iteration computes boundary rows, starts the exchange, then the
 * interior).  y_dev is indexed by matrix row.  Stream-ordered. */
so_status so_spmv_device_rows(const so_matrix* m, const double* x_dev, double* y_dev,
                              int64_t row_lo, int64_t row_hi, void* stream);
/* Row-partitioned iteration with the halo exchange fused into the multiply
 * (config 5; no reference counterpart -- the reference is single-node CPU):
 * rows [row_lo, row_hi) of y = A x are written to y_dev (indexed by matrix
 * row) AND to remote_dev[i - row_lo], a neighbour's window mapped with
 * so_ipc_open (NVLink peer memory).  When every CTA is done, the last one
 * stores flag_value to *remote_flag (release, system scope).  ticket_dev: a
 * zeroed device unsigned owned by this call site (left zeroed again).
 * DIA / pure-DIA HDC only.  Stream-ordered. */
so_status so_spmv_rows_push(const so_matrix* m, const double* x_dev, double* y_dev,
                            int64_t row_lo, int64_t row_hi, double* remote_dev,
                            unsigned* ticket_dev, unsigned long long* remote_flag,
                            unsigned long long flag_value, void* stream);
/* Stream-ordered wait until *flag_dev >= value (acquire, system scope);
 * pairs with so_spmv_rows_push on the neighbour. */
so_status so_wait_flag(const unsigned long long* flag_dev, unsigned long long value,
                       void* stream);
/* Waits that gave up after 60 s (a neighbour that never published) on the
 * current device since the library loaded; the iterate is then invalid. */
int64_t so_wait_flag_timeouts(void);
/* Peer-shareable device memory (cudaMalloc + CUDA IPC), zero-filled. */
typedef struct so_ipc_handle {
    unsigned char bytes[64];
} so_ipc_handle;
so_status so_ipc_alloc(int64_t bytes, void** dev_ptr, so_ipc_handle* handle);
so_status so_ipc_open(const so_ipc_handle* handle, void** dev_ptr);
so_status so_ipc_close(void* dev_ptr);
so_status so_ipc_free(void* dev_ptr);
/* spmv(m, x): host vectors, synchronous; y may alias x (y = A x of the
 * original x).  Pinned x and y on a DIA-window matrix: one zero-copy kernel
 * (narrow windows) or a chunked copy pipeline; otherwise H2D x, kernel(s),
 * D2H y. */
so_status so_spmv(const so_matrix* m, const double* x, int64_t xlen, double* y);
/* spmv(m, x) returning a NEW vector (spmv.hpp:20, spmv.cpp:203-219): the
 * library calls make_y(ctx, nrows) exactly once, on the calling thread, for
 * y's storage (NULL = out of memory) -- for a pageable x while host threads
 * stage x and the device multiplies, so building the caller's vector (its
 * value-initialisation) overlaps the work.  Same results as so_spmv. */
typedef double* (*so_make_output)(void* ctx, int64_t nrows);
so_status so_spmv_new(const so_matrix* m, const double* x, int64_t xlen, so_make_output make_y, void* ctx);
/* time_spmv: x uploaded once, 1 untimed warm-up, then `reps` multiplies each
 * timed with a cudaEvent pair on the launching stream.  total = sum. */
so_status so_time_spmv(const so_matrix* m, const double* x, int64_t xlen,
                       int64_t reps, double* per_rep_seconds,
                       double* total_seconds);
/* Algorithmic (compulsory) HBM bytes of one multiply, DESIGN.md §4. */
int64_t so_spmv_bytes(const so_matrix* m);

/* ---- features  (features.hpp:33-42, features.cpp:82-153) ------------------- */
so_status so_extract_features(const so_matrix* m, double true_diag_ratio,
                              so_feature_vector* out, so_scan_stats* stats);

/* ---- model  (model.hpp:18-53, model.cpp:202-228) --------------------------- */
/* kind 0 = tree (predict uses trees.front(), tuners.cpp:103-105), 1 = forest.
 * Flat nodes: tree t owns [node_off[t], node_off[t+1]); child indices are
 * tree-local.  feature == -1 marks a leaf. */
so_status so_forest_upload(int32_t kind, int32_t n_trees, const int64_t* node_off,
                           const int32_t* feature, const double* threshold,
                           const int32_t* left, const int32_t* right,
                           const int32_t* cls, so_forest** out);
void so_forest_free(so_forest* f);
/* predict on a host feature vector (one device launch). */
so_status so_predict(const so_forest* f, const so_feature_vector* x, int32_t* out);
/* Batched predict: rows is [n][10] in features_to_row order (throughput
 * path: one thread per (row, tree) over the flat node layout). */
so_status so_predict_rows(const so_forest* f, int64_t n, const double* rows,
                          int32_t* out);
/* The same prediction through the single-row latency path of so_tune_ml
 * (blocked layout, warp-cooperative walk, one CTA per row); a kind-0 (tree)
 * model evaluates its first tree only (tuners.cpp:103-105).  so_predict
 * uses it. */
so_status so_predict_rows_latency(const so_forest* f, int64_t n, const double* rows,
                                  int32_t* out);

/* ---- tuner  (tuners.hpp:57-63, tuners.cpp:92-114) ------------------------- */
/* tune_ml: features -> predict -> feasibility/CSR fallback fully on the device;
 * one small D2H of the outcome.  Never runs SpMV, never mutates m. */
so_status so_tune_ml(const so_matrix* m, const so_forest* f, double true_diag_ratio,
                     const so_conversion_config* cfg, so_tune_outcome* out);

/* ---- synthetic generators (device; bench / multi-GPU inputs) ------------- */
/* 27-point stencil on a g^3 grid (row-major z,y,x), restricted to global rows
 * [row_lo, row_hi) and global columns [col_lo, col_hi), as a DIA matrix of
 * (row_hi-row_lo) x (col_hi-col_lo) with offsets off + (row_lo - col_lo).
 * Values are a deterministic hash of (seed, global row, neighbour) in
 * +-[0.5, 2), so every row slice of the global matrix is consistent
 * (config 5: row-partitioned iteration). */
so_status so_gen_stencil27_dia(int64_t g, int64_t row_lo, int64_t row_hi,
                               int64_t col_lo, int64_t col_hi, uint64_t seed,
                               so_matrix** out);

/* ---- row-partitioned iterated SpMV across GPUs (config 5) ---
 * Replaces the reference's row-block partition of one multiply over
 * std::threads (spmv.cpp:142-189) with a row partition over ranks, one
 * process (or thread) per GPU; x <- A x iterated with the x exchange done by
 * the library's own kernels over NVLink peer memory (no collective).
 * Rank q owns global rows [row_starts[q], row_starts[q+1]).
 *   SO_DIST_HALO: `local` is the DIA-window block (rows owned) x (columns of
 *     the window [r0-halo, r1+halo) clipped to [0, n)); only halo rows move,
 *     pushed into the neighbours' windows by the boundary multiply itself.
 *   SO_DIST_ALLGATHER: `local` is (rows owned) x (all n columns), any format;
 *     every rank's new rows are stored into every peer's x (all-gather fused
 *     into the iteration's epilogue).
 * Setup: so_dist_create -> so_dist_handle (exchange the handles with any
 * transport, e.g. MPI_Allgather / torch all_gather_object) -> so_dist_connect
 * -> write the initial x into so_dist_x(d, 0) (the whole window / vector) ->
 * so_dist_iterate.  `local` must outlive the so_dist.  The P-rank iterate is
 * bitwise equal to the 1-rank iterate (row summation orders unchanged). */
enum { SO_DIST_HALO = 0, SO_DIST_ALLGATHER = 1 };
typedef struct so_dist so_dist;
so_status so_dist_create(const so_matrix* local, int32_t kind, int32_t rank, int32_t world,
                         const int64_t* row_starts, int64_t halo, so_dist** out);
/* this rank's shared block (both x buffers + flags), one CUDA IPC handle */
so_status so_dist_handle(const so_dist* d, so_ipc_handle* out);
/* handles[q] for every rank q (own entry ignored; HALO maps only neighbours) */
so_status so_dist_connect(so_dist* d, const so_ipc_handle* handles);
/* x buffer `which` (0/1; -1 = the one holding the latest iterate): device
 * pointer, global index of its first element, length */
so_status so_dist_x(const so_dist* d, int32_t which, double** x_dev, int64_t* offset,
                    int64_t* len);
/* enqueue `iters` iterations on `stream` (null: the library stream) */
so_status so_dist_iterate(so_dist* d, int64_t iters, void* stream);
/* peer waits that gave up after 60 s (a dead rank): nonzero = invalid iterate */
int64_t so_dist_timeouts(void);
void so_dist_free(so_dist* d);

#ifdef __cplusplus
}
#endif
#endif /* SPARSEORACLE_B200_H */
