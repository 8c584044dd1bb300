/* TEST INFRASTRUCTURE ONLY -- the parity oracle, never the product.
 *
 * Plain-C restatement of the reference hot path (SpMV in six formats, the
 * canonical-COO -> format conversions, the ten-feature scan, tree/forest
 * predict, format_feasible) and of the reference test suite's seeded
 * generators.  Every function cites the /root/reference/proj file:line it
 * follows.  Index type is int64 throughout, exactly as the reference
 * (formats.hpp:15 `using index_t = std::int64_t`).
 *
 * Pinning: tests/test_oracle.py checks this restatement against (a) every
 * golden vector / known-answer test the reference's own suites hold
 * (test_formats.cpp, test_spmv.cpp, test_features.cpp, test_model.cpp,
 * test_tuners.cpp) and (b) the reference itself compiled in place into
 * oracle/_ref/ (oracle/Makefile), on the reference suites' seeded matrices.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library. */
#ifndef SPARSEORACLE_ORACLE_H
#define SPARSEORACLE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* same numbering as the product C-ABI (include/sparseoracle_b200.h) */
enum {
    OC_OK = 0,
    OC_INVALID_INPUT = 1,
    OC_PADDING_OVERFLOW = 2,
    OC_DIMENSION_MISMATCH = 3,
    OC_EMPTY_MATRIX = 4,
    OC_INDEX_OUT_OF_RANGE = 6,
};

enum { OC_COO = 0, OC_CSR = 1, OC_DIA = 2, OC_ELL = 3, OC_HYB = 4, OC_HDC = 5 };

/* ---- rng.hpp:12-56 ---------------------------------------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} oc_rng;

void oc_rng_seed(oc_rng* r, uint64_t seed);
uint64_t oc_rng_next(oc_rng* r);
uint64_t oc_rng_uniform_index(oc_rng* r, uint64_t n);
double oc_rng_uniform_real(oc_rng* r, double lo, double hi);
uint64_t oc_derive_seed(uint64_t seed, uint64_t stream);
int oc_rng_size(void);

/* tests/support/oracles.hpp:183-204.  Buffers need max_dim*max_dim slots. */
void oc_random_coo(oc_rng* r, int64_t max_dim, double min_d, double max_d,
                   int64_t* nrows, int64_t* ncols, int64_t* nnz, int64_t* row,
                   int64_t* col, double* val);
void oc_random_vector(oc_rng* r, int64_t n, double* out);

/* ---- formats.cpp ----------------------------------------------------- */
int oc_from_triplets(int64_t nrows, int64_t ncols, int64_t n, int64_t* row,
                     int64_t* col, double* val, int64_t* nnz_out);
int oc_is_canonical(int64_t nrows, int64_t ncols, int64_t z, const int64_t* row,
                    const int64_t* col);
int64_t oc_padded_entry_cap(double factor, int64_t max_padded, int64_t nnz);
int64_t oc_effective_kh(int64_t kh_override, int64_t nnz, int64_t nrows);
int64_t oc_true_diag_threshold(double ratio, int64_t nrows, int64_t ncols);

void oc_coo_to_csr(int64_t nrows, int64_t z, const int64_t* row, int64_t* row_ptr);
/* mask may be NULL (all entries); offsets needs nrows+ncols-1 slots */
int oc_dia_plan(int64_t nrows, int64_t ncols, int64_t z, const int64_t* row,
                const int64_t* col, const uint8_t* mask, int64_t cap,
                int64_t* ndiags, int64_t* offsets);
void oc_dia_fill(int64_t nrows, int64_t ncols, int64_t z, const int64_t* row,
                 const int64_t* col, const double* val, const uint8_t* mask,
                 int64_t ndiags, const int64_t* offsets, double* values,
                 int64_t* stored_nnz);
int oc_ell_plan(int64_t nrows, int64_t z, const int64_t* row, int64_t cap,
                int64_t* width);
void oc_ell_fill(int64_t nrows, int64_t z, const int64_t* row, const int64_t* col,
                 const double* val, int64_t width, int64_t* ell_col,
                 double* ell_val);
int oc_hyb_plan(int64_t nrows, int64_t z, const int64_t* row, int64_t kh,
                int64_t cap, int64_t* width, int64_t* coo_nnz);
void oc_hyb_fill(int64_t nrows, int64_t z, const int64_t* row, const int64_t* col,
                 const double* val, int64_t kh, int64_t width, int64_t* ell_col,
                 double* ell_val, int64_t* coo_row, int64_t* coo_col,
                 double* coo_val);
int oc_hdc_plan(int64_t nrows, int64_t ncols, int64_t z, const int64_t* row,
                const int64_t* col, int64_t threshold, int64_t cap,
                int64_t* ndiags, int64_t* offsets, int64_t* csr_nnz);
void oc_hdc_fill(int64_t nrows, int64_t ncols, int64_t z, const int64_t* row,
                 const int64_t* col, const double* val, int64_t threshold,
                 int64_t ndiags, const int64_t* offsets, double* dia_values,
                 int64_t* dia_stored_nnz, int64_t* csr_row_ptr, int64_t* csr_col,
                 double* csr_val);

/* ---- spmv.cpp:21-108 (y is zero-filled first, spmv.cpp:193) ---------- */
void oc_spmv_coo(int64_t nrows, int64_t z, const int64_t* row, const int64_t* col,
                 const double* val, const double* x, double* y, int accumulate);
void oc_spmv_csr(int64_t nrows, const int64_t* row_ptr, const int64_t* col,
                 const double* val, const double* x, double* y, int accumulate);
void oc_spmv_dia(int64_t nrows, int64_t ncols, int64_t ndiags, const int64_t* offsets,
                 const double* values, const double* x, double* y, int accumulate);
void oc_spmv_ell(int64_t nrows, int64_t width, const int64_t* col, const double* val,
                 const double* x, double* y, int accumulate);

/* ---- features.cpp:10-153.  out10 in features_to_row order ------------- */
typedef struct {
    int format;
    int64_t nrows, ncols;
    /* COO / HYB-coo part */
    int64_t coo_nnz;
    const int64_t *coo_row, *coo_col;
    /* CSR / HDC-csr part */
    const int64_t *csr_row_ptr, *csr_col;
    /* DIA / HDC-dia part */
    int64_t ndiags;
    const int64_t* offsets;
    const double* dia_values;
    /* ELL / HYB-ell part (row-major) */
    int64_t width;
    const int64_t* ell_col;
} oc_matrix_view;

int oc_extract_features(const oc_matrix_view* m, double ratio, double* out10,
                        int64_t* stats2);

/* ---- model.cpp:202-228, tuners.cpp:26-45 ------------------------------- */
int oc_predict_tree(const int32_t* feature, const double* threshold,
                    const int32_t* left, const int32_t* right, const int32_t* cls,
                    const double* row10);
int oc_predict_forest(int n_trees, const int64_t* node_off, const int32_t* feature,
                      const double* threshold, const int32_t* left,
                      const int32_t* right, const int32_t* cls, const double* row10);
int oc_format_feasible(int fmt, const double* row10, int64_t kh_override,
                       double pad_factor, int64_t max_padded);

#ifdef __cplusplus
}
#endif
#endif
