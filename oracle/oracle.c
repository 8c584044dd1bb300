/* TEST INFRASTRUCTURE ONLY -- the parity oracle, never the product.
 * Plain-C restatement of the reference hot path; see oracle.h for the pinning
 * story.  Compiled with -ffp-contract=off: the reference is built with
 * -O3 -DNDEBUG and no -march (proj/CMakeLists.txt:8-10), i.e. x86-64
 * baseline without FMA, so every a*b+c below is two roundings. */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ===================== rng.hpp:12-56 (std::mt19937_64) ===================== */

#define MT_N 312
#define MT_M 156

void oc_rng_seed(oc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
}

int oc_rng_size(void) { return (int)sizeof(oc_rng); }

uint64_t oc_rng_next(oc_rng* r) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    if (r->idx >= MT_N) {
        for (int i = 0; i < MT_N; ++i) {
            uint64_t y = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
            uint64_t v = r->mt[(i + MT_M) % MT_N] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = v;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* rng.hpp:19-27 rejection sampling */
uint64_t oc_rng_uniform_index(oc_rng* r, uint64_t n) {
    uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t v;
    do {
        v = oc_rng_next(r);
    } while (v >= limit);
    return v % n;
}

/* rng.hpp:30-36 */
double oc_rng_uniform_real(oc_rng* r, double lo, double hi) {
    double u = (double)(oc_rng_next(r) >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u;
}

/* rng.hpp:51-56 splitmix64 */
uint64_t oc_derive_seed(uint64_t seed, uint64_t stream) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* ========== triplet sort (formats.cpp:249-252 / 303-306 order) ========== */

typedef struct {
    int64_t row, col;
    double val;
} trip;

static void merge_sort(trip* a, trip* tmp, int64_t n) {
    /* stable bottom-up merge sort by (row, col) */
    for (int64_t w = 1; w < n; w *= 2) {
        for (int64_t lo = 0; lo < n; lo += 2 * w) {
            int64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            int64_t i = lo, j = mid, k = lo;
            while (i < mid && j < hi) {
                int take_right = a[j].row < a[i].row || (a[j].row == a[i].row && a[j].col < a[i].col);
                tmp[k++] = take_right ? a[j++] : a[i++];
            }
            while (i < mid) tmp[k++] = a[i++];
            while (j < hi) tmp[k++] = a[j++];
        }
        memcpy(a, tmp, (size_t)n * sizeof(trip));
    }
}

/* formats.cpp:293-322: range check, sort, sum duplicates in sorted order.
 * The reference uses std::sort (tie order unspecified); this oracle is stable. */
int oc_from_triplets(int64_t nrows, int64_t ncols, int64_t n, int64_t* row,
                     int64_t* col, double* val, int64_t* nnz_out) {
    for (int64_t k = 0; k < n; ++k)
        if (row[k] < 0 || row[k] >= nrows || col[k] < 0 || col[k] >= ncols)
            return OC_INDEX_OUT_OF_RANGE;
    trip* a = (trip*)malloc((size_t)(n > 0 ? n : 1) * sizeof(trip));
    trip* t = (trip*)malloc((size_t)(n > 0 ? n : 1) * sizeof(trip));
    for (int64_t k = 0; k < n; ++k) a[k] = (trip){row[k], col[k], val[k]};
    merge_sort(a, t, n);
    int64_t z = 0;
    for (int64_t k = 0; k < n; ++k) {
        if (z > 0 && row[z - 1] == a[k].row && col[z - 1] == a[k].col) {
            val[z - 1] += a[k].val;
        } else {
            row[z] = a[k].row;
            col[z] = a[k].col;
            val[z] = a[k].val;
            ++z;
        }
    }
    free(a);
    free(t);
    *nnz_out = z;
    return OC_OK;
}

/* ===================== oracles.hpp:176-223 generators ===================== */

static double random_value(oc_rng* r) { /* oracles.hpp:178-181 */
    double v = oc_rng_uniform_real(r, 0.5, 2.0);
    return oc_rng_next(r) % 2 == 0 ? v : -v;
}

void oc_random_coo(oc_rng* r, int64_t max_dim, double min_d, double max_d,
                   int64_t* nrows_out, int64_t* ncols_out, int64_t* nnz, int64_t* row,
                   int64_t* col, double* val) {
    int64_t nrows = 1 + (int64_t)oc_rng_uniform_index(r, (uint64_t)max_dim);
    int64_t ncols = 1 + (int64_t)oc_rng_uniform_index(r, (uint64_t)max_dim);
    double density = oc_rng_uniform_real(r, min_d, max_d);
    int64_t target = (int64_t)(density * (double)nrows * (double)ncols);
    int64_t cells_n = nrows * ncols;
    uint64_t* cells = (uint64_t*)malloc((size_t)cells_n * sizeof(uint64_t));
    for (int64_t i = 0; i < cells_n; ++i) cells[i] = (uint64_t)i;
    for (int64_t i = cells_n; i > 1; --i) { /* rng.hpp:40-44 Fisher-Yates */
        uint64_t j = oc_rng_uniform_index(r, (uint64_t)i);
        uint64_t tmp = cells[i - 1];
        cells[i - 1] = cells[j];
        cells[j] = tmp;
    }
    int64_t take = target < cells_n ? target : cells_n;
    for (int64_t k = 0; k < take; ++k) {
        int64_t cell = (int64_t)cells[k];
        row[k] = cell / ncols;
        col[k] = cell % ncols;
        val[k] = random_value(r);
    }
    free(cells);
    oc_from_triplets(nrows, ncols, take, row, col, val, nnz);
    *nrows_out = nrows;
    *ncols_out = ncols;
}

void oc_random_vector(oc_rng* r, int64_t n, double* out) { /* oracles.hpp:219-223 */
    for (int64_t i = 0; i < n; ++i) out[i] = oc_rng_uniform_real(r, -1.0, 1.0);
}

/* ===================== formats.cpp conversions ===================== */

/* formats.cpp:324-340 */
int oc_is_canonical(int64_t nrows, int64_t ncols, int64_t z, const int64_t* row,
                    const int64_t* col) {
    if (nrows < 0 || ncols < 0) return 0;
    for (int64_t k = 0; k < z; ++k) {
        if (row[k] < 0 || row[k] >= nrows || col[k] < 0 || col[k] >= ncols) return 0;
        if (k > 0 && !(row[k - 1] < row[k] || (row[k - 1] == row[k] && col[k - 1] < col[k])))
            return 0;
    }
    return 1;
}

/* formats.cpp:348-355 */
int64_t oc_padded_entry_cap(double factor, int64_t max_padded, int64_t nnz) {
    if (max_padded > 0) return max_padded;
    double cap = factor * (double)nnz;
    if (cap >= (double)INT64_MAX) return INT64_MAX;
    return (int64_t)cap;
}

/* formats.cpp:357-361 */
int64_t oc_effective_kh(int64_t kh_override, int64_t nnz, int64_t nrows) {
    if (kh_override > 0) return kh_override;
    if (nrows <= 0 || nnz <= 0) return 0;
    return (nnz + nrows - 1) / nrows;
}

/* formats.cpp:363-367 */
int64_t oc_true_diag_threshold(double ratio, int64_t nrows, int64_t ncols) {
    double len = (double)(nrows < ncols ? nrows : ncols);
    return (int64_t)ceil(ratio * len);
}

/* formats.cpp:14-20 */
static int64_t checked_mul(int64_t a, int64_t b) {
    if (a == 0 || b == 0) return 0;
    if (a > INT64_MAX / b) return INT64_MAX;
    return a * b;
}

/* formats.cpp:45-60 */
void oc_coo_to_csr(int64_t nrows, int64_t z, const int64_t* row, int64_t* row_ptr) {
    memset(row_ptr, 0, (size_t)(nrows + 1) * sizeof(int64_t));
    for (int64_t k = 0; k < z; ++k) row_ptr[row[k] + 1]++;
    for (int64_t i = 0; i < nrows; ++i) row_ptr[i + 1] += row_ptr[i];
}

/* formats.cpp:64-82 (offset discovery + cap check, before allocation) */
int oc_dia_plan(int64_t nrows, int64_t ncols, int64_t z, const int64_t* row,
                const int64_t* col, const uint8_t* mask, int64_t cap, int64_t* ndiags,
                int64_t* offsets) {
    int64_t nk = nrows + ncols;
    uint8_t* seen = (uint8_t*)calloc((size_t)(nk > 0 ? nk : 1), 1);
    for (int64_t k = 0; k < z; ++k)
        if (!mask || mask[k]) seen[col[k] - row[k] + nrows - 1] = 1;
    int64_t d = 0;
    for (int64_t key = 0; key < nrows + ncols - 1 && nrows > 0 && ncols > 0; ++key)
        if (seen[key]) offsets[d++] = key - (nrows - 1);
    free(seen);
    *ndiags = d;
    return checked_mul(d, nrows) > cap ? OC_PADDING_OVERFLOW : OC_OK;
}

/* formats.cpp:84-95 */
void oc_dia_fill(int64_t nrows, int64_t ncols, int64_t z, const int64_t* row,
                 const int64_t* col, const double* val, const uint8_t* mask,
                 int64_t ndiags, const int64_t* offsets, double* values,
                 int64_t* stored_nnz) {
    int64_t nk = nrows + ncols;
    int64_t* slot = (int64_t*)malloc((size_t)(nk > 0 ? nk : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < nk; ++i) slot[i] = -1;
    for (int64_t d = 0; d < ndiags; ++d) slot[offsets[d] + nrows - 1] = d;
    memset(values, 0, (size_t)(ndiags * nrows) * sizeof(double));
    int64_t s = 0;
    for (int64_t k = 0; k < z; ++k) {
        if (mask && !mask[k]) continue;
        int64_t d = slot[col[k] - row[k] + nrows - 1];
        values[d * nrows + row[k]] = val[k];
        if (val[k] != 0.0) s++;
    }
    free(slot);
    *stored_nnz = s;
}

/* formats.cpp:132-138 + 111-112 */
int oc_ell_plan(int64_t nrows, int64_t z, const int64_t* row, int64_t cap, int64_t* width) {
    int64_t* cnt = (int64_t*)calloc((size_t)(nrows > 0 ? nrows : 1), sizeof(int64_t));
    for (int64_t k = 0; k < z; ++k) cnt[row[k]]++;
    int64_t w = 0;
    for (int64_t i = 0; i < nrows; ++i)
        if (cnt[i] > w) w = cnt[i];
    free(cnt);
    *width = w;
    return checked_mul(w, nrows) > cap ? OC_PADDING_OVERFLOW : OC_OK;
}

/* formats.cpp:109-130 (row-major slot i*K + fill) */
void oc_ell_fill(int64_t nrows, int64_t z, const int64_t* row, const int64_t* col,
                 const double* val, int64_t width, int64_t* ell_col, double* ell_val) {
    int64_t n = width * nrows;
    for (int64_t s = 0; s < n; ++s) {
        ell_col[s] = -1;
        ell_val[s] = 0.0;
    }
    int64_t* fill = (int64_t*)calloc((size_t)(nrows > 0 ? nrows : 1), sizeof(int64_t));
    for (int64_t k = 0; k < z; ++k) {
        int64_t s = row[k] * width + fill[row[k]]++;
        ell_col[s] = col[k];
        ell_val[s] = val[k];
    }
    free(fill);
}

/* formats.cpp:140-172 split rule: the first kh entries of a row -> ELL */
int oc_hyb_plan(int64_t nrows, int64_t z, const int64_t* row, int64_t kh, int64_t cap,
                int64_t* width, int64_t* coo_nnz) {
    int64_t w = 0, fillc = 0, prev = -1, surplus = 0;
    for (int64_t k = 0; k < z; ++k) {
        if (row[k] != prev) {
            prev = row[k];
            fillc = 0;
        }
        if (!(fillc < kh)) surplus++;
        ++fillc;
        if (fillc <= kh && fillc > w) w = fillc;
    }
    *width = w;
    *coo_nnz = surplus;
    return checked_mul(w, nrows) > cap ? OC_PADDING_OVERFLOW : OC_OK;
}

void oc_hyb_fill(int64_t nrows, int64_t z, const int64_t* row, const int64_t* col,
                 const double* val, int64_t kh, int64_t width, int64_t* ell_col,
                 double* ell_val, int64_t* coo_row, int64_t* coo_col, double* coo_val) {
    int64_t n = width * nrows;
    for (int64_t s = 0; s < n; ++s) {
        ell_col[s] = -1;
        ell_val[s] = 0.0;
    }
    int64_t fillc = 0, prev = -1, c = 0;
    for (int64_t k = 0; k < z; ++k) {
        if (row[k] != prev) {
            prev = row[k];
            fillc = 0;
        }
        if (fillc < kh) {
            int64_t s = row[k] * width + fillc;
            ell_col[s] = col[k];
            ell_val[s] = val[k];
        } else {
            coo_row[c] = row[k];
            coo_col[c] = col[k];
            coo_val[c] = val[k];
            ++c;
        }
        ++fillc;
    }
}

/* formats.cpp:174-205 */
static int64_t* hdc_diag_counts(int64_t nrows, int64_t ncols, int64_t z,
                                const int64_t* row, const int64_t* col) {
    int64_t nk = nrows + ncols;
    int64_t* cnt = (int64_t*)calloc((size_t)(nk > 0 ? nk : 1), sizeof(int64_t));
    for (int64_t k = 0; k < z; ++k) cnt[col[k] - row[k] + nrows - 1]++;
    return cnt;
}

static uint8_t* hdc_mask(int64_t nrows, int64_t ncols, int64_t z, const int64_t* row,
                         const int64_t* col, int64_t threshold, int64_t* n_in) {
    int64_t* cnt = hdc_diag_counts(nrows, ncols, z, row, col);
    uint8_t* mask = (uint8_t*)malloc((size_t)(z > 0 ? z : 1));
    int64_t c = 0;
    for (int64_t k = 0; k < z; ++k) {
        mask[k] = cnt[col[k] - row[k] + nrows - 1] >= threshold;
        c += mask[k];
    }
    free(cnt);
    *n_in = c;
    return mask;
}

int oc_hdc_plan(int64_t nrows, int64_t ncols, int64_t z, const int64_t* row,
                const int64_t* col, int64_t threshold, int64_t cap, int64_t* ndiags,
                int64_t* offsets, int64_t* csr_nnz) {
    int64_t n_in;
    uint8_t* mask = hdc_mask(nrows, ncols, z, row, col, threshold, &n_in);
    int st = oc_dia_plan(nrows, ncols, z, row, col, mask, cap, ndiags, offsets);
    free(mask);
    *csr_nnz = z - n_in;
    return st;
}

void oc_hdc_fill(int64_t nrows, int64_t ncols, int64_t z, const int64_t* row,
                 const int64_t* col, const double* val, int64_t threshold,
                 int64_t ndiags, const int64_t* offsets, double* dia_values,
                 int64_t* dia_stored_nnz, int64_t* csr_row_ptr, int64_t* csr_col,
                 double* csr_val) {
    int64_t n_in;
    uint8_t* mask = hdc_mask(nrows, ncols, z, row, col, threshold, &n_in);
    oc_dia_fill(nrows, ncols, z, row, col, val, mask, ndiags, offsets, dia_values,
                dia_stored_nnz);
    memset(csr_row_ptr, 0, (size_t)(nrows + 1) * sizeof(int64_t));
    int64_t c = 0;
    for (int64_t k = 0; k < z; ++k) {
        if (mask[k]) continue;
        csr_row_ptr[row[k] + 1]++;
        csr_col[c] = col[k];
        csr_val[c] = val[k];
        ++c;
    }
    for (int64_t i = 0; i < nrows; ++i) csr_row_ptr[i + 1] += csr_row_ptr[i];
    free(mask);
}

/* ===================== spmv.cpp:21-108 ===================== */

static void zero_y(int64_t n, double* y, int accumulate) {
    if (!accumulate) /* multiply_into: std::fill(y, 0), spmv.cpp:193 */
        for (int64_t i = 0; i < n; ++i) y[i] = 0.0;
}

void oc_spmv_coo(int64_t nrows, int64_t z, const int64_t* row, const int64_t* col,
                 const double* val, const double* x, double* y, int accumulate) {
    zero_y(nrows, y, accumulate);
    for (int64_t k = 0; k < z; ++k) y[row[k]] += val[k] * x[col[k]]; /* :21-28 */
}

void oc_spmv_csr(int64_t nrows, const int64_t* row_ptr, const int64_t* col,
                 const double* val, const double* x, double* y, int accumulate) {
    zero_y(nrows, y, accumulate);
    for (int64_t i = 0; i < nrows; ++i) { /* :30-41 */
        double sum = 0.0;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) sum += val[k] * x[col[k]];
        y[i] += sum;
    }
}

void oc_spmv_dia(int64_t nrows, int64_t ncols, int64_t ndiags, const int64_t* offsets,
                 const double* values, const double* x, double* y, int accumulate) {
    zero_y(nrows, y, accumulate);
    for (int64_t d = 0; d < ndiags; ++d) { /* :45-56 */
        int64_t off = offsets[d];
        int64_t lo = 0 > -off ? 0 : -off;
        int64_t hi = nrows < ncols - off ? nrows : ncols - off;
        const double* diag = values + d * nrows;
        for (int64_t i = lo; i < hi; ++i) y[i] += diag[i] * x[i + off];
    }
}

void oc_spmv_ell(int64_t nrows, int64_t width, const int64_t* col, const double* val,
                 const double* x, double* y, int accumulate) {
    zero_y(nrows, y, accumulate);
    for (int64_t i = 0; i < nrows; ++i) { /* :59-71 */
        double sum = 0.0;
        for (int64_t k = 0; k < width; ++k) {
            int64_t c = col[i * width + k];
            if (c == -1) break;
            sum += val[i * width + k] * x[c];
        }
        y[i] += sum;
    }
}

/* ===================== features.cpp:10-153 ===================== */

typedef struct {
    int64_t* row_counts;
    int64_t* diag_counts;
    int64_t nrows;
    int64_t visits, structure;
} scan_acc;

static void visit(scan_acc* a, int64_t r, int64_t c) { /* :22-26 */
    a->row_counts[r]++;
    a->diag_counts[c - r + a->nrows - 1]++;
    a->visits++;
}

static void scan_coo(scan_acc* a, int64_t z, const int64_t* row, const int64_t* col) {
    for (int64_t k = 0; k < z; ++k) visit(a, row[k], col[k]); /* :33-38 */
}

static void scan_csr(scan_acc* a, int64_t n, const int64_t* rp, const int64_t* col) {
    for (int64_t i = 0; i < n; ++i) /* :40-47 */
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) visit(a, i, col[k]);
}

static void scan_dia(scan_acc* a, int64_t n, int64_t m, int64_t nd, const int64_t* off,
                     const double* v) {
    for (int64_t d = 0; d < nd; ++d) { /* :51-64, only v != 0.0 counts */
        int64_t o = off[d];
        int64_t lo = 0 > -o ? 0 : -o, hi = n < m - o ? n : m - o;
        for (int64_t i = lo; i < hi; ++i) {
            if (v[d * n + i] != 0.0)
                visit(a, i, i + o);
            else
                a->structure++;
        }
    }
}

static void scan_ell(scan_acc* a, int64_t n, int64_t w, const int64_t* col) {
    for (int64_t i = 0; i < n; ++i) /* :66-78 */
        for (int64_t k = 0; k < w; ++k) {
            int64_t c = col[i * w + k];
            if (c == -1) {
                a->structure++;
                break;
            }
            visit(a, i, c);
        }
}

int oc_extract_features(const oc_matrix_view* m, double ratio, double* out10,
                        int64_t* stats2) {
    int64_t n = m->nrows, nc = m->ncols;
    if (n < 1 || nc < 1) return OC_EMPTY_MATRIX; /* :86-88 */
    if (!(ratio > 0.0) || ratio > 1.0) return OC_INVALID_INPUT; /* :89-91 */
    scan_acc a;
    a.row_counts = (int64_t*)calloc((size_t)n, sizeof(int64_t));
    a.diag_counts = (int64_t*)calloc((size_t)(n + nc), sizeof(int64_t));
    a.nrows = n;
    a.visits = a.structure = 0;
    switch (m->format) {
        case OC_COO: scan_coo(&a, m->coo_nnz, m->coo_row, m->coo_col); break;
        case OC_CSR: scan_csr(&a, n, m->csr_row_ptr, m->csr_col); break;
        case OC_DIA: scan_dia(&a, n, nc, m->ndiags, m->offsets, m->dia_values); break;
        case OC_ELL: scan_ell(&a, n, m->width, m->ell_col); break;
        case OC_HYB:
            scan_ell(&a, n, m->width, m->ell_col);
            scan_coo(&a, m->coo_nnz, m->coo_row, m->coo_col);
            break;
        case OC_HDC:
            scan_dia(&a, n, nc, m->ndiags, m->offsets, m->dia_values);
            scan_csr(&a, n, m->csr_row_ptr, m->csr_col);
            break;
    }
    /* :121-144 */
    int64_t z = 0, mx = 0, mn = a.row_counts[0];
    for (int64_t i = 0; i < n; ++i) {
        int64_t c = a.row_counts[i];
        z += c;
        if (c > mx) mx = c;
        if (c < mn) mn = c;
    }
    double avg = (double)z / (double)n;
    double density = (double)z / ((double)n * (double)nc);
    double sq = 0.0;
    for (int64_t i = 0; i < n; ++i) { /* sequential, :139-143 */
        double dev = (double)a.row_counts[i] - avg;
        sq += dev * dev;
    }
    double spread = sq / (double)n;
    int64_t thr = (int64_t)ceil(ratio * (double)(n < nc ? n : nc)); /* :146-147 */
    int64_t nd = 0, ntd = 0;
    for (int64_t k = 0; k < n + nc; ++k) {
        if (a.diag_counts[k] >= 1) nd++;
        if (a.diag_counts[k] >= thr) ntd++;
    }
    /* features_to_row order, features.cpp:155-166 */
    out10[0] = (double)n;
    out10[1] = (double)nc;
    out10[2] = (double)z;
    out10[3] = avg;
    out10[4] = density;
    out10[5] = (double)mx;
    out10[6] = (double)mn;
    out10[7] = spread;
    out10[8] = (double)nd;
    out10[9] = (double)ntd;
    if (stats2) {
        stats2[0] = a.visits;
        stats2[1] = a.structure;
    }
    free(a.row_counts);
    free(a.diag_counts);
    return OC_OK;
}

/* ===================== model.cpp:202-228 ===================== */

int oc_predict_tree(const int32_t* feature, const double* threshold, const int32_t* left,
                    const int32_t* right, const int32_t* cls, const double* row10) {
    int32_t node = 0;
    while (feature[node] != -1) node = row10[feature[node]] <= threshold[node] ? left[node] : right[node];
    return cls[node];
}

int oc_predict_forest(int n_trees, const int64_t* node_off, const int32_t* feature,
                      const double* threshold, const int32_t* left, const int32_t* right,
                      const int32_t* cls, const double* row10) {
    int votes[6] = {0, 0, 0, 0, 0, 0};
    for (int t = 0; t < n_trees; ++t) {
        int64_t b = node_off[t];
        votes[oc_predict_tree(feature + b, threshold + b, left + b, right + b, cls + b, row10)]++;
    }
    int best = 0;
    for (int c = 1; c < 6; ++c)
        if (votes[c] > votes[best]) best = c;
    return best;
}

/* ===================== tuners.cpp:26-45 ===================== */

int oc_format_feasible(int fmt, const double* row10, int64_t kh_override, double pad_factor,
                       int64_t max_padded) {
    /* row_to_features (features.cpp:168-181) casts back to index_t */
    int64_t nrows = (int64_t)row10[0], nnz = (int64_t)row10[2];
    int64_t mx = (int64_t)row10[5], nd = (int64_t)row10[8], ntd = (int64_t)row10[9];
    int64_t cap = oc_padded_entry_cap(pad_factor, max_padded, nnz);
    switch (fmt) {
        case OC_COO:
        case OC_CSR: return 1;
        case OC_DIA: return nd * nrows <= cap;
        case OC_ELL: return mx * nrows <= cap;
        case OC_HYB: {
            int64_t kh = oc_effective_kh(kh_override, nnz, nrows);
            return (kh < mx ? kh : mx) * nrows <= cap;
        }
        case OC_HDC: return ntd * nrows <= cap;
    }
    return 0;
}
