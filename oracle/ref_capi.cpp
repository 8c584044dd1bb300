// TEST INFRASTRUCTURE ONLY -- part of the parity oracle, never the product.
//
// extern "C" shim around the UNMODIFIED reference C++ library
// (/root/reference/proj/src/{formats,spmv,features,model,tuners}.cpp, compiled
// in place by oracle/build_ref.sh with -Dsparseoracle=sparseoracle_ref).  It
// lets pytest (ctypes) and bench.py's reference arm drive the reference's own
// code path on the same inputs as the B200 library.  Only tests/, smoke() and
// bench.py's CPU-baseline leg load the resulting oracle/_ref/*.so.
//
// Every entry point catches the reference's exceptions and maps them to the
// same status codes the product C-ABI uses (include/sparseoracle_b200.h).

#include <cstdint>
#include <cstring>
#include <exception>
#include <new>
#include <string>
#include <vector>

#include "sparseoracle/features.hpp"
#include "sparseoracle/formats.hpp"
#include "sparseoracle/model.hpp"
#include "sparseoracle/rng.hpp"
#include "sparseoracle/spmv.hpp"
#include "sparseoracle/tuners.hpp"
#include "support/oracles.hpp"

using namespace sparseoracle;

namespace {

enum {
    ST_OK = 0,
    ST_INVALID_INPUT = 1,
    ST_PADDING_OVERFLOW = 2,
    ST_DIMENSION_MISMATCH = 3,
    ST_EMPTY_MATRIX = 4,
    ST_MALFORMED_MODEL = 5,
    ST_INDEX_OUT_OF_RANGE = 6,
    ST_ALL_FORMATS_INFEASIBLE = 7,
    ST_ERROR = 10,
};

thread_local std::string g_msg;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return ST_OK;
    } catch (const PaddingOverflow& e) {
        g_msg = e.what();
        return ST_PADDING_OVERFLOW;
    } catch (const InvalidInput& e) {
        g_msg = e.what();
        return ST_INVALID_INPUT;
    } catch (const DimensionMismatch& e) {
        g_msg = e.what();
        return ST_DIMENSION_MISMATCH;
    } catch (const EmptyMatrix& e) {
        g_msg = e.what();
        return ST_EMPTY_MATRIX;
    } catch (const MalformedModel& e) {
        g_msg = e.what();
        return ST_MALFORMED_MODEL;
    } catch (const IndexOutOfRange& e) {
        g_msg = e.what();
        return ST_INDEX_OUT_OF_RANGE;
    } catch (const AllFormatsInfeasible& e) {
        g_msg = e.what();
        return ST_ALL_FORMATS_INFEASIBLE;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return ST_ERROR;
    }
}

ConversionConfig make_cfg(int64_t kh_override, double ratio, double pad_factor,
                          int64_t max_padded) {
    ConversionConfig c;
    c.kh_override = kh_override;
    c.true_diag_ratio = ratio;
    c.max_padding_factor = pad_factor;
    c.max_padded_entries = max_padded;
    return c;
}

FeatureVector fv_from(const double* row) {
    std::array<double, kNumFeatures> r{};
    for (int i = 0; i < kNumFeatures; ++i) r[i] = row[i];
    return row_to_features(r);
}

void fv_to(const FeatureVector& f, double* out) {
    auto r = features_to_row(f);
    for (int i = 0; i < kNumFeatures; ++i) out[i] = r[i];
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_msg.c_str(); }

// ---- canonical COO -------------------------------------------------------

// from_triplets (sort + duplicate sum).  Returns a DynamicMatrix(COO) handle.
int ref_coo_from_triplets(int64_t nrows, int64_t ncols, int64_t n,
                          const int64_t* row, const int64_t* col,
                          const double* val, void** out) {
    return guard([&] {
        std::vector<Triplet> t(static_cast<std::size_t>(n));
        for (int64_t k = 0; k < n; ++k) t[k] = {row[k], col[k], val[k]};
        *out = new DynamicMatrix(CooMatrix::from_triplets(nrows, ncols, std::move(t)));
    });
}

// Wraps arrays as-is (no sort) -- used for non-canonical error tests.
int ref_coo_raw(int64_t nrows, int64_t ncols, int64_t n, const int64_t* row,
                const int64_t* col, const double* val, void** out) {
    return guard([&] {
        CooMatrix c;
        c.nrows = nrows;
        c.ncols = ncols;
        c.row_idx.assign(row, row + n);
        c.col_idx.assign(col, col + n);
        c.values.assign(val, val + n);
        *out = new DynamicMatrix(std::move(c));
    });
}

void ref_free(void* h) { delete static_cast<DynamicMatrix*>(h); }

int ref_clone(void* h, void** out) {
    return guard([&] { *out = new DynamicMatrix(*static_cast<DynamicMatrix*>(h)); });
}

int ref_format(void* h) { return static_cast<int>(static_cast<DynamicMatrix*>(h)->format()); }

void ref_dims(void* h, int64_t* dims3) {
    auto* m = static_cast<DynamicMatrix*>(h);
    dims3[0] = m->nrows();
    dims3[1] = m->ncols();
    dims3[2] = m->nnz();
}

// from_coo(to_coo(h)) -- h must currently hold canonical COO for from_coo; we
// call from_coo on the COO payload exactly as the reference API does.
int ref_from_coo(void* coo_h, int fmt, int64_t kh_override, double ratio,
                 double pad_factor, int64_t max_padded, void** out) {
    return guard([&] {
        auto* m = static_cast<DynamicMatrix*>(coo_h);
        *out = new DynamicMatrix(from_coo(m->as<CooMatrix>(), format_from_id(fmt),
                                          make_cfg(kh_override, ratio, pad_factor,
                                                   max_padded)));
    });
}

int ref_switch_format(void* h, int fmt, int64_t kh_override, double ratio,
                      double pad_factor, int64_t max_padded) {
    return guard([&] {
        switch_format(*static_cast<DynamicMatrix*>(h), format_from_id(fmt),
                      make_cfg(kh_override, ratio, pad_factor, max_padded));
    });
}

// to_coo -> new COO handle
int ref_to_coo(void* h, void** out) {
    return guard([&] { *out = new DynamicMatrix(to_coo(*static_cast<DynamicMatrix*>(h))); });
}

// Raw host-visible arrays of the active payload.  Pointers stay valid while
// the handle lives.  Layout (slot: meaning):
//   COO: a0 row, a1 col, a2 val
//   CSR: a0 row_ptr, a1 col, a2 val
//   DIA: a0 offsets, a1 values;           s0 stored_nnz
//   ELL: a0 col (row-major), a1 val;     s0 stored_nnz, s1 K
//   HYB: a0 ell col, a1 ell val, a2 coo row, a3 coo col, a4 coo val;
//        s0 ell stored_nnz, s1 ell K, s2 kh
//   HDC: a0 dia offsets, a1 dia values, a2 csr row_ptr, a3 csr col, a4 csr val;
//        s0 dia stored_nnz, s1 threshold
void ref_export(void* h, int64_t* scalars, const void** arrays, int64_t* lens) {
    auto* m = static_cast<DynamicMatrix*>(h);
    for (int i = 0; i < 8; ++i) {
        scalars[i] = 0;
        arrays[i] = nullptr;
        lens[i] = 0;
    }
    auto put = [&](int i, const auto& v) {
        arrays[i] = v.data();
        lens[i] = static_cast<int64_t>(v.size());
    };
    switch (m->format()) {
        case FormatId::coo: {
            const auto& c = m->as<CooMatrix>();
            put(0, c.row_idx); put(1, c.col_idx); put(2, c.values);
            break;
        }
        case FormatId::csr: {
            const auto& c = m->as<CsrMatrix>();
            put(0, c.row_ptr); put(1, c.col_idx); put(2, c.values);
            break;
        }
        case FormatId::dia: {
            const auto& d = m->as<DiaMatrix>();
            put(0, d.offsets); put(1, d.values);
            scalars[0] = d.stored_nnz;
            break;
        }
        case FormatId::ell: {
            const auto& e = m->as<EllMatrix>();
            put(0, e.col_idx); put(1, e.values);
            scalars[0] = e.stored_nnz;
            scalars[1] = e.entries_per_row;
            break;
        }
        case FormatId::hyb: {
            const auto& y = m->as<HybMatrix>();
            put(0, y.ell_part.col_idx); put(1, y.ell_part.values);
            put(2, y.coo_part.row_idx); put(3, y.coo_part.col_idx);
            put(4, y.coo_part.values);
            scalars[0] = y.ell_part.stored_nnz;
            scalars[1] = y.ell_part.entries_per_row;
            scalars[2] = y.kh;
            break;
        }
        case FormatId::hdc: {
            const auto& y = m->as<HdcMatrix>();
            put(0, y.dia_part.offsets); put(1, y.dia_part.values);
            put(2, y.csr_part.row_ptr); put(3, y.csr_part.col_idx);
            put(4, y.csr_part.values);
            scalars[0] = y.dia_part.stored_nnz;
            scalars[1] = y.true_diag_threshold;
            break;
        }
    }
}

// ---- SpMV ----------------------------------------------------------------

int ref_spmv(void* h, const double* x, int64_t xlen, double* y, int nthreads) {
    return guard([&] {
        auto* m = static_cast<DynamicMatrix*>(h);
        DenseVector xv(x, x + xlen);
        DenseVector yv = nthreads <= 1 ? spmv(*m, xv) : spmv_parallel(*m, xv, nthreads);
        std::memcpy(y, yv.data(), yv.size() * sizeof(double));
    });
}

int ref_time_spmv(void* h, const double* x, int64_t xlen, int64_t reps,
                  int nthreads, double* per_rep, double* total) {
    return guard([&] {
        auto* m = static_cast<DynamicMatrix*>(h);
        DenseVector xv(x, x + xlen);
        TimingSample s = time_spmv(*m, xv, reps, nthreads);
        for (int64_t r = 0; r < reps; ++r) per_rep[r] = s.per_rep_seconds[r];
        *total = s.total_seconds;
    });
}

// ---- features / model / tuners ---------------------------------------------

int ref_extract_features(void* h, double ratio, double* out10, int64_t* stats2) {
    return guard([&] {
        FeatureScanStats st;
        FeatureVector f = extract_features(*static_cast<DynamicMatrix*>(h), ratio, &st);
        fv_to(f, out10);
        stats2[0] = st.entry_visits;
        stats2[1] = st.structure_reads;
    });
}

// Flat forest: for tree t, nodes [node_off[t], node_off[t+1]).  Per node:
// feature, threshold, left, right, cls, counts[6].
int ref_forest_create(int kind, int n_trees, const int64_t* node_off,
                      const int32_t* feature, const double* threshold,
                      const int32_t* left, const int32_t* right,
                      const int32_t* cls, const int64_t* counts, void** out) {
    return guard([&] {
        auto* f = new ForestModel();
        f->kind = kind == 0 ? ModelKind::tree : ModelKind::forest;
        for (int t = 0; t < n_trees; ++t) {
            DecisionTreeModel tree;
            for (int64_t i = node_off[t]; i < node_off[t + 1]; ++i) {
                TreeNode n;
                n.feature_index = feature[i];
                n.threshold = threshold[i];
                n.left = left[i];
                n.right = right[i];
                n.predicted_class = cls[i];
                for (int c = 0; c < kNumFormats; ++c) n.class_counts[c] = counts[i * 6 + c];
                tree.nodes.push_back(n);
            }
            f->trees.push_back(std::move(tree));
        }
        *out = f;
    });
}

void ref_forest_free(void* f) { delete static_cast<ForestModel*>(f); }

int ref_load_model(const char* path, void** out) {
    return guard([&] { *out = new ForestModel(load_model(path)); });
}

int ref_save_model(void* f, const char* path) {
    return guard([&] { save_model(*static_cast<ForestModel*>(f), path); });
}

// Sizes of a loaded forest, then its flat arrays (same layout as create).
void ref_forest_shape(void* fh, int* kind, int* n_trees, int64_t* n_nodes) {
    auto* f = static_cast<ForestModel*>(fh);
    *kind = f->kind == ModelKind::tree ? 0 : 1;
    *n_trees = f->n_estimators();
    int64_t n = 0;
    for (const auto& t : f->trees) n += static_cast<int64_t>(t.nodes.size());
    *n_nodes = n;
}

void ref_forest_export(void* fh, int64_t* node_off, int32_t* feature,
                       double* threshold, int32_t* left, int32_t* right,
                       int32_t* cls, int64_t* counts, int32_t* depth) {
    auto* f = static_cast<ForestModel*>(fh);
    int64_t i = 0;
    for (int t = 0; t < f->n_estimators(); ++t) {
        node_off[t] = i;
        depth[t] = f->trees[t].depth;
        for (const TreeNode& n : f->trees[t].nodes) {
            feature[i] = n.feature_index;
            threshold[i] = n.threshold;
            left[i] = n.left;
            right[i] = n.right;
            cls[i] = n.predicted_class;
            for (int c = 0; c < kNumFormats; ++c) counts[i * 6 + c] = n.class_counts[c];
            ++i;
        }
    }
    node_off[f->n_estimators()] = i;
}

int ref_predict_tree(void* f, int tree, const double* row10) {
    auto* fm = static_cast<ForestModel*>(f);
    return static_cast<int>(predict_tree(fm->trees[tree], fv_from(row10)));
}

int ref_predict_forest(void* f, const double* row10) {
    return static_cast<int>(predict_forest(*static_cast<ForestModel*>(f), fv_from(row10)));
}

int ref_format_feasible(int fmt, const double* row10, int64_t kh_override,
                        double ratio, double pad_factor, int64_t max_padded) {
    return format_feasible(format_from_id(fmt), fv_from(row10),
                           make_cfg(kh_override, ratio, pad_factor, max_padded))
               ? 1
               : 0;
}

// outcome: [chosen, source, switched, fallback_csr]; times: [t_fe, t_pred]
int ref_tune_ml(void* h, void* forest, double ratio, int64_t kh_override,
                double pad_factor, int64_t max_padded, int32_t* outcome4,
                double* times2) {
    return guard([&] {
        TunerConfig cfg;
        cfg.true_diag_ratio = ratio;
        cfg.conversion = make_cfg(kh_override, ratio, pad_factor, max_padded);
        TuneOutcome o = tune_ml(*static_cast<DynamicMatrix*>(h), cfg,
                                *static_cast<ForestModel*>(forest));
        outcome4[0] = static_cast<int>(o.chosen);
        outcome4[1] = static_cast<int>(o.source);
        outcome4[2] = o.switched ? 1 : 0;
        outcome4[3] = o.fallback_csr ? 1 : 0;
        times2[0] = o.feature_time_seconds;
        times2[1] = o.predict_time_seconds;
    });
}

// tuner: 0 run_first, 1 decision_tree, 2 random_forest.  y has nrows slots.
int ref_tune_multiply(void* h, const double* x, int64_t xlen, int tuner,
                      void* forest, int64_t reps, int nthreads, double* y,
                      int32_t* outcome4) {
    return guard([&] {
        TunerConfig cfg;
        cfg.repetitions = reps;
        cfg.nthreads = nthreads;
        DenseVector xv(x, x + xlen);
        auto [yv, o] = tune_multiply(*static_cast<DynamicMatrix*>(h), xv,
                                     static_cast<TunerKind>(tuner), cfg,
                                     static_cast<ForestModel*>(forest));
        std::memcpy(y, yv.data(), yv.size() * sizeof(double));
        outcome4[0] = static_cast<int>(o.chosen);
        outcome4[1] = static_cast<int>(o.source);
        outcome4[2] = o.switched ? 1 : 0;
        outcome4[3] = o.fallback_csr ? 1 : 0;
    });
}

// ---- the reference test suite's seeded generators (tests/support/oracles.hpp)

void* ref_rng_new(uint64_t seed) { return new Rng(seed); }
void ref_rng_free(void* r) { delete static_cast<Rng*>(r); }
uint64_t ref_rng_next(void* r) { return static_cast<Rng*>(r)->next_u64(); }
double ref_rng_uniform_real(void* r, double lo, double hi) {
    return static_cast<Rng*>(r)->uniform_real(lo, hi);
}
uint64_t ref_rng_uniform_index(void* r, uint64_t n) {
    return static_cast<Rng*>(r)->uniform_index(n);
}
uint64_t ref_derive_seed(uint64_t seed, uint64_t stream) { return derive_seed(seed, stream); }

int ref_random_coo(void* r, int64_t max_dim, double min_d, double max_d, void** out) {
    return guard([&] {
        *out = new DynamicMatrix(
            testing::random_coo(*static_cast<Rng*>(r), max_dim, min_d, max_d));
    });
}

void ref_random_vector(void* r, int64_t n, double* out) {
    DenseVector v = testing::random_vector(*static_cast<Rng*>(r), n);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
}

int ref_band_matrix(int64_t n, int64_t half_band, void** out) {
    return guard([&] { *out = new DynamicMatrix(testing::band_matrix(n, half_band)); });
}

// Dense-scan feature oracle of the reference test suite (oracles.hpp:125-160).
int ref_dense_features(void* coo_h, double ratio, double* out10) {
    return guard([&] {
        const auto& c = static_cast<DynamicMatrix*>(coo_h)->as<CooMatrix>();
        fv_to(testing::dense_features(testing::dense_from_coo(c), ratio), out10);
    });
}

// Dense mat-vec oracle of the reference test suite (oracles.hpp:112-122).
int ref_dense_matvec(void* coo_h, const double* x, double* y) {
    return guard([&] {
        const auto& c = static_cast<DynamicMatrix*>(coo_h)->as<CooMatrix>();
        DenseVector xv(x, x + c.ncols);
        DenseVector yv = testing::dense_matvec(testing::dense_from_coo(c), xv);
        std::memcpy(y, yv.data(), yv.size() * sizeof(double));
    });
}

}  // extern "C"
