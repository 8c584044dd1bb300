// TEST INFRASTRUCTURE ONLY -- extern "C" shim over the reference's pipeline /
// trainer / CSV wire formats (src/pipeline.cpp, src/trainer.cpp,
// src/ingest.cpp compiled in place, namespace renamed to sparseoracle_ref).
// Lets tests and tools feed B200 profiling CSVs to the reference trainer
// (cmd_train, pipeline.cpp:190-252) and read them back with the reference's
// own parsers (ingest.cpp:419-470).
#include <cstdint>
#include <cstring>
#include <string>

#include "sparseoracle/ingest.hpp"
#include "sparseoracle/pipeline.hpp"

namespace {
thread_local std::string g_err;
template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
}  // namespace

extern "C" {

const char* refp_last_error(void) { return g_err.c_str(); }

// cmd_train(features_csv + profiles_csv -> model_out), default CLI grid.
int refp_cmd_train(const char* features_csv, const char* profiles_csv, const char* model_out, uint64_t seed,
                   int folds, double* heldout_acc, double* heldout_bacc, int64_t* n_train, int64_t* n_test) {
    return guard([&] {
        sparseoracle::TrainOptions o;
        o.features_csv = features_csv;
        o.profiles_csv = std::filesystem::path(profiles_csv);
        o.model_out = model_out;
        o.split_seed = seed;
        o.folds = folds;
        o.backend_label = "b200-sm_100a";
        const sparseoracle::TrainResult r = sparseoracle::cmd_train(o);
        *heldout_acc = r.heldout.accuracy;
        *heldout_bacc = r.heldout.balanced_accuracy;
        *n_train = int64_t(r.n_train);
        *n_test = int64_t(r.n_test);
    });
}

// Parse a profile CSV with the reference reader: number of records, and the
// (format, repetitions, total_seconds, feasible) of record i (i < 0: count only).
int refp_read_profile_csv(const char* path, int64_t i, int64_t* count, int32_t* format, int64_t* reps,
                          double* total_seconds, int32_t* feasible) {
    return guard([&] {
        const auto recs = sparseoracle::read_profile_csv(path);
        *count = int64_t(recs.size());
        if (i >= 0 && i < int64_t(recs.size())) {
            const auto& r = recs[size_t(i)];
            *format = int32_t(r.format);
            *reps = r.repetitions;
            *total_seconds = r.total_seconds;
            *feasible = r.feasible ? 1 : 0;
        }
    });
}

// Join features + profiles into a training CSV (build_training_csv):
// rows written and rows skipped.
int refp_build_training_csv(const char* features_csv, const char* profiles_csv, const char* out_csv,
                            int64_t* written, int64_t* skipped) {
    return guard([&] {
        const auto r = sparseoracle::build_training_csv(sparseoracle::read_feature_csv(features_csv),
                                                        sparseoracle::read_profile_csv(profiles_csv), out_csv);
        *written = int64_t(r.rows_written);
        *skipped = int64_t(r.skipped.size());
    });
}

// read_matrix_market through the reference (ingest.cpp:135-208).  kind: 0 ok,
// 1 ParseError, 2 UnsupportedFormat, 3 IndexOutOfRange, 4 other (message in
// refp_last_error); the matrix is kept for refp_mm_arrays.
thread_local sparseoracle::CooMatrix g_mm;

int refp_read_mm(const char* path, int64_t* nrows, int64_t* ncols, int64_t* nnz, int32_t* kind) {
    *kind = 0;
    try {
        g_mm = sparseoracle::read_matrix_market(path);
        *nrows = g_mm.nrows;
        *ncols = g_mm.ncols;
        *nnz = g_mm.nnz();
        return 0;
    } catch (const sparseoracle::ParseError& e) {
        *kind = 1;
        g_err = e.what();
    } catch (const sparseoracle::UnsupportedFormat& e) {
        *kind = 2;
        g_err = e.what();
    } catch (const sparseoracle::IndexOutOfRange& e) {
        *kind = 3;
        g_err = e.what();
    } catch (const std::exception& e) {
        *kind = 4;
        g_err = e.what();
    }
    return 1;
}

void refp_mm_arrays(int64_t* row, int64_t* col, double* val) {
    for (size_t k = 0; k < g_mm.values.size(); ++k) {
        row[k] = g_mm.row_idx[k];
        col[k] = g_mm.col_idx[k];
        val[k] = g_mm.values[k];
    }
}

// write_matrix_market of a canonical COO given as arrays
int refp_write_mm(const char* path, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* row,
                  const int64_t* col, const double* val) {
    return guard([&] {
        sparseoracle::CooMatrix m;
        m.nrows = nrows;
        m.ncols = ncols;
        m.row_idx.assign(row, row + nnz);
        m.col_idx.assign(col, col + nnz);
        m.values.assign(val, val + nnz);
        sparseoracle::write_matrix_market(m, path);
    });
}

}  // extern "C"
