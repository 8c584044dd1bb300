// extract_features over the B200 C-ABI (reference: proj/src/features.cpp).
#include "sparseoracle/device.hpp"
#include "sparseoracle/features.hpp"

namespace sparseoracle {

FeatureVector extract_features(const DynamicMatrix& m, double true_diag_ratio, FeatureScanStats* stats) {
    if (m.nrows() < 1 || m.ncols() < 1)  // features.cpp:86-88, before any device work
        throw EmptyMatrix("extract_features: matrix has a zero dimension");
    if (!(true_diag_ratio > 0.0) || true_diag_ratio > 1.0)
        throw InvalidInput("extract_features: true_diag_ratio must be in (0, 1]");
    so_feature_vector f{};
    so_scan_stats st{};
    detail::check(so_extract_features(m.device().get(), true_diag_ratio, &f, &st));
    if (stats) {
        stats->entry_visits += st.entry_visits;
        stats->structure_reads += st.structure_reads;
    }
    FeatureVector out;
    out.nrows = f.nrows;
    out.ncols = f.ncols;
    out.nnz = f.nnz;
    out.avg_nnz_per_row = f.avg_nnz_per_row;
    out.density = f.density;
    out.max_nnz_per_row = f.max_nnz_per_row;
    out.min_nnz_per_row = f.min_nnz_per_row;
    out.nnz_row_spread = f.nnz_row_spread;
    out.ndiags = f.ndiags;
    out.ntrue_diags = f.ntrue_diags;
    return out;
}

std::array<double, kNumFeatures> features_to_row(const FeatureVector& f) {  // features.cpp:155-166
    return {static_cast<double>(f.nrows),           static_cast<double>(f.ncols),
            static_cast<double>(f.nnz),             f.avg_nnz_per_row,
            f.density,                              static_cast<double>(f.max_nnz_per_row),
            static_cast<double>(f.min_nnz_per_row), f.nnz_row_spread,
            static_cast<double>(f.ndiags),          static_cast<double>(f.ntrue_diags)};
}

FeatureVector row_to_features(const std::array<double, kNumFeatures>& r) {  // features.cpp:168-181
    FeatureVector f;
    f.nrows = static_cast<index_t>(r[0]);
    f.ncols = static_cast<index_t>(r[1]);
    f.nnz = static_cast<index_t>(r[2]);
    f.avg_nnz_per_row = r[3];
    f.density = r[4];
    f.max_nnz_per_row = static_cast<index_t>(r[5]);
    f.min_nnz_per_row = static_cast<index_t>(r[6]);
    f.nnz_row_spread = r[7];
    f.ndiags = static_cast<index_t>(r[8]);
    f.ntrue_diags = static_cast<index_t>(r[9]);
    return f;
}

}  // namespace sparseoracle
