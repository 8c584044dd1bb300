// spmv / spmv_parallel / time_spmv over the B200 C-ABI (reference:
// proj/src/spmv.cpp:203-246).  The dimension and argument checks keep the
// reference's order and messages; the arithmetic runs in the sm_100a kernels.
#include <string>

#include "sparseoracle/device.hpp"
#include "sparseoracle/spmv.hpp"

namespace sparseoracle {

DenseVector spmv(const DynamicMatrix& m, const DenseVector& x) {
    if (static_cast<index_t>(x.size()) != m.ncols())  // spmv.cpp:12-19
        throw DimensionMismatch("spmv: vector length " + std::to_string(x.size()) + " does not match ncols " +
                                std::to_string(m.ncols()));
    // y is sized (value-initialised: a single-threaded zero fill) by the
    // library's callback on this thread while host threads stage x and the
    // device multiplies (so_spmv_new); never throws across the C-ABI
    DenseVector y;
    auto make = [](void* ctx, int64_t n) noexcept -> double* {
        try {
            auto* v = static_cast<DenseVector*>(ctx);
            v->resize(static_cast<std::size_t>(n));
            return v->data();
        } catch (...) {
            return nullptr;
        }
    };
    detail::check(so_spmv_new(m.device().get(), x.data(), static_cast<int64_t>(x.size()), make, &y));
    return y;
}

DenseVector spmv_parallel(const DynamicMatrix& m, const DenseVector& x, int nthreads) {
    if (static_cast<index_t>(x.size()) != m.ncols())
        throw DimensionMismatch("spmv: vector length " + std::to_string(x.size()) + " does not match ncols " +
                                std::to_string(m.ncols()));
    if (nthreads < 1) throw InvalidInput("spmv_parallel: nthreads must be >= 1");  // spmv.cpp:213-215
    return spmv(m, x);
}

TimingSample time_spmv(const DynamicMatrix& m, const DenseVector& x, index_t repetitions, int /*nthreads*/) {
    if (repetitions < 1) throw InvalidInput("time_spmv: repetitions must be >= 1");  // spmv.cpp:223-225
    if (static_cast<index_t>(x.size()) != m.ncols())
        throw DimensionMismatch("spmv: vector length " + std::to_string(x.size()) + " does not match ncols " +
                                std::to_string(m.ncols()));
    TimingSample s;
    s.format = m.format();
    s.repetitions = repetitions;
    s.per_rep_seconds.resize(static_cast<std::size_t>(repetitions));
    detail::check(so_time_spmv(m.device().get(), x.data(), static_cast<int64_t>(x.size()), repetitions,
                               s.per_rep_seconds.data(), &s.total_seconds));
    // the reference accumulates total in rep order (spmv.cpp:241-243)
    double total = 0.0;
    for (double t : s.per_rep_seconds) total += t;
    s.total_seconds = total;
    return s;
}

}  // namespace sparseoracle
