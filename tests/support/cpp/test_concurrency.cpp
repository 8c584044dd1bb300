// Concurrent readers of one immutable matrix (the reference's threading
// contract): eight threads multiply and read the host arrays of
// the same const DynamicMatrix whose device copy and host arrays are both
// materialised lazily -- every thread must see the same arrays and the same y.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <thread>
#include <vector>

#include "sparseoracle/formats.hpp"
#include "sparseoracle/spmv.hpp"
#include "support/oracles.hpp"

using namespace sparseoracle;
using namespace sparseoracle::testing;

TEST_CASE("concurrent readers of a lazily materialised matrix") {
    Rng rng(97);
    for (int trial = 0; trial < 6; ++trial) {
        CooMatrix coo = random_coo(rng, 300);
        DenseVector x = random_vector(rng, coo.ncols);
        for (FormatId f : {FormatId::csr, FormatId::coo, FormatId::hdc}) {
            const DynamicMatrix m = from_coo(coo, f);  // device-produced: host arrays not downloaded yet
            const DenseVector want = spmv(DynamicMatrix(from_coo(coo, f)), x);
            std::vector<DenseVector> got(8);
            std::vector<index_t> nnz(8);
            std::vector<std::thread> pool;
            for (int t = 0; t < 8; ++t)
                pool.emplace_back([&, t] {
                    got[size_t(t)] = spmv(m, x);
                    nnz[size_t(t)] = m.nnz();
                    (void)m.payload();
                });
            for (auto& th : pool) th.join();
            for (int t = 0; t < 8; ++t) {
                CHECK(got[size_t(t)] == want);
                CHECK(nnz[size_t(t)] == m.nnz());
            }
        }
    }
}
