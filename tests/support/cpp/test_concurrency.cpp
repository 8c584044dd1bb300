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
#include "sparseoracle/tuners.hpp"
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

// A stump forest on nnz (test_tuners.cpp:142-153 shape) plus a depth-3 tree,
// built in code so the test needs no model file.
static ForestModel small_forest() {
    ForestModel f;
    f.kind = ModelKind::forest;
    DecisionTreeModel stump;
    stump.nodes.resize(3);
    stump.nodes[0].feature_index = 2;
    stump.nodes[0].threshold = 150.0;
    stump.nodes[0].left = 1;
    stump.nodes[0].right = 2;
    stump.nodes[1].predicted_class = 1;
    stump.nodes[2].predicted_class = 0;
    f.trees.push_back(stump);
    f.trees.push_back(stump);
    DecisionTreeModel t;
    t.nodes.resize(5);
    t.nodes[0].feature_index = 5;  // max_nnz_per_row
    t.nodes[0].threshold = 4.0;
    t.nodes[0].left = 1;
    t.nodes[0].right = 2;
    t.nodes[1].predicted_class = 3;
    t.nodes[2].feature_index = 8;  // ndiags
    t.nodes[2].threshold = 40.0;
    t.nodes[2].left = 3;
    t.nodes[2].right = 4;
    t.nodes[3].predicted_class = 2;
    t.nodes[4].predicted_class = 4;
    f.trees.push_back(t);
    return f;
}

// ADVICE (r1, high): tune_ml captures a CUDA graph on first use; that capture
// must not swallow other threads' work on the same device.  Threads multiply
// (host and device paths) while others tune fresh matrices (every tune_ml
// call captures a new graph) -- every product and every outcome must equal
// the single-threaded one.
TEST_CASE("tune_ml captures while other threads multiply") {
    Rng rng(4242);
    const ForestModel forest = small_forest();
    TunerConfig cfg;
    std::vector<CooMatrix> coos;
    std::vector<DenseVector> xs;
    for (int k = 0; k < 24; ++k) {
        coos.push_back(random_coo(rng, 200 + 40 * k));
        xs.push_back(random_vector(rng, coos.back().ncols));
    }
    auto spmv_fmt = [](size_t k) { return k % 3 == 0 ? FormatId::coo : FormatId::csr; };
    std::vector<DenseVector> want_y;
    std::vector<FormatId> want_fmt;
    for (size_t k = 0; k < coos.size(); ++k) {
        want_y.push_back(spmv(DynamicMatrix(from_coo(coos[k], spmv_fmt(k))), xs[k]));
        want_fmt.push_back(tune_ml(DynamicMatrix(from_coo(coos[k], FormatId::csr)), cfg, forest).chosen);
    }
    for (int round = 0; round < 3; ++round) {
        std::vector<std::thread> pool;
        std::vector<int> bad(8, 0);
        for (int t = 0; t < 8; ++t)
            pool.emplace_back([&, t] {
                for (size_t k = size_t(t); k < coos.size(); k += 8) {
                    if (t % 2 == 0) {
                        // fresh matrix: first tune_ml on it captures its graph
                        const DynamicMatrix m = from_coo(coos[k], FormatId::csr);
                        for (int r = 0; r < 3; ++r)
                            if (tune_ml(m, cfg, forest).chosen != want_fmt[k]) bad[size_t(t)]++;
                    } else {
                        const DynamicMatrix m = from_coo(coos[k], spmv_fmt(k));
                        for (int r = 0; r < 5; ++r)
                            if (!(spmv(m, xs[k]) == want_y[k])) bad[size_t(t)]++;
                    }
                }
            });
        for (auto& th : pool) th.join();
        for (int t = 0; t < 8; t += 2) CHECK(bad[size_t(t)] == 0);  // tune_ml threads
        for (int t = 1; t < 8; t += 2) CHECK(bad[size_t(t)] == 0);  // spmv threads
    }
}

TEST_CASE("tune_ml on distinct matrices runs concurrently and on one matrix takes turns") {
    Rng rng(99);
    const ForestModel forest = small_forest();
    TunerConfig cfg;
    const CooMatrix coo = random_coo(rng, 500);
    const DynamicMatrix shared = from_coo(coo, FormatId::csr);
    const FormatId want = tune_ml(DynamicMatrix(from_coo(coo, FormatId::csr)), cfg, forest).chosen;
    std::vector<std::thread> pool;
    std::vector<int> bad(6, 0);
    for (int t = 0; t < 6; ++t)
        pool.emplace_back([&, t] {
            for (int r = 0; r < 20; ++r)
                if (tune_ml(shared, cfg, forest).chosen != want) bad[size_t(t)]++;
        });
    for (auto& th : pool) th.join();
    for (int t = 0; t < 6; ++t) CHECK(bad[size_t(t)] == 0);
}

// ADVICE (r1, low): a random forest without trees votes nothing and the
// reference's predict_forest returns COO (model.cpp:215-228), which is always
// feasible -- tune_ml must return COO, not fail the upload.
TEST_CASE("empty forest tunes to COO") {
    Rng rng(5);
    const CooMatrix coo = random_coo(rng, 64);
    ForestModel empty;
    empty.kind = ModelKind::forest;
    TunerConfig cfg;
    const DynamicMatrix m = from_coo(coo, FormatId::csr);
    const TuneOutcome o = tune_ml(m, cfg, empty);
    CHECK(o.chosen == FormatId::coo);
    CHECK(!o.fallback_csr);
    CHECK(o.switched);
    CHECK(o.source == TunerKind::random_forest);
    CHECK(predict_forest(empty, extract_features(m)) == FormatId::coo);
}
