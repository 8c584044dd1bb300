// The Matrix Market cases of the reference suite (proj/tests/test_ingest.cpp:
// 62-156), restated against this repo's drop-in C++ API (the rest of
// test_ingest.cpp covers the reference's offline corpus/CSV pipeline, out of
// scope, so the file cannot compile unmodified here).  Built by
// `make reftests` with the reference's own test support (oracles.hpp).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <filesystem>
#include <fstream>

#include "sparseoracle/ingest.hpp"
#include "support/oracles.hpp"

using namespace sparseoracle;
using namespace sparseoracle::testing;

namespace {
std::filesystem::path temp_dir(const std::string& name) {
    std::filesystem::path dir = std::filesystem::temp_directory_path() / name;
    std::filesystem::remove_all(dir);
    std::filesystem::create_directories(dir);
    return dir;
}
std::filesystem::path write_text(const std::filesystem::path& path, const std::string& text) {
    std::ofstream out(path, std::ios::binary);
    out << text;
    return path;
}
const char* kExampleMtx =
    "%%MatrixMarket matrix coordinate real general\n"
    "% the worked example\n"
    "3 3 5\n"
    "1 1 1\n"
    "1 3 2\n"
    "2 2 3\n"
    "3 1 4\n"
    "3 3 5\n";
}  // namespace

TEST_CASE("coordinate real general file round-trips the worked example") {
    std::filesystem::path dir = temp_dir("so_b200_ingest_basic");
    CooMatrix m = read_matrix_market(write_text(dir / "a.mtx", kExampleMtx));
    CHECK(m == worked_example_matrix());
}

TEST_CASE("symmetric files mirror off-diagonal entries only") {
    std::filesystem::path dir = temp_dir("so_b200_ingest_sym");
    CooMatrix m = read_matrix_market(write_text(dir / "s.mtx",
                                                "%%MatrixMarket matrix coordinate real symmetric\n"
                                                "2 2 2\n"
                                                "1 1 5\n"
                                                "2 1 7\n"));
    CHECK(m.nnz() == 3);
    DenseMatrix d = dense_from_coo(m);
    CHECK(d.at(0, 0) == 5.0);
    CHECK(d.at(1, 0) == 7.0);
    CHECK(d.at(0, 1) == 7.0);
    CHECK(d.at(1, 1) == 0.0);
}

TEST_CASE("pattern and integer fields") {
    std::filesystem::path dir = temp_dir("so_b200_ingest_fields");
    CooMatrix pattern = read_matrix_market(write_text(dir / "p.mtx",
                                                      "%%MatrixMarket matrix coordinate pattern general\n"
                                                      "2 2 2\n"
                                                      "1 2\n"
                                                      "2 1\n"));
    CHECK(pattern.values == std::vector<double>{1.0, 1.0});
    CooMatrix integer = read_matrix_market(write_text(dir / "i.mtx",
                                                      "%%MatrixMarket matrix coordinate integer general\n"
                                                      "1 2 1\n"
                                                      "1 2 -3\n"));
    CHECK(integer.values == std::vector<double>{-3.0});
}

TEST_CASE("unsupported headers are rejected") {
    std::filesystem::path dir = temp_dir("so_b200_ingest_unsupported");
    CHECK_THROWS_AS(read_matrix_market(write_text(dir / "c.mtx",
                                                  "%%MatrixMarket matrix coordinate complex general\n"
                                                  "1 1 1\n1 1 1 0\n")),
                    UnsupportedFormat);
    CHECK_THROWS_AS(
        read_matrix_market(write_text(dir / "a.mtx", "%%MatrixMarket matrix array real general\n1 1\n1\n")),
        UnsupportedFormat);
    CHECK_THROWS_AS(read_matrix_market(write_text(dir / "k.mtx",
                                                  "%%MatrixMarket matrix coordinate real skew-symmetric\n"
                                                  "2 2 1\n2 1 1\n")),
                    UnsupportedFormat);
}

TEST_CASE("parse errors carry line information") {
    std::filesystem::path dir = temp_dir("so_b200_ingest_parse");
    CHECK_THROWS_AS(read_matrix_market(write_text(dir / "short.mtx",
                                                  "%%MatrixMarket matrix coordinate real general\n"
                                                  "3 3 5\n1 1 1\n1 3 2\n2 2 3\n3 1 4\n")),
                    ParseError);
    CHECK_THROWS_AS(read_matrix_market(write_text(dir / "long.mtx",
                                                  "%%MatrixMarket matrix coordinate real general\n"
                                                  "2 2 1\n1 1 1\n2 2 2\n")),
                    ParseError);
    CHECK_THROWS_WITH_AS(read_matrix_market(write_text(dir / "bad.mtx",
                                                       "%%MatrixMarket matrix coordinate real general\n"
                                                       "2 2 1\n1 x 1\n")),
                         doctest::Contains(":3"), ParseError);
    CHECK_THROWS_AS(read_matrix_market(write_text(dir / "oob.mtx",
                                                  "%%MatrixMarket matrix coordinate real general\n"
                                                  "2 2 1\n3 1 1\n")),
                    IndexOutOfRange);
}

TEST_CASE("write then read is the identity on canonical matrices") {
    std::filesystem::path dir = temp_dir("so_b200_ingest_roundtrip");
    Rng rng(61);
    for (int trial = 0; trial < 20; ++trial) {
        CooMatrix m = random_coo(rng, 40);
        std::filesystem::path path = dir / ("m" + std::to_string(trial) + ".mtx");
        write_matrix_market(m, path);
        CHECK(read_matrix_market(path) == m);
    }
}
