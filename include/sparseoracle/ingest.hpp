#pragma once
// Matrix Market I/O of the reference API (proj/include/sparseoracle/
// ingest.hpp:14-29), over the B200 C-ABI: the file is parsed by all host
// threads (so_read_matrix_market) and canonicalized on the device.  Same
// accepted subset, error types and messages as the reference.
//
// Only the Matrix Market part of the reference header is provided: corpus
// manifests, HTTP fetching and the profiling/training CSV helpers belong to
// the reference's offline pipeline, which stays out of this hot path
// (DESIGN.md §8); code that needs them keeps linking the reference for them.

#include <filesystem>

#include "sparseoracle/formats.hpp"

namespace sparseoracle {

// Accepted subset: matrix coordinate {real, integer, pattern} with symmetry
// {general, symmetric}. Everything else raises UnsupportedFormat.
struct MatrixMarketHeader {
    enum class Field { real, integer, pattern };
    enum class Symmetry { general, symmetric };
    Field field = Field::real;
    Symmetry symmetry = Symmetry::general;
};

// 1-based indices become 0-based, symmetric off-diagonals are mirrored,
// pattern entries get value 1.0, and the result is canonicalized.
CooMatrix read_matrix_market(const std::filesystem::path& path);

// Header line '%%MatrixMarket matrix coordinate real general', 1-based
// indices, shortest round-trip decimals.
void write_matrix_market(const CooMatrix& m, const std::filesystem::path& path);

}  // namespace sparseoracle
