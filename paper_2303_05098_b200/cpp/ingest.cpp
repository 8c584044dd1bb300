// sparseoracle:: Matrix Market I/O over the B200 C-ABI (reference:
// proj/src/ingest.cpp:135-224).  Parsing runs on all host threads inside the
// library (so_read_matrix_market, csrc/ingest.cu); the canonical COO comes
// back from the device.
#include "sparseoracle/ingest.hpp"

#include <string>

#include "sparseoracle/device.hpp"

namespace sparseoracle {

CooMatrix read_matrix_market(const std::filesystem::path& path) {
    so_matrix* out = nullptr;
    detail::check(so_read_matrix_market(path.string().c_str(), &out));
    detail::DeviceMirror coo(out);
    return std::get<CooMatrix>(coo.download());
}

void write_matrix_market(const CooMatrix& m, const std::filesystem::path& path) {
    if (!m.is_canonical()) throw InvalidInput("write_matrix_market: matrix is not canonical");
    auto dev = detail::DeviceMirror::upload(DynamicMatrix::Payload(m));
    detail::check(so_write_matrix_market(dev->get(), path.string().c_str()));
}

}  // namespace sparseoracle
