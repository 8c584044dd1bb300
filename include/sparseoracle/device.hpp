#pragma once
// Device residency helpers of the B200 implementation (not part of the
// reference API): the RAII owner of an so_matrix and the status -> exception
// bridge every C++ entry point uses.

#include <memory>
#include <string>

#include "sparseoracle/formats.hpp"
#include "sparseoracle_b200.h"

namespace sparseoracle {
namespace detail {

// Throws the sparseoracle::Error subclass that matches an so_status.
void check(so_status st);

class DeviceMirror {
public:
    explicit DeviceMirror(so_matrix* m);
    ~DeviceMirror();
    DeviceMirror(const DeviceMirror&) = delete;
    DeviceMirror& operator=(const DeviceMirror&) = delete;

    so_matrix* get() const { return m_; }
    const so_matrix_info& info() const { return info_; }

    // host payload -> device
    static std::shared_ptr<DeviceMirror> upload(const DynamicMatrix::Payload& p);
    // device -> host payload (reference host layout)
    DynamicMatrix::Payload download() const;

private:
    so_matrix* m_;
    so_matrix_info info_{};
};

inline std::shared_ptr<DeviceMirror> make_mirror(so_matrix* m) { return std::make_shared<DeviceMirror>(m); }

}  // namespace detail
}  // namespace sparseoracle
