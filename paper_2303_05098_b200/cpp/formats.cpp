// sparseoracle:: containers and conversions over the B200 C-ABI
// (reference: proj/src/formats.cpp).
#include <algorithm>
#include <cctype>
#include <cmath>
#include <limits>
#include <mutex>
#include <string>

#include "sparseoracle/device.hpp"
#include "sparseoracle/formats.hpp"

namespace sparseoracle {

namespace detail {

void check(so_status st) {
    if (st == SO_OK) return;
    const std::string msg = so_last_error();
    switch (st) {
        case SO_INVALID_INPUT: throw InvalidInput(msg);
        case SO_PADDING_OVERFLOW: throw PaddingOverflow(msg);
        case SO_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        case SO_EMPTY_MATRIX: throw EmptyMatrix(msg);
        case SO_MALFORMED_MODEL: throw MalformedModel(msg);
        case SO_INDEX_OUT_OF_RANGE: throw IndexOutOfRange(msg);
        case SO_ALL_FORMATS_INFEASIBLE: throw AllFormatsInfeasible(msg);
        case SO_OUT_OF_MEMORY: throw DeviceOutOfMemory(msg);
        case SO_CUDA_ERROR: throw DeviceError(msg);
        case SO_PARSE_ERROR: throw ParseError(msg);
        case SO_UNSUPPORTED_FORMAT: throw UnsupportedFormat(msg);
        default: throw Error(msg);
    }
}

DeviceMirror::DeviceMirror(so_matrix* m) : m_(m) { check(so_matrix_info_get(m_, &info_)); }

DeviceMirror::~DeviceMirror() { so_matrix_free(m_); }

std::shared_ptr<DeviceMirror> DeviceMirror::upload(const DynamicMatrix::Payload& p) {
    so_matrix* out = nullptr;
    std::visit(
        [&](const auto& h) {
            using T = std::decay_t<decltype(h)>;
            if constexpr (std::is_same_v<T, CooMatrix>) {
                check(so_matrix_upload_coo(h.nrows, h.ncols, h.nnz(), h.row_idx.data(), h.col_idx.data(),
                                           h.values.data(), &out));
            } else if constexpr (std::is_same_v<T, CsrMatrix>) {
                check(so_matrix_upload_csr(h.nrows, h.ncols, h.nnz(), h.row_ptr.data(), h.col_idx.data(),
                                           h.values.data(), &out));
            } else if constexpr (std::is_same_v<T, DiaMatrix>) {
                check(so_matrix_upload_dia(h.nrows, h.ncols, h.ndiags(), h.offsets.data(), h.values.data(),
                                           h.stored_nnz, &out));
            } else if constexpr (std::is_same_v<T, EllMatrix>) {
                check(so_matrix_upload_ell(h.nrows, h.ncols, h.entries_per_row, h.col_idx.data(), h.values.data(),
                                           h.stored_nnz, &out));
            } else if constexpr (std::is_same_v<T, HybMatrix>) {
                const EllMatrix& e = h.ell_part;
                const CooMatrix& c = h.coo_part;
                check(so_matrix_upload_hyb(e.nrows, e.ncols, e.entries_per_row, e.col_idx.data(), e.values.data(),
                                           e.stored_nnz, c.nnz(), c.row_idx.data(), c.col_idx.data(),
                                           c.values.data(), h.kh, &out));
            } else {
                const DiaMatrix& d = h.dia_part;
                const CsrMatrix& c = h.csr_part;
                check(so_matrix_upload_hdc(c.nrows, c.ncols, d.ndiags(), d.offsets.data(), d.values.data(),
                                           d.stored_nnz, c.nnz(), c.row_ptr.data(), c.col_idx.data(),
                                           c.values.data(), h.true_diag_threshold, &out));
            }
        },
        p);
    return make_mirror(out);
}

DynamicMatrix::Payload DeviceMirror::download() const {
    const so_matrix_info& i = info_;
    const auto n = static_cast<std::size_t>(i.nrows);
    so_host_arrays a{};
    auto coo = [&](CooMatrix& c) {
        c.nrows = i.nrows;
        c.ncols = i.ncols;
        c.row_idx.resize(static_cast<std::size_t>(i.coo_nnz));
        c.col_idx.resize(static_cast<std::size_t>(i.coo_nnz));
        c.values.resize(static_cast<std::size_t>(i.coo_nnz));
        a.coo_row = c.row_idx.data();
        a.coo_col = c.col_idx.data();
        a.coo_val = c.values.data();
    };
    auto csr = [&](CsrMatrix& c) {
        c.nrows = i.nrows;
        c.ncols = i.ncols;
        c.row_ptr.resize(n + 1);
        c.col_idx.resize(static_cast<std::size_t>(i.csr_nnz));
        c.values.resize(static_cast<std::size_t>(i.csr_nnz));
        a.csr_row_ptr = c.row_ptr.data();
        a.csr_col = c.col_idx.data();
        a.csr_val = c.values.data();
    };
    auto dia = [&](DiaMatrix& d) {
        d.nrows = i.nrows;
        d.ncols = i.ncols;
        d.offsets.resize(static_cast<std::size_t>(i.ndiags));
        d.values.resize(static_cast<std::size_t>(i.ndiags) * n);
        d.stored_nnz = i.dia_stored_nnz;
        a.dia_offsets = d.offsets.data();
        a.dia_values = d.values.data();
    };
    auto ell = [&](EllMatrix& e) {
        e.nrows = i.nrows;
        e.ncols = i.ncols;
        e.entries_per_row = i.ell_width;
        e.col_idx.resize(static_cast<std::size_t>(i.ell_width) * n);
        e.values.resize(static_cast<std::size_t>(i.ell_width) * n);
        e.stored_nnz = i.ell_stored_nnz;
        a.ell_col = e.col_idx.data();
        a.ell_val = e.values.data();
    };
    DynamicMatrix::Payload p;
    switch (static_cast<FormatId>(i.format)) {
        case FormatId::coo: {
            CooMatrix c;
            coo(c);
            check(so_matrix_download(m_, &a));
            p = std::move(c);
            break;
        }
        case FormatId::csr: {
            CsrMatrix c;
            csr(c);
            check(so_matrix_download(m_, &a));
            p = std::move(c);
            break;
        }
        case FormatId::dia: {
            DiaMatrix d;
            dia(d);
            check(so_matrix_download(m_, &a));
            p = std::move(d);
            break;
        }
        case FormatId::ell: {
            EllMatrix e;
            ell(e);
            check(so_matrix_download(m_, &a));
            p = std::move(e);
            break;
        }
        case FormatId::hyb: {
            HybMatrix h;
            ell(h.ell_part);
            coo(h.coo_part);
            h.kh = i.kh;
            check(so_matrix_download(m_, &a));
            p = std::move(h);
            break;
        }
        case FormatId::hdc: {
            HdcMatrix h;
            dia(h.dia_part);
            csr(h.csr_part);
            h.true_diag_threshold = i.true_diag_threshold;
            check(so_matrix_download(m_, &a));
            p = std::move(h);
            break;
        }
    }
    return p;
}

}  // namespace detail

// ---------------------------------------------------------------- names

namespace {
constexpr std::array<std::string_view, kNumFormats> kNames = {"COO", "CSR", "DIA", "ELL", "HYB", "HDC"};
}

std::string_view format_name(FormatId id) { return kNames[static_cast<std::size_t>(id)]; }

std::optional<FormatId> format_from_name(std::string_view name) {  // case-insensitive (formats.cpp:273-283)
    std::string up;
    up.reserve(name.size());
    for (char c : name) up.push_back(static_cast<char>(std::toupper(static_cast<unsigned char>(c))));
    for (int k = 0; k < kNumFormats; ++k)
        if (kNames[static_cast<std::size_t>(k)] == up) return static_cast<FormatId>(k);
    return std::nullopt;
}

FormatId format_from_id(int id) {
    if (id < 0 || id >= kNumFormats)
        throw InvalidInput("format id " + std::to_string(id) + " outside 0.." + std::to_string(kNumFormats - 1));
    return static_cast<FormatId>(id);
}

// ---------------------------------------------------------------- COO

// formats.cpp:293-322 on the device (so_coo_from_triplets): range check,
// stable radix sort by (row, col), duplicates summed in input order; the
// canonical result is downloaded into the host container.
CooMatrix CooMatrix::from_triplets(index_t nrows, index_t ncols, std::vector<Triplet> triplets) {
    const std::size_t n = triplets.size();
    std::vector<index_t> r(n), c(n);
    std::vector<double> v(n);
    for (std::size_t k = 0; k < n; ++k) {
        r[k] = triplets[k].row;
        c[k] = triplets[k].col;
        v[k] = triplets[k].value;
    }
    for (std::size_t k = 0; k < n; ++k)  // message of formats.cpp:296-300
        if (r[k] < 0 || r[k] >= nrows || c[k] < 0 || c[k] >= ncols)
            throw IndexOutOfRange("triplet (" + std::to_string(r[k]) + ", " + std::to_string(c[k]) + ") outside " +
                                  std::to_string(nrows) + "x" + std::to_string(ncols));
    so_matrix* out = nullptr;
    detail::check(so_coo_from_triplets(nrows, ncols, static_cast<int64_t>(n), r.data(), c.data(), v.data(), &out));
    detail::DeviceMirror coo(out);
    return std::get<CooMatrix>(coo.download());
}

bool CooMatrix::is_canonical() const {  // formats.cpp:324-340
    if (nrows < 0 || ncols < 0) return false;
    const std::size_t z = values.size();
    if (row_idx.size() != z || col_idx.size() != z) return false;
    for (std::size_t k = 0; k < z; ++k) {
        if (row_idx[k] < 0 || row_idx[k] >= nrows || col_idx[k] < 0 || col_idx[k] >= ncols) return false;
        if (k > 0 && !(row_idx[k - 1] < row_idx[k] || (row_idx[k - 1] == row_idx[k] && col_idx[k - 1] < col_idx[k])))
            return false;
    }
    return true;
}

bool operator==(const CooMatrix& a, const CooMatrix& b) {
    return a.nrows == b.nrows && a.ncols == b.ncols && a.row_idx == b.row_idx && a.col_idx == b.col_idx &&
           a.values == b.values;
}

// ---------------------------------------------------------------- config

index_t ConversionConfig::padded_entry_cap(index_t nnz) const {  // formats.cpp:348-355
    if (max_padded_entries > 0) return max_padded_entries;
    const double cap = max_padding_factor * static_cast<double>(nnz);
    if (cap >= static_cast<double>(std::numeric_limits<index_t>::max())) return std::numeric_limits<index_t>::max();
    return static_cast<index_t>(cap);
}

index_t ConversionConfig::effective_kh(index_t nnz, index_t nrows) const {  // :357-361
    if (kh_override > 0) return kh_override;
    if (nrows <= 0 || nnz <= 0) return 0;
    return (nnz + nrows - 1) / nrows;
}

index_t ConversionConfig::true_diag_threshold(index_t nrows, index_t ncols) const {  // :363-367
    return static_cast<index_t>(std::ceil(true_diag_ratio * static_cast<double>(std::min(nrows, ncols))));
}

// ---------------------------------------------------------------- DynamicMatrix

namespace {
std::mutex& lazy_mu() {  // serialises lazy host downloads / device uploads
    static std::mutex mu;
    return mu;
}
}  // namespace

DynamicMatrix::DynamicMatrix(const DynamicMatrix& o) : fmt_(o.fmt_) {
    std::lock_guard<std::mutex> lk(lazy_mu());
    const bool hv = o.host_valid_.load(std::memory_order_acquire);
    payload_ = hv ? o.payload_ : Payload(CooMatrix{});
    host_valid_.store(hv, std::memory_order_release);
    dev_ = o.dev_;
}

DynamicMatrix::DynamicMatrix(DynamicMatrix&& o) noexcept
    : payload_(std::move(o.payload_)),
      fmt_(o.fmt_),
      host_valid_(o.host_valid_.load(std::memory_order_acquire)),
      dev_(std::move(o.dev_)) {}

DynamicMatrix& DynamicMatrix::operator=(const DynamicMatrix& o) {
    if (this != &o) {
        std::lock_guard<std::mutex> lk(lazy_mu());
        const bool hv = o.host_valid_.load(std::memory_order_acquire);
        payload_ = hv ? o.payload_ : Payload(CooMatrix{});
        fmt_ = o.fmt_;
        host_valid_.store(hv, std::memory_order_release);
        dev_ = o.dev_;  // device copies are immutable once built: share
    }
    return *this;
}

DynamicMatrix& DynamicMatrix::operator=(DynamicMatrix&& o) noexcept {
    payload_ = std::move(o.payload_);
    fmt_ = o.fmt_;
    host_valid_.store(o.host_valid_.load(std::memory_order_acquire), std::memory_order_release);
    dev_ = std::move(o.dev_);
    return *this;
}

DynamicMatrix::~DynamicMatrix() = default;

DynamicMatrix DynamicMatrix::adopt(std::shared_ptr<detail::DeviceMirror> device) {
    DynamicMatrix m;
    m.fmt_ = static_cast<FormatId>(device->info().format);
    m.host_valid_ = false;
    m.dev_ = std::move(device);
    return m;
}

void DynamicMatrix::materialize() const {
    if (host_valid_.load(std::memory_order_acquire)) return;
    std::lock_guard<std::mutex> lk(lazy_mu());
    if (host_valid_.load(std::memory_order_relaxed)) return;
    payload_ = dev_->download();
    host_valid_.store(true, std::memory_order_release);
}

void DynamicMatrix::detach_device() { dev_.reset(); }

const detail::DeviceMirror& DynamicMatrix::device() const {
    std::lock_guard<std::mutex> lk(lazy_mu());
    if (!dev_) dev_ = detail::DeviceMirror::upload(payload_);
    return *dev_;
}

index_t DynamicMatrix::nrows() const {
    if (!host_valid_) return dev_->info().nrows;
    return std::visit(
        [](const auto& m) -> index_t {
            using T = std::decay_t<decltype(m)>;
            if constexpr (std::is_same_v<T, HybMatrix> || std::is_same_v<T, HdcMatrix>)
                return m.nrows();
            else
                return m.nrows;
        },
        payload_);
}

index_t DynamicMatrix::ncols() const {
    if (!host_valid_) return dev_->info().ncols;
    return std::visit(
        [](const auto& m) -> index_t {
            using T = std::decay_t<decltype(m)>;
            if constexpr (std::is_same_v<T, HybMatrix> || std::is_same_v<T, HdcMatrix>)
                return m.ncols();
            else
                return m.ncols;
        },
        payload_);
}

index_t DynamicMatrix::nnz() const {  // formats.cpp:397-409
    if (!host_valid_) return dev_->info().nnz;
    return std::visit(
        [](const auto& m) -> index_t {
            using T = std::decay_t<decltype(m)>;
            if constexpr (std::is_same_v<T, DiaMatrix> || std::is_same_v<T, EllMatrix>)
                return m.stored_nnz;
            else
                return m.nnz();
        },
        payload_);
}

// ---------------------------------------------------------------- conversions

namespace {
so_conversion_config to_c(const ConversionConfig& c) {
    return so_conversion_config{c.kh_override, c.true_diag_ratio, c.max_padding_factor, c.max_padded_entries};
}
}  // namespace

DynamicMatrix from_coo(const CooMatrix& src, FormatId target, const ConversionConfig& config) {
    so_matrix* coo = nullptr;
    detail::check(so_matrix_upload_coo(src.nrows, src.ncols, src.nnz(), src.row_idx.data(), src.col_idx.data(),
                                       src.values.data(), &coo));
    auto coo_mirror = detail::make_mirror(coo);
    if (target == FormatId::coo) {
        // formats.cpp:413-417: canonical check, then the payload itself
        so_matrix* copy = nullptr;
        const so_conversion_config c = to_c(config);
        detail::check(so_from_coo(coo, SO_COO, &c, &copy));
        DynamicMatrix m(src);
        m.dev_ = detail::make_mirror(copy);
        return m;
    }
    const so_conversion_config c = to_c(config);
    so_matrix* out = nullptr;
    detail::check(so_from_coo(coo, static_cast<int32_t>(target), &c, &out));
    return DynamicMatrix::adopt(detail::make_mirror(out));
}

CooMatrix to_coo(const DynamicMatrix& m) {
    if (m.format() == FormatId::coo) return m.as<CooMatrix>();  // formats.cpp:436-437
    so_matrix* out = nullptr;
    detail::check(so_to_coo(m.device().get(), &out));
    detail::DeviceMirror coo(out);
    return std::get<CooMatrix>(coo.download());
}

void switch_format(DynamicMatrix& m, FormatId target, const ConversionConfig& config) {
    if (m.format() == target) return;
    const so_conversion_config c = to_c(config);
    so_matrix* out = nullptr;
    detail::check(so_convert(m.device().get(), static_cast<int32_t>(target), &c, &out));
    m = DynamicMatrix::adopt(detail::make_mirror(out));
}

}  // namespace sparseoracle
