// Matrix Market I/O feeding the device canonicalization:
// read_matrix_market (ingest.cpp:135-208) and write_matrix_market
// (ingest.cpp:210-224) with the reference's accepted subset, error types,
// messages and line numbers, but parsed by all host cores: the body is cut
// into newline-aligned slices, every thread tokenizes and converts its slice
// with std::from_chars (the reference's own number parser), and the first
// error in FILE order wins, exactly as in the reference's sequential loop.
// The triplets (symmetric off-diagonals mirrored right after their entry, as
// the reference pushes them) go to the device radix-sort canonicalization
// (so_coo_from_triplets).  Host code only; no kernels here.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "matrix.cuh"

namespace sob {
namespace {

// ---------------------------------------------------------------- errors --
// ParseError carries "path:line: what" (ingest.cpp:22-25)
[[noreturn]] void parse_fail(const std::string& path, int64_t line, const std::string& what) {
    fail(SO_PARSE_ERROR, path + ":" + std::to_string(line) + ": " + what);
}

std::string lower(std::string s) {
    for (char& c : s) c = char(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// whitespace tokens of [b, e) (istringstream >> semantics), at most `cap`+1
int tokenize(const char* b, const char* e, const char** tok, size_t* len, int cap) {
    int n = 0;
    while (b < e) {
        while (b < e && is_space(*b)) ++b;
        if (b >= e) break;
        const char* s = b;
        while (b < e && !is_space(*b)) ++b;
        if (n < cap) {
            tok[n] = s;
            len[n] = size_t(b - s);
        }
        ++n;
        if (n > cap) break;
    }
    return n;
}

bool parse_i64(const char* s, size_t n, int64_t& v) {
    auto r = std::from_chars(s, s + n, v);
    return r.ec == std::errc() && r.ptr == s + n;
}
bool parse_f64(const char* s, size_t n, double& v) {
    auto r = std::from_chars(s, s + n, v);
    return r.ec == std::errc() && r.ptr == s + n;
}

struct Header {
    bool pattern = false, symmetric = false;
};

// ingest.cpp:63-101
Header parse_header(const std::string& line, const std::string& path) {
    const char* tok[6];
    size_t len[6];
    const int n = tokenize(line.data(), line.data() + line.size(), tok, len, 5);
    auto t = [&](int i) { return i < n && i < 5 ? std::string(tok[i], len[i]) : std::string(); };
    if (t(0) != "%%MatrixMarket") parse_fail(path, 1, "missing %%MatrixMarket banner");
    if (lower(t(1)) != "matrix") fail(SO_UNSUPPORTED_FORMAT, path + ": object '" + t(1) + "' not supported");
    if (lower(t(2)) != "coordinate")
        fail(SO_UNSUPPORTED_FORMAT, path + ": format '" + t(2) + "' not supported (coordinate only)");
    Header h;
    const std::string f = lower(t(3));
    if (f == "pattern")
        h.pattern = true;
    else if (f != "real" && f != "integer")
        fail(SO_UNSUPPORTED_FORMAT, path + ": field '" + t(3) + "' not supported");
    const std::string s = lower(t(4));
    if (s == "symmetric")
        h.symmetric = true;
    else if (s != "general")
        fail(SO_UNSUPPORTED_FORMAT, path + ": symmetry '" + t(4) + "' not supported");
    return h;
}

// One newline-aligned slice of the body.
struct Slice {
    const char* b;
    const char* e;
    int64_t first_line = 0;  // file line number of the slice's first line
    // results
    std::vector<int64_t> row, col;
    std::vector<double> val;
    int64_t entries = 0;       // data lines parsed before the first error (or all)
    int64_t err_line = -1;     // first error in the slice
    so_status err_status = SO_OK;
    std::string err_msg;
};

// Parse lines of [b, e) until the first error.  `stop_after`: stop (without
// error) once this many data lines were seen (used to locate the line of the
// (declared+1)-th entry).  Returns the line number where it stopped.
void parse_slice(Slice& sl, const std::string& path, const Header& h, int64_t nrows, int64_t ncols,
                 int64_t stop_after, int64_t* stop_line) {
    const char* p = sl.b;
    int64_t line = sl.first_line;
    const int want = h.pattern ? 2 : 3;
    while (p < sl.e) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', size_t(sl.e - p)));
        const char* le = nl ? nl : sl.e;
        const char* lend = le;
        if (lend > p && lend[-1] == '\r') --lend;  // ingest.cpp:155
        if (lend > p && p[0] != '%') {
            const char* tok[4];
            size_t len[4];
            const int n = tokenize(p, lend, tok, len, 3);
            auto err = [&](so_status st, const std::string& msg) {
                sl.err_line = line;
                sl.err_status = st;
                sl.err_msg = msg;
            };
            if (n != want) {  // ingest.cpp:176-181, checked before the entry count
                err(SO_PARSE_ERROR, path + ":" + std::to_string(line) + ": " +
                                        (h.pattern ? "expected 'row col'" : "expected 'row col value'"));
                return;
            }
            if (stop_after >= 0 && sl.entries == stop_after) {  // this line is entry stop_after+1
                *stop_line = line;
                return;
            }
            // counted before the numbers are parsed (ingest.cpp:182-186)
            ++sl.entries;
            int64_t r = 0, c = 0;
            double v = 1.0;
            if (!parse_i64(tok[0], len[0], r)) {
                err(SO_PARSE_ERROR, path + ":" + std::to_string(line) + ": expected integer, got '" +
                                        std::string(tok[0], len[0]) + "'");
                return;
            }
            if (!parse_i64(tok[1], len[1], c)) {
                err(SO_PARSE_ERROR, path + ":" + std::to_string(line) + ": expected integer, got '" +
                                        std::string(tok[1], len[1]) + "'");
                return;
            }
            if (r < 1 || r > nrows || c < 1 || c > ncols) {
                err(SO_INDEX_OUT_OF_RANGE, path + ":" + std::to_string(line) + ": entry (" +
                                               std::string(tok[0], len[0]) + ", " + std::string(tok[1], len[1]) +
                                               ") outside " + std::to_string(nrows) + "x" + std::to_string(ncols));
                return;
            }
            if (!h.pattern && !parse_f64(tok[2], len[2], v)) {
                err(SO_PARSE_ERROR, path + ":" + std::to_string(line) + ": expected number, got '" +
                                        std::string(tok[2], len[2]) + "'");
                return;
            }
            if (stop_after < 0) {
                sl.row.push_back(r - 1);
                sl.col.push_back(c - 1);
                sl.val.push_back(v);
                if (h.symmetric && r != c) {  // ingest.cpp:197-199
                    sl.row.push_back(c - 1);
                    sl.col.push_back(r - 1);
                    sl.val.push_back(v);
                }
            }
        }
        ++line;
        p = nl ? nl + 1 : sl.e;
    }
}

}  // namespace

// The whole file in one uninitialised buffer, read by all host threads with
// pread (a char-by-char stream copy ran at ~0.3 GB/s: most of the ingest).
std::unique_ptr<char[]> read_file(const std::string& path, size_t& size) {
    const int fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) fail(SO_PARSE_ERROR, "cannot open " + path);
    struct stat stt;
    if (::fstat(fd, &stt) != 0) {
        ::close(fd);
        fail(SO_PARSE_ERROR, "cannot open " + path);
    }
    size = size_t(stt.st_size);
    std::unique_ptr<char[]> buf(new char[size + 1]);
    const int nt = int(std::max<size_t>(1, std::min<size_t>(std::thread::hardware_concurrency(), size >> 22)));
    std::atomic<bool> bad{false};
    auto part = [&](int t) {
        size_t a = size * size_t(t) / size_t(nt);
        const size_t e = size * size_t(t + 1) / size_t(nt);
        while (a < e) {
            const ssize_t got = ::pread(fd, buf.get() + a, e - a, off_t(a));
            if (got <= 0) {
                bad = true;
                return;
            }
            a += size_t(got);
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(part, t);
    part(0);
    for (auto& th : pool) th.join();
    ::close(fd);
    if (bad) fail(SO_PARSE_ERROR, "cannot read " + path);
    return buf;
}

so_matrix* read_matrix_market(const std::string& path, cudaStream_t s) {
    size_t fsize = 0;
    const std::unique_ptr<char[]> buf = read_file(path, fsize);
    const char* p = buf.get();
    const char* end = p + fsize;
    if (fsize == 0) parse_fail(path, 1, "empty file");
    auto next_line = [&](const char* q) {
        const char* nl = static_cast<const char*>(std::memchr(q, '\n', size_t(end - q)));
        return nl ? nl : end;
    };
    // header (line 1); the reference reads it with getline (no '\r' strip)
    const char* le = next_line(p);
    const Header h = parse_header(std::string(p, le), path);
    int64_t line = 1;
    p = le < end ? le + 1 : end;
    // dimension line: first non-empty, non-comment line (ingest.cpp:153-174)
    int64_t nrows = 0, ncols = 0, declared = 0;
    bool have_dims = false;
    while (p < end) {
        le = next_line(p);
        ++line;
        const char* lend = le;
        if (lend > p && lend[-1] == '\r') --lend;
        const char* lp = p;
        p = le < end ? le + 1 : end;
        if (lend == lp || lp[0] == '%') continue;
        const char* tok[4];
        size_t len[4];
        if (tokenize(lp, lend, tok, len, 3) != 3) parse_fail(path, line, "expected 'rows cols nnz'");
        int64_t* dst[3] = {&nrows, &ncols, &declared};
        for (int k = 0; k < 3; ++k)
            if (!parse_i64(tok[k], len[k], *dst[k]))
                parse_fail(path, line, "expected integer, got '" + std::string(tok[k], len[k]) + "'");
        if (nrows < 0 || ncols < 0 || declared < 0) parse_fail(path, line, "negative dimension");
        if (h.symmetric && nrows != ncols) parse_fail(path, line, "symmetric matrix must be square");
        have_dims = true;
        break;
    }
    if (!have_dims) parse_fail(path, line, "missing dimension line");

    // newline-aligned slices, one per host thread
    const int64_t bytes = int64_t(end - p);
    int nt = int(std::max(1u, std::thread::hardware_concurrency()));
    nt = int(std::min<int64_t>(nt, std::max<int64_t>(1, bytes >> 20)));  // >= 1 MB per slice
    std::vector<Slice> sl(static_cast<size_t>(nt));
    const char* cur = p;
    for (int t = 0; t < nt; ++t) {
        sl[size_t(t)].b = cur;
        const char* cut = t + 1 == nt ? end : std::min(end, p + bytes * (t + 1) / nt);
        if (cut < end && cut > cur) {
            const char* nl = static_cast<const char*>(std::memchr(cut - 1, '\n', size_t(end - (cut - 1))));
            cut = nl ? nl + 1 : end;
        }
        if (cut < cur) cut = cur;
        sl[size_t(t)].e = cut;
        cur = cut;
    }
    // every slice's first line number (newline counts in parallel), then the
    // slices parsed in parallel, each into buffers sized from its bytes
    std::vector<int64_t> nls(sl.size(), 0);
    auto run_all = [&](const std::function<void(int)>& fn) {
        std::vector<std::thread> pool;
        for (int t = 1; t < nt; ++t) pool.emplace_back(fn, t);
        fn(0);
        for (auto& th : pool) th.join();
    };
    run_all([&](int t) { nls[size_t(t)] = int64_t(std::count(sl[size_t(t)].b, sl[size_t(t)].e, '\n')); });
    int64_t base = line + 1, body_nl = 0;
    for (size_t t = 0; t < sl.size(); ++t) {
        sl[t].first_line = base;
        base += nls[t];
        body_nl += nls[t];
    }
    // total line count as the reference's getline loop reports it
    const int64_t last_line = line + body_nl + ((end > p && end[-1] != '\n') ? 1 : 0);
    run_all([&](int t) {
        Slice& x = sl[size_t(t)];
        const size_t guess = size_t(nls[size_t(t)] + 1) * (h.symmetric ? 2 : 1);
        x.row.reserve(guess);
        x.col.reserve(guess);
        x.val.reserve(guess);
        parse_slice(x, path, h, nrows, ncols, -1, nullptr);
    });
    // first event in file order: an error line, or the (declared+1)-th entry
    int64_t seen = 0;
    for (auto& x : sl) {
        if (seen + x.entries > declared) {
            int64_t stop_line = 0;
            Slice probe{x.b, x.e, x.first_line};
            parse_slice(probe, path, h, nrows, ncols, declared - seen, &stop_line);
            parse_fail(path, stop_line, "more than the declared " + std::to_string(declared) + " entries");
        }
        if (x.err_line >= 0) fail(x.err_status, x.err_msg);
        seen += x.entries;
    }
    if (seen != declared)
        parse_fail(path, last_line, "declared " + std::to_string(declared) + " entries, found " + std::to_string(seen));
    // the slices in file order, uploaded where they lie, canonicalized on the device
    std::vector<TripletSegment> segs;
    for (auto& x : sl) segs.push_back(TripletSegment{x.row.data(), x.col.data(), x.val.data(), int64_t(x.row.size())});
    return coo_from_triplet_segments(nrows, ncols, segs.data(), int(segs.size()), s);
}

// ingest.cpp:210-224: banner, "rows cols nnz", 1-based entries with the
// shortest round-trip decimal (format_double = std::to_chars).  The entries
// are formatted by all host threads (contiguous ranges), then written at
// their byte offsets with pwrite: the same bytes as one sequential writer.
void write_matrix_market(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* row, const int64_t* col,
                         const double* val, const std::string& path) {
    std::string head = "%%MatrixMarket matrix coordinate real general\n";
    head += std::to_string(nrows) + " " + std::to_string(ncols) + " " + std::to_string(nnz) + "\n";
    const int nt = int(std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), nnz >> 16)));
    std::vector<std::string> part(static_cast<size_t>(nt));
    auto format = [&](int t) {
        const int64_t a = nnz * t / nt, e = nnz * (t + 1) / nt;
        std::string& out = part[size_t(t)];
        out.reserve(size_t(e - a) * 32);
        char num[64];
        for (int64_t k = a; k < e; ++k) {
            auto r1 = std::to_chars(num, num + sizeof(num), row[k] + 1);
            out.append(num, r1.ptr);
            out.push_back(' ');
            auto r2 = std::to_chars(num, num + sizeof(num), col[k] + 1);
            out.append(num, r2.ptr);
            out.push_back(' ');
            auto r3 = std::to_chars(num, num + sizeof(num), val[k]);
            out.append(num, r3.ptr);
            out.push_back('\n');
        }
    };
    {
        std::vector<std::thread> pool;
        for (int t = 1; t < nt; ++t) pool.emplace_back(format, t);
        format(0);
        for (auto& th : pool) th.join();
    }
    std::vector<off_t> at(static_cast<size_t>(nt) + 1);
    at[0] = off_t(head.size());
    for (int t = 0; t < nt; ++t) at[size_t(t) + 1] = at[size_t(t)] + off_t(part[size_t(t)].size());
    const int fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (fd < 0) fail(SO_ERROR, "cannot open " + path + " for writing");
    std::atomic<bool> bad{false};
    auto put = [&](const char* data, size_t n, off_t off) {
        while (n > 0) {
            const ssize_t w = ::pwrite(fd, data, n, off);
            if (w <= 0) {
                bad = true;
                return;
            }
            data += w;
            n -= size_t(w);
            off += off_t(w);
        }
    };
    put(head.data(), head.size(), 0);
    {
        std::vector<std::thread> pool;
        for (int t = 1; t < nt; ++t)
            pool.emplace_back([&, t] { put(part[size_t(t)].data(), part[size_t(t)].size(), at[size_t(t)]); });
        put(part[0].data(), part[0].size(), at[0]);
        for (auto& th : pool) th.join();
    }
    if (::close(fd) != 0) bad = true;
    if (bad) fail(SO_ERROR, "write failed for " + path);
}

}  // namespace sob
