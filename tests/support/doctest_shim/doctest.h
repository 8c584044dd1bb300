// Minimal doctest-compatible harness (test infrastructure).
//
// The reference's unit suites (proj/tests/test_*.cpp) are written against the
// vendored doctest, which is not mounted (proj/.gitignore:2).  This header
// implements exactly the subset those suites use -- TEST_CASE, CHECK,
// REQUIRE, CAPTURE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, FAIL,
// doctest::Approx(..).epsilon(..), doctest::Contains -- so the suites can be
// compiled unmodified against the B200 library's C++ API (Makefile target
// `reftests`) and run on the GPU (tests/test_gpu_reference_suites.py).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    bool matches(double lhs) const {
        return std::fabs(lhs - value_) < eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(value_)));
    }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
};
inline bool operator==(double lhs, const Approx& a) { return a.matches(lhs); }
inline bool operator==(const Approx& a, double rhs) { return a.matches(rhs); }
inline bool operator!=(double lhs, const Approx& a) { return !a.matches(lhs); }

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    std::string needle;
    bool check(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};

namespace detail {

struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) {
        registry().push_back({name, fn, file, line});
    }
};

struct RequireFailed {};

inline int& failures() {
    static int f = 0;
    return f;
}
inline int& assertions() {
    static int a = 0;
    return a;
}
inline std::vector<std::string>& captures() {
    static std::vector<std::string> c;
    return c;
}

inline void report(const char* file, int line, const char* what, bool require) {
    ++failures();
    std::fprintf(stderr, "%s:%d: %s FAILED: %s\n", file, line, require ? "REQUIRE" : "CHECK", what);
    for (const auto& c : captures()) std::fprintf(stderr, "    with %s\n", c.c_str());
    if (require) throw RequireFailed{};
}

struct CaptureGuard {
    template <typename T>
    CaptureGuard(const char* expr, const T& v) {
        std::ostringstream os;
        os << expr << " := " << v;
        captures().push_back(os.str());
    }
    ~CaptureGuard() { captures().pop_back(); }
};

inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        const int before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::fprintf(stderr, "%s:%d: TEST CASE '%s' threw: %s\n", c.file, c.line, c.name, e.what());
        } catch (...) {
            ++failures();
            std::fprintf(stderr, "%s:%d: TEST CASE '%s' threw an unknown exception\n", c.file, c.line, c.name);
        }
        captures().clear();
        const bool ok = failures() == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("test cases: %zu | %zu passed | %d failed | assertions: %d\n", registry().size(),
                registry().size() - static_cast<std::size_t>(failed_cases), failed_cases, assertions());
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                                             \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                             \
    static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                        \
        name, &DOCTEST_CAT(doctest_case_, __LINE__), __FILE__, __LINE__);                           \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()

#define DOCTEST_ASSERT_(expr, require)                                                              \
    do {                                                                                            \
        ++::doctest::detail::assertions();                                                          \
        if (!(expr)) ::doctest::detail::report(__FILE__, __LINE__, #expr, require);                 \
    } while (0)

#define CHECK(...) DOCTEST_ASSERT_((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_((__VA_ARGS__), true)
#define FAIL(msg) ::doctest::detail::report(__FILE__, __LINE__, "FAIL", true)
#define CAPTURE(x) ::doctest::detail::CaptureGuard DOCTEST_CAT(doctest_capture_, __LINE__)(#x, x)

#define CHECK_THROWS_AS(expr, ...)                                                                  \
    do {                                                                                            \
        ++::doctest::detail::assertions();                                                          \
        bool caught_ = false;                                                                       \
        try {                                                                                       \
            (void)(expr);                                                                           \
        } catch (const __VA_ARGS__&) {                                                              \
            caught_ = true;                                                                         \
        } catch (...) {                                                                             \
        }                                                                                           \
        if (!caught_) ::doctest::detail::report(__FILE__, __LINE__, #expr " throws " #__VA_ARGS__, false); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                    \
    do {                                                                                            \
        ++::doctest::detail::assertions();                                                          \
        bool ok_ = false;                                                                           \
        try {                                                                                       \
            (void)(expr);                                                                           \
        } catch (const __VA_ARGS__& e_) {                                                           \
            ok_ = (matcher).check(e_.what());                                                       \
        } catch (...) {                                                                             \
        }                                                                                           \
        if (!ok_) ::doctest::detail::report(__FILE__, __LINE__, #expr " throws " #__VA_ARGS__ " with " #matcher, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
