// TEST INFRASTRUCTURE ONLY (oracle). Minimal doctest-compatible header so the
// reference's unit suites (/root/reference/proj/tests/test_*.cpp) compile and
// run unmodified without the vendored doctest (absent: proj/.gitignore:2).
// Implements only what those suites use: TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx(..).epsilon(..),
// doctest::Contains, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Approx follows the
// published doctest rule |a-b| < eps*(scale + max(|a|,|b|)), scale=1,
// default eps = 100*FLT_EPSILON.
#pragma once
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
namespace detail {
struct TestCase {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}
struct RequireFailed {};
struct Registrar {
    Registrar(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); }
};
inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
    ++checks();
    if (!ok) {
        ++failures();
        std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
        if (require) throw RequireFailed{};
    }
}
}  // namespace detail

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
    }
    friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }

private:
    double value_;
    double eps_ = 100.0 * FLT_EPSILON;
    double scale_ = 1.0;
};

struct Contains {
    explicit Contains(const char* s) : str(s) {}
    std::string str;
    bool matches(const std::string& what) const { return what.find(str) != std::string::npos; }
};
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                           \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                             \
    static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                      \
        name, &DOCTEST_CAT(doctest_fn_, __LINE__), __FILE__, __LINE__);                           \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                               \
    do {                                                                                          \
        bool doctest_ok_ = false;                                                                 \
        try {                                                                                     \
            (void)(expr);                                                                         \
        } catch (const type&) {                                                                   \
            doctest_ok_ = true;                                                                   \
        } catch (...) {                                                                           \
        }                                                                                         \
        ::doctest::detail::check(doctest_ok_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                                 \
    do {                                                                                          \
        bool doctest_ok_ = false;                                                                 \
        try {                                                                                     \
            (void)(expr);                                                                         \
        } catch (const type& e_) {                                                                \
            doctest_ok_ = (matcher).matches(e_.what());                                           \
        } catch (...) {                                                                           \
        }                                                                                         \
        ::doctest::detail::check(doctest_ok_, "throws-with " #type ": " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int cases_failed = 0;
    for (auto& tc : ::doctest::detail::registry()) {
        int before = ::doctest::detail::failures();
        try {
            tc.fn();
        } catch (const ::doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++::doctest::detail::failures();
            std::fprintf(stderr, "%s:%d: unexpected exception in \"%s\": %s\n", tc.file, tc.line, tc.name, e.what());
        }
        if (::doctest::detail::failures() != before) {
            ++cases_failed;
            std::fprintf(stderr, "TEST CASE FAILED: %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | passed: %zu | failed: %d | checks: %d | failed checks: %d\n",
                ::doctest::detail::registry().size(), ::doctest::detail::registry().size() - cases_failed,
                cases_failed, ::doctest::detail::checks(), ::doctest::detail::failures());
    return cases_failed == 0 ? 0 : 1;
}
#endif
