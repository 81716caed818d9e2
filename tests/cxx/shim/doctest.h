// doctest.h -- a minimal stand-in for the doctest macros the reference's test files use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS, CHECK_THROWS_AS, doctest::Approx),
// so proj/tests/*.cpp compile UNMODIFIED against the drop-in headers (include/ngram).  The
// reference build fetches doctest itself; this image has no copy.
// TEST INFRASTRUCTURE ONLY.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {
namespace detail {
struct test_entry {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<test_entry>& registry() {
    static std::vector<test_entry> r;
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
struct registrar {
    registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};
struct require_failed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    ++checks();
    if (ok) return;
    ++failures();
    std::printf("%s:%d: FAILED: %s( %s )\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw require_failed{};
}
}  // namespace detail

// doctest::Approx: |a - b| < epsilon * (scale + max(|a|, |b|)), default epsilon = float eps * 100
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
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.value_) < b.eps_ * (b.scale_ + std::fmax(std::fabs(a), std::fabs(b.value_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator!=(const Approx& b, double a) { return !(a == b); }

  private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;
    double scale_ = 1.0;
};
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_(fn, name)                                                              \
    static void fn();                                                                             \
    static doctest::detail::registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);       \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_(DOCTEST_CAT(doctest_test_, __COUNTER__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS(...)                                                                          \
    do {                                                                                           \
        bool thrown_ = false;                                                                      \
        try {                                                                                      \
            (void)(__VA_ARGS__);                                                                   \
        } catch (...) {                                                                            \
            thrown_ = true;                                                                        \
        }                                                                                          \
        doctest::detail::report(thrown_, "THROWS " #__VA_ARGS__, __FILE__, __LINE__, false);       \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                 \
    do {                                                                                           \
        bool thrown_ = false;                                                                      \
        try {                                                                                      \
            (void)(expr);                                                                          \
        } catch (const __VA_ARGS__&) {                                                             \
            thrown_ = true;                                                                        \
        } catch (...) {                                                                            \
        }                                                                                          \
        doctest::detail::report(thrown_, "THROWS_AS " #expr ", " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& t : doctest::detail::registry()) {
        const int before = doctest::detail::failures();
        try {
            t.fn();
        } catch (const doctest::detail::require_failed&) {
        } catch (const std::exception& e) {
            ++doctest::detail::failures();
            std::printf("%s:%d: unexpected exception: %s\n", t.file, t.line, e.what());
        }
        const bool ok = doctest::detail::failures() == before;
        failed_cases += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? "ok" : "FAILED", t.name);
    }
    std::printf("[doctest] test cases: %zu | %zu passed | %d failed | checks: %d | failures: %d\n",
                doctest::detail::registry().size(), doctest::detail::registry().size() - size_t(failed_cases),
                failed_cases, doctest::detail::checks(), doctest::detail::failures());
    return failed_cases == 0 ? 0 : 1;
}
#endif
