// Minimal doctest-compatible test harness (our own, for compiling test cases
// written against the doctest API without the vendored doctest, which the
// reference keeps out of its tree): TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW and doctest::Approx with doctest's published
// comparison rule |a - b| < eps * (scale + max(|a|, |b|)).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
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
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
    }
    friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
    friend bool operator<=(double lhs, const Approx& r) { return lhs < r.value_ || lhs == r; }
    friend bool operator>=(double lhs, const Approx& r) { return lhs > r.value_ || lhs == r; }

  private:
    double value_, eps_ = 1.1920929e-05, scale_ = 1.0;  // float epsilon * 100, as doctest
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> cases;
    return cases;
}
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    ++checks();
    if (ok) return;
    ++failures();
    std::printf("%s:%d: FAILED %s\n", file, line, expr);
    if (require) throw RequireFailed{};
}
inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        const int before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::printf("TEST CASE \"%s\" threw: %s\n", c.name, e.what());
        }
        if (failures() != before) {
            ++failed_cases;
            std::printf("TEST CASE \"%s\" failed\n", c.name);
        }
    }
    std::printf("[doctest shim] test cases: %zu | %d failed | assertions: %d | %d failed\n", registry().size(),
                failed_cases, checks(), failures());
    return failures() == 0 ? 0 : 1;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_IMPL(fn, reg, name)                                  \
    static void fn();                                                     \
    static const ::doctest::detail::Registrar reg(name, &fn);             \
    static void fn()
#define TEST_CASE(name) \
    DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), DOCTEST_CAT(doctest_reg_, __LINE__), name)
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                      \
    do {                                                                                 \
        bool doctest_ok_ = false;                                                        \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (const type&) {                                                          \
            doctest_ok_ = true;                                                          \
        } catch (...) {                                                                  \
        }                                                                                \
        ::doctest::detail::report(doctest_ok_, #expr " throws " #type, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                              \
    do {                                                                                 \
        bool doctest_ok_ = true;                                                         \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (...) {                                                                  \
            doctest_ok_ = false;                                                         \
        }                                                                                \
        ::doctest::detail::report(doctest_ok_, #expr " does not throw", __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
