// Minimal doctest-compatible test shim (test infrastructure, not product).
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) include
// <doctest.h> from a vendor/ directory that is absent from the reference
// checkout. This header implements exactly the subset those files use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH,
// doctest::Approx(..).epsilon(..)) so the unmodified test sources compile
// against either the reference library (oracle/_ref) or the B200 library.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <stdexcept>
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
    // doctest semantics: |a - b| < eps * (scale + max(|a|, |b|)), scale = 1
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

  private:
    double value_;
    double eps_ = 1.1920929e-7 * 100;
};

namespace detail {

struct Registry {
    struct Case {
        const char* name;
        void (*fn)();
    };
    std::vector<Case> cases;
    long long checks = 0;
    long long failures = 0;
    static Registry& get() {
        static Registry r;
        return r;
    }
};

struct RequireFailed {};

struct Registrar {
    Registrar(const char* name, void (*fn)()) { Registry::get().cases.push_back({name, fn}); }
};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    Registry& r = Registry::get();
    ++r.checks;
    if (ok) return;
    ++r.failures;
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
    if (fatal) throw RequireFailed{};
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                              \
    static void fn();                                                                 \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);               \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, exc)                                                     \
    do {                                                                               \
        bool doctest_ok_ = false;                                                      \
        try {                                                                          \
            (void)(expr);                                                              \
        } catch (const exc&) {                                                         \
            doctest_ok_ = true;                                                        \
        } catch (...) {                                                                \
        }                                                                              \
        doctest::detail::report(doctest_ok_, "throws " #exc ": " #expr, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_THROWS_WITH(expr, msg)                                                   \
    do {                                                                               \
        bool doctest_ok_ = false;                                                      \
        try {                                                                          \
            (void)(expr);                                                              \
        } catch (const std::exception& e_) {                                           \
            doctest_ok_ = std::string(e_.what()) == std::string(msg);                  \
        } catch (...) {                                                                \
        }                                                                              \
        doctest::detail::report(doctest_ok_, "throws '" msg "': " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    auto& r = doctest::detail::Registry::get();
    int failed_cases = 0;
    for (const auto& c : r.cases) {
        const long long before = r.failures;
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "test case '%s' threw: %s\n", c.name, e.what());
            ++r.failures;
        }
        if (r.failures != before) {
            ++failed_cases;
            std::fprintf(stderr, "[case failed] %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %lld | %lld failed\n",
                r.cases.size(), r.cases.size() - failed_cases, failed_cases, r.checks, r.failures);
    return failed_cases == 0 ? 0 : 1;
}
#endif
