// Minimal stand-in for doctest (not in this image): the macros the
// reference's unit tests use -- TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW, doctest::Approx -- with a main that runs
// every registered case and prints doctest's summary line. TEST INFRASTRUCTURE.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline int& failures() {
    static int f = 0;
    return f;
}
inline bool& case_failed() {
    static bool f = false;
    return f;
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
inline void fail(const char* file, int line, const char* expr) {
    std::printf("%s:%d: CHECK( %s ) failed\n", file, line, expr);
    ++failures();
    case_failed() = true;
}
struct RequireFailed {};
class Approx {
  public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) <= b.eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }

  private:
    double v_, eps_ = 1.1920928955078125e-05 * 100;
};
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE_IMPL(fn, name)                                             \
    static void fn();                                                        \
    static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);              \
    static void fn()
#define TEST_CASE(name) TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define CHECK(...) \
    do { if (!(__VA_ARGS__)) doctest::fail(__FILE__, __LINE__, #__VA_ARGS__); } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                     \
    do {                                                                                 \
        if (!(__VA_ARGS__)) {                                                            \
            doctest::fail(__FILE__, __LINE__, #__VA_ARGS__);                             \
            throw doctest::RequireFailed{};                                              \
        }                                                                                \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                           \
    do {                                                                      \
        bool caught_ = false;                                                 \
        try {                                                                 \
            (void)(expr);                                                     \
        } catch (const type&) {                                               \
            caught_ = true;                                                   \
        } catch (...) {                                                       \
        }                                                                     \
        if (!caught_) doctest::fail(__FILE__, __LINE__, "throws " #type ": " #expr); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                  \
    do {                                                                     \
        try {                                                                \
            (void)(expr);                                                    \
        } catch (...) {                                                      \
            doctest::fail(__FILE__, __LINE__, "nothrow: " #expr);            \
        }                                                                    \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0, n = 0;
    for (const doctest::Case& c : doctest::registry()) {
        ++n;
        doctest::case_failed() = false;
        try {
            c.fn();
        } catch (const doctest::RequireFailed&) {
        } catch (const std::exception& e) {
            std::printf("TEST CASE \"%s\": unexpected exception: %s\n", c.name, e.what());
            doctest::case_failed() = true;
        }
        if (doctest::case_failed()) {
            ++failed_cases;
            std::printf("TEST CASE \"%s\" FAILED\n", c.name);
        }
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed\n", n, n - failed_cases, failed_cases);
    return failed_cases == 0 ? 0 : 1;
}
#endif
