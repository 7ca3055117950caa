// TEST INFRASTRUCTURE ONLY - a minimal doctest-compatible harness, just enough
// to compile the reference's own hot-path unit tests
// (proj/tests/test_{ensf,rng,ensemble,parallel}.cpp) against the B200
// library.  doctest itself is not shipped with the reference (proj/vendor/ is
// absent); this is an independent implementation of the macros those files
// use.  Reports one line per failed check and a summary per test case.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + std::fmax(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }

private:
    double v_;
    double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default: float eps * 100
    double scale_ = 1.0;
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
inline int& failures() {
    static int f = 0;
    return f;
}
struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) {
        registry().push_back({name, fn, file, line});
    }
};
struct RequireFailed {};
inline void report(const char* file, int line, const char* what) {
    ++failures();
    std::printf("  CHECK FAILED %s:%d: %s\n", file, line, what);
}
}  // namespace detail
}  // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define DT_CASE(fn, name)                                                                     \
    static void fn();                                                                         \
    static doctest::detail::Registrar DT_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);        \
    static void fn()
#define TEST_CASE(name) DT_CASE(DT_CAT(dt_case_, __LINE__), name)

#define CHECK(...)                                                                            \
    do {                                                                                      \
        if (!(__VA_ARGS__)) doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);         \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                          \
    do {                                                                                      \
        if (!(__VA_ARGS__)) {                                                                 \
            doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);                        \
            throw doctest::detail::RequireFailed{};                                          \
        }                                                                                     \
    } while (0)
#define FAIL(msg)                                                                             \
    do {                                                                                      \
        doctest::detail::report(__FILE__, __LINE__, msg);                                     \
        throw doctest::detail::RequireFailed{};                                              \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                           \
    do {                                                                                      \
        bool caught_ = false;                                                                 \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const type&) {                                                               \
            caught_ = true;                                                                   \
        } catch (...) {                                                                       \
        }                                                                                     \
        if (!caught_) doctest::detail::report(__FILE__, __LINE__, "throws " #type ": " #expr); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                   \
    do {                                                                                      \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (...) {                                                                       \
            doctest::detail::report(__FILE__, __LINE__, "nothrow: " #expr);                   \
        }                                                                                     \
    } while (0)
