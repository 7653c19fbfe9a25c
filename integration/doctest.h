// Minimal doctest-compatible shim: the subset deltakit's own unit tests use
// (P:tests/test_delta.cpp, test_serve.cpp): TEST_CASE, CHECK, CHECK_FALSE,
// CHECK_THROWS_AS, REQUIRE, FAIL, doctest::Approx (same tolerance rule as doctest
// 2.4: |a - b| < eps * (scale + max(|a|, |b|)), eps = 100 * FLT_EPSILON, scale 1).
// doctest itself is not in this image; the test sources compile unchanged against
// this header. main() lives in doctest_main.cpp.
#pragma once

#include <algorithm>
#include <cmath>
#include <iostream>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

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
struct Reg {
    Reg(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); }
};
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& assertions() {
    static int a = 0;
    return a;
}
struct RequireFailed {};
inline void report(const char* file, int line, const std::string& what) {
    std::cerr << file << ":" << line << ": FAILED: " << what << "\n";
    ++failures();
}

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + std::max(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator!=(const Approx& b, double a) { return !(a == b); }
    friend bool operator<=(double a, const Approx& b) { return a < b.v_ || a == b; }
    friend bool operator>=(double a, const Approx& b) { return a > b.v_ || a == b; }
    friend bool operator<(double a, const Approx& b) { return a < b.v_ && a != b; }
    friend bool operator>(double a, const Approx& b) { return a > b.v_ && a != b; }

private:
    double v_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double scale_ = 1.0;
};

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                            \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                              \
    static doctest::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_fn_, __LINE__), \
                                                            __FILE__, __LINE__);                   \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...)                                                                       \
    do {                                                                                 \
        ++doctest::assertions();                                                         \
        if (!(__VA_ARGS__)) doctest::report(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
    } while (0)
#define CHECK_FALSE(...)                                                                       \
    do {                                                                                       \
        ++doctest::assertions();                                                               \
        if ((__VA_ARGS__)) doctest::report(__FILE__, __LINE__, "CHECK_FALSE(" #__VA_ARGS__ ")"); \
    } while (0)
#define REQUIRE(...)                                                             \
    do {                                                                         \
        ++doctest::assertions();                                                 \
        if (!(__VA_ARGS__)) {                                                    \
            doctest::report(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");    \
            throw doctest::RequireFailed{};                                      \
        }                                                                        \
    } while (0)
#define FAIL(msg)                                            \
    do {                                                     \
        doctest::report(__FILE__, __LINE__, std::string(msg)); \
        throw doctest::RequireFailed{};                      \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                          \
    do {                                                                                    \
        ++doctest::assertions();                                                            \
        bool doctest_ok_ = false;                                                           \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (const __VA_ARGS__&) {                                                      \
            doctest_ok_ = true;                                                             \
        } catch (...) {                                                                     \
        }                                                                                   \
        if (!doctest_ok_)                                                                   \
            doctest::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); \
    } while (0)
