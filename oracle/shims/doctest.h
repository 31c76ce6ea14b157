/*
 * TEST INFRASTRUCTURE ONLY (oracle build shim).
 *
 * Minimal doctest-compatible header so the reference's own
 * tests/test_fc_core.cpp can be compiled, unmodified, against the shimmed
 * oracle build (doctest.h is expected under the git-ignored /vendor and is
 * absent from the image). Supports TEST_CASE, CHECK,
 * CHECK_THROWS_AS and doctest::Approx(...).epsilon(...), with doctest's
 * published Approx rule |a-b| < eps*(scale + max(|a|,|b|)), scale = 1,
 * default eps = 100 * FLT_EPSILON.
 */
#ifndef ORACLE_SHIM_DOCTEST_H
#define ORACLE_SHIM_DOCTEST_H

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct TestEntry {
    const char* name;
    void (*fn)();
};
inline std::vector<TestEntry>& registry() {
    static std::vector<TestEntry> r;
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
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

class Approx {
  public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    bool eq(double o) const {
        return std::fabs(o - v_) < eps_ * (1.0 + std::max(std::fabs(o), std::fabs(v_)));
    }
    friend bool operator==(double a, const Approx& b) { return b.eq(a); }
    friend bool operator==(const Approx& a, double b) { return a.eq(b); }

  private:
    double v_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100;
};

inline void report(bool ok, const char* expr, const char* file, int line) {
    ++checks();
    if (!ok) {
        ++failures();
        std::printf("%s:%d: CHECK FAILED: %s\n", file, line, expr);
    }
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                   \
    static void fn();                                                               \
    static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);                     \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define CHECK(expr) doctest::report(static_cast<bool>(expr), #expr, __FILE__, __LINE__)
#define CHECK_THROWS_AS(expr, exc)                                                  \
    do {                                                                            \
        bool caught_ = false;                                                       \
        try {                                                                       \
            (void)(expr);                                                           \
        } catch (const exc&) {                                                      \
            caught_ = true;                                                         \
        } catch (...) {                                                             \
        }                                                                           \
        doctest::report(caught_, "THROWS_AS(" #expr ", " #exc ")", __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& t : doctest::registry()) {
        const int before = doctest::failures();
        t.fn();
        const bool ok = doctest::failures() == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", t.name);
    }
    std::printf("test cases: %zu, failed: %d; checks: %d, failed: %d\n", doctest::registry().size(),
                failed_cases, doctest::checks(), doctest::failures());
    return failed_cases == 0 ? 0 : 1;
}
#endif

#endif
