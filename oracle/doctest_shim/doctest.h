// doctest.h -- minimal stand-in for the doctest macros the reference's unit tests use
// (TEST_CASE, CHECK[_FALSE], REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CAPTURE,
// doctest::Approx).  TEST INFRASTRUCTURE ONLY: doctest itself is not vendored in the
// reference mount (proj/.gitignore) and there is no network.  It lets
// proj/tests/test_*.cpp compile UNMODIFIED against include/taco/*.hpp and run against
// libtaco_b200.so (oracle/Makefile target `reftests`).
#pragma once
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    Approx& scale(double s) { scl = s; return *this; }
    double value, eps = std::numeric_limits<float>::epsilon() * 100, scl = 1.0;
};
inline bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value) < r.eps * (r.scl + std::max(std::fabs(lhs), std::fabs(r.value)));
}
inline bool operator==(const Approx& r, double lhs) { return lhs == r; }
inline bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }

namespace detail {
struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct Abort {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}
inline const char*& current() {
    static const char* c = "";
    return c;
}
inline void report(const char* file, int line, const char* what) {
    ++failures();
    std::printf("%s:%d: ERROR in \"%s\": %s\n", file, line, current(), what);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                                  \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                                    \
    static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__,          \
                                                                    &DOCTEST_CAT(doctest_fn_, __LINE__)); \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define DOCTEST_CHECK_IMPL(cond, text, fatal)                                              \
    do {                                                                                   \
        ++doctest::detail::checks();                                                       \
        bool ok_ = false;                                                                  \
        try { ok_ = static_cast<bool>(cond); } catch (const std::exception& e_) {           \
            doctest::detail::report(__FILE__, __LINE__, (std::string("threw: ") + e_.what()).c_str()); \
            if (fatal) throw doctest::detail::Abort{};                                     \
            break;                                                                         \
        }                                                                                  \
        if (!ok_) {                                                                        \
            doctest::detail::report(__FILE__, __LINE__, text);                             \
            if (fatal) throw doctest::detail::Abort{};                                     \
        }                                                                                  \
    } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), "CHECK( " #__VA_ARGS__ " )", false)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), "CHECK_FALSE( " #__VA_ARGS__ " )", false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), "REQUIRE( " #__VA_ARGS__ " )", true)
#define CHECK_THROWS_AS(expr, type)                                                                 \
    do {                                                                                            \
        ++doctest::detail::checks();                                                                \
        bool got_ = false;                                                                          \
        try { (void)(expr); } catch (const type&) { got_ = true; } catch (...) {}                    \
        if (!got_) doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #type " )"); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, type)                                                       \
    do {                                                                                            \
        ++doctest::detail::checks();                                                                \
        bool got_ = false;                                                                          \
        std::string what_ = "<no exception>";                                                       \
        try { (void)(expr); } catch (const type& e_) { what_ = e_.what(); got_ = what_ == std::string(msg); } \
        catch (const std::exception& e_) { what_ = e_.what(); } catch (...) {}                       \
        if (!got_) doctest::detail::report(__FILE__, __LINE__, (std::string("CHECK_THROWS_WITH_AS( " #expr ", ") + \
                                            msg + " ) got: " + what_).c_str());                    \
    } while (0)
#define CAPTURE(x) ((void)0)
#define FAIL(msg)                                                    \
    do {                                                             \
        doctest::detail::report(__FILE__, __LINE__, "FAIL: " msg);  \
        throw doctest::detail::Abort{};                              \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0, n = 0;
    for (auto& c : doctest::detail::registry()) {
        ++n;
        doctest::detail::current() = c.name;
        const int before = doctest::detail::failures();
        try {
            c.fn();
        } catch (const doctest::detail::Abort&) {
        } catch (const std::exception& e) {
            doctest::detail::report(c.file, c.line, (std::string("unexpected exception: ") + e.what()).c_str());
        }
        const bool ok = doctest::detail::failures() == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %d | %d failed\n", n,
                n - failed_cases, failed_cases, doctest::detail::checks(), doctest::detail::failures());
    return failed_cases ? 1 : 0;
}
#endif
