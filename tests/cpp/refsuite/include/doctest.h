// doctest.h — the subset of doctest the reference's unit suite uses
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_NOTHROW, CHECK_THROWS_AS,
// doctest::Approx with epsilon), so proj/tests/test_*.cpp compile unchanged without the vendored
// header (absent from the reference).  Test infrastructure.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx &epsilon(double e)
    {
        eps = e;
        return *this;
    }
    double value;
    double eps = 1.1920929e-7 * 100;  // doctest's default: float epsilon * 100
};
inline bool operator==(double a, const Approx &b)
{
    return std::fabs(a - b.value) < b.eps * (1.0 + std::fmax(std::fabs(a), std::fabs(b.value)));
}
inline bool operator==(const Approx &b, double a) { return a == b; }
inline bool operator!=(double a, const Approx &b) { return !(a == b); }

namespace detail {
struct Case {
    const char *name, *file;
    int line;
    void (*fn)();
};
inline std::vector<Case> &registry()
{
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(const char *n, const char *f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
inline int &failures()
{
    static int n = 0;
    return n;
}
inline int &checks()
{
    static int n = 0;
    return n;
}
inline const char *&current()
{
    static const char *c = "";
    return c;
}
inline void fail(const char *file, int line, const char *what)
{
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, current(), what);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                              \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                              \
    static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__,        \
                                                                    &DOCTEST_CAT(doctest_case_, __LINE__)); \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define CHECK(...)                                                                       \
    do {                                                                                 \
        ++doctest::detail::checks();                                                     \
        if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
// REQUIRE: a failed requirement ends the test case (doctest throws too)
namespace doctest { namespace detail { struct RequireFailed {}; } }
#define REQUIRE(...)                                                                     \
    do {                                                                                 \
        ++doctest::detail::checks();                                                     \
        if (!(__VA_ARGS__)) {                                                            \
            doctest::detail::fail(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");     \
            throw doctest::detail::RequireFailed{};                                      \
        }                                                                                \
    } while (0)
#define CHECK_NOTHROW(...)                                                               \
    do {                                                                                 \
        ++doctest::detail::checks();                                                     \
        try {                                                                            \
            __VA_ARGS__;                                                                 \
        } catch (const std::exception &e) {                                            \
            doctest::detail::fail(__FILE__, __LINE__, ("CHECK_NOTHROW threw: " + std::string(e.what())).c_str()); \
        }                                                                                \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                      \
    do {                                                                                 \
        ++doctest::detail::checks();                                                     \
        bool doctest_threw = false;                                                      \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (const type &) {                                                         \
            doctest_threw = true;                                                        \
        } catch (...) {                                                                  \
        }                                                                                \
        if (!doctest_threw) doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #type ")"); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char **argv)
{
    // optional filter: run only test cases whose name contains argv[1]
    const char *filter = argc > 1 ? argv[1] : nullptr;
    int cases = 0, failed_cases = 0;
    for (auto &c : doctest::detail::registry()) {
        if (filter && std::string(c.name).find(filter) == std::string::npos) continue;
        const int before = doctest::detail::failures();
        doctest::detail::current() = c.name;
        ++cases;
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed &) {
            // recorded by REQUIRE
        } catch (const std::exception &e) {
            doctest::detail::fail(c.file, c.line, ("unexpected exception: " + std::string(e.what())).c_str());
        }
        const bool ok = doctest::detail::failures() == before;
        failed_cases += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? "pass" : "FAIL", c.name);
    }
    std::printf("test cases: %d | %d passed | %d failed; checks: %d, failed: %d\n", cases, cases - failed_cases,
                failed_cases, doctest::detail::checks(), doctest::detail::failures());
    return failed_cases == 0 ? 0 : 1;
}
#endif
