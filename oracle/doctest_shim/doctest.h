// Minimal doctest-compatible shim (TEST INFRASTRUCTURE ONLY).
// doctest itself is not in this image; this header implements the subset the
// reference tests use so that the reference's own
// test_label.cpp / test_grid.cpp compile unmodified from /root/reference and
// pin the reference build that oracle/_ref uses.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
    double v, eps = 1e-5;
    explicit Approx(double x) : v(x) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v) <= b.eps * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
};
namespace detail {
struct Case { const char* name; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline int& failures() { static int f = 0; return f; }
struct Reg { Reg(const char* n, void (*f)()) { registry().push_back({n, f}); } };
struct Abort {};
inline void report(const char* file, int line, const char* what) {
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what);
    ++failures();
}
}  // namespace detail
}  // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define DT_TEST(fn, name)                                                  \
    static void fn();                                                      \
    static ::doctest::detail::Reg DT_CAT(fn, _reg)(name, &fn);             \
    static void fn()
#define TEST_CASE(name) DT_TEST(DT_CAT(dt_case_, __LINE__), name)
#define SUBCASE(name) if (true)
#define CAPTURE(x) ((void)0)
#define INFO(...) ((void)0)
#define MESSAGE(...) ((void)0)
#define FAIL(msg)                                                          \
    do { ::doctest::detail::report(__FILE__, __LINE__, "FAIL");            \
         throw ::doctest::detail::Abort{}; } while (0)
#define CHECK(...)                                                         \
    do { if (!(__VA_ARGS__)) ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__); } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                       \
    do { if (!(__VA_ARGS__)) { ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__); \
         throw ::doctest::detail::Abort{}; } } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, T)                                           \
    do { bool dt_ok_ = false;                                              \
         try { (void)(expr); } catch (const T&) { dt_ok_ = true; } catch (...) {} \
         if (!dt_ok_) ::doctest::detail::report(__FILE__, __LINE__, "throws " #T); } while (0)
#define CHECK_THROWS(expr)                                                 \
    do { bool dt_ok_ = false;                                              \
         try { (void)(expr); } catch (...) { dt_ok_ = true; }              \
         if (!dt_ok_) ::doctest::detail::report(__FILE__, __LINE__, "throws"); } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, T)                                 \
    do { bool dt_ok_ = false;                                              \
         try { (void)(expr); } catch (const T& dt_e_) {                    \
             dt_ok_ = std::string(dt_e_.what()) == std::string(msg); } catch (...) {} \
         if (!dt_ok_) ::doctest::detail::report(__FILE__, __LINE__, "throws-with " #T); } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int cases = 0, failed_cases = 0;
    for (auto& c : ::doctest::detail::registry()) {
        const int before = ::doctest::detail::failures();
        ++cases;
        try { c.fn(); } catch (const ::doctest::detail::Abort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "case '%s' threw: %s\n", c.name, e.what());
            ++::doctest::detail::failures();
        }
        if (::doctest::detail::failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d\n", cases,
                cases - failed_cases, failed_cases);
    return failed_cases ? 1 : 0;
}
#endif
