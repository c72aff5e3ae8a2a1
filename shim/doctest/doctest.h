// Minimal doctest-compatible test harness (the reference's test suites include <doctest.h>, which is vendored by
// its CMake build and absent from the image).  Covers exactly what proj/tests/*.cpp use: TEST_CASE, SUBCASE
// (re-entrant: the test body runs once per leaf subcase, as doctest does), CHECK / CHECK_FALSE / REQUIRE /
// CHECK_THROWS_AS / CHECK_NOTHROW / FAIL, doctest::Approx(...).epsilon(...) and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// Command line: --tc=<substring>[,<substring>...] runs only matching test cases; --list lists them.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

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
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.v_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.v_)));
    }
    friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
    friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }
    friend bool operator<=(double lhs, const Approx& r) { return lhs < r.v_ || lhs == r; }
    friend bool operator>=(double lhs, const Approx& r) { return lhs > r.v_ || lhs == r; }

private:
    double v_;
    double eps_ = 1.1920928955078125e-05;  // doctest's default: float epsilon * 100
    double scale_ = 1.0;
};

namespace detail {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Reg {
    Reg(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct RequireFailed {};

struct State {
    int sub_target = 0, sub_seen = 0;
    long checks = 0, failed_checks = 0;
    bool case_failed = false;
    std::string current_sub;
};
inline State& st() {
    static State s;
    return s;
}
inline bool enter_subcase(const char* name) {
    State& s = st();
    const bool in = s.sub_seen++ == s.sub_target;
    if (in) s.current_sub = name;
    return in;
}
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool require) {
    State& s = st();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    s.case_failed = true;
    std::printf("  %s:%d: FAILED %s( %s )%s%s\n", file, line, kind, expr, s.current_sub.empty() ? "" : "  [subcase ",
                s.current_sub.empty() ? "" : (s.current_sub + "]").c_str());
    if (require) throw RequireFailed{};
}

inline int run(int argc, char** argv) {
    std::vector<std::string> filters;
    bool list = false;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("--tc=", 0) == 0 || a.rfind("-tc=", 0) == 0) {
            std::string v = a.substr(a.find('=') + 1);
            size_t p = 0;
            while (p <= v.size()) {
                size_t q = v.find(',', p);
                if (q == std::string::npos) q = v.size();
                if (q > p) filters.push_back(v.substr(p, q - p));
                p = q + 1;
            }
        } else if (a == "--list") {
            list = true;
        }
    }
    int cases = 0, failed = 0;
    for (const TestCase& tc : registry()) {
        std::string nm = tc.name;
        if (!filters.empty() &&
            std::none_of(filters.begin(), filters.end(), [&](const std::string& f) { return nm.find(f) != nm.npos; }))
            continue;
        if (list) {
            std::printf("%s\n", tc.name);
            continue;
        }
        ++cases;
        State& s = st();
        s.case_failed = false;
        for (s.sub_target = 0;; ++s.sub_target) {
            s.sub_seen = 0;
            s.current_sub.clear();
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                s.case_failed = true;
                ++s.failed_checks;
                std::printf("  %s:%d: FAILED: unexpected exception: %s\n", tc.file, tc.line, e.what());
            } catch (...) {
                s.case_failed = true;
                ++s.failed_checks;
                std::printf("  %s:%d: FAILED: unexpected unknown exception\n", tc.file, tc.line);
            }
            if (s.sub_seen <= s.sub_target + 1) break;
        }
        std::printf("[%s] %s\n", s.case_failed ? "FAIL" : " ok ", tc.name);
        std::fflush(stdout);
        if (s.case_failed) ++failed;
    }
    if (!list)
        std::printf("test cases: %d | %d passed | %d failed; assertions: %ld | %ld failed\n", cases, cases - failed,
                    failed, st().checks, st().failed_checks);
    return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(f, name)                                                                 \
    static void f();                                                                         \
    static ::doctest::detail::Reg DOCTEST_CAT(f, _reg)(name, __FILE__, __LINE__, &f);        \
    static void f()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::detail::enter_subcase(name))
#define DOCTEST_CHECK_(kind, cond, expr, req)                                                      \
    do {                                                                                           \
        bool ok_ = false;                                                                          \
        try {                                                                                      \
            ok_ = static_cast<bool>(cond);                                                         \
        } catch (...) {                                                                            \
            ok_ = false;                                                                           \
        }                                                                                          \
        ::doctest::detail::report(ok_, kind, expr, __FILE__, __LINE__, req);                        \
    } while (0)
#define CHECK(...) DOCTEST_CHECK_("CHECK", (__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_CHECK_("CHECK_FALSE", !(__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_CHECK_("REQUIRE", (__VA_ARGS__), #__VA_ARGS__, true)
#define FAIL(msg)                                                                                   \
    ::doctest::detail::report(false, "FAIL", msg, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                                 \
    do {                                                                                           \
        bool ok_ = false;                                                                          \
        try {                                                                                      \
            (void)(expr);                                                                          \
        } catch (const __VA_ARGS__&) {                                                             \
            ok_ = true;                                                                            \
        } catch (...) {                                                                            \
        }                                                                                          \
        ::doctest::detail::report(ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_NOTHROW(...)                                                                         \
    do {                                                                                           \
        bool ok_ = true;                                                                           \
        try {                                                                                      \
            (void)(__VA_ARGS__);                                                                   \
        } catch (...) {                                                                            \
            ok_ = false;                                                                           \
        }                                                                                          \
        ::doctest::detail::report(ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, false);  \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
