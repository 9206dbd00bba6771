// TEST INFRASTRUCTURE — a minimal doctest-compatible harness (doctest itself is absent from
// this image).  Implements exactly the macros the reference's suites use:
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// CHECK_NOTHROW, doctest::Approx(..).epsilon(..), doctest::Contains.  Lets the reference's
// own test files compile unchanged against the drop-in library.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
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
    friend bool operator==(double a, const Approx& b) {
        return std::abs(a - b.v_) < b.eps_ * (1.0 + std::max(std::abs(a), std::abs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }

private:
    double v_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
};

struct Contains {
    std::string s;
    explicit Contains(const char* x) : s(x) {}
    bool operator()(const std::string& what) const { return what.find(s) != std::string::npos; }
};

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
struct Stats {
    long checks = 0, failed = 0;
    const char* current = "";
    bool case_failed = false;
};
inline Stats& stats() {
    static Stats s;
    return s;
}
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    Stats& s = stats();
    ++s.checks;
    if (ok) return;
    ++s.failed;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, s.current, expr);
    if (require) throw RequireFailed{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC(fn, name)                                                                       \
    static void fn();                                                                              \
    static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);            \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, Type)                                                                \
    do {                                                                                           \
        bool _ok = false;                                                                          \
        try {                                                                                      \
            (void)(expr);                                                                          \
        } catch (const Type&) {                                                                    \
            _ok = true;                                                                            \
        } catch (...) {                                                                            \
        }                                                                                          \
        ::doctest::detail::report(_ok, "throws " #Type ": " #expr, __FILE__, __LINE__, false);     \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, Type)                                                  \
    do {                                                                                           \
        bool _ok = false;                                                                          \
        try {                                                                                      \
            (void)(expr);                                                                          \
        } catch (const Type& _e) {                                                                 \
            _ok = (matcher)(std::string(_e.what()));                                               \
        } catch (...) {                                                                            \
        }                                                                                          \
        ::doctest::detail::report(_ok, "throws " #Type " with message: " #expr, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_NOTHROW(expr)                                                                        \
    do {                                                                                           \
        bool _ok = true;                                                                           \
        try {                                                                                      \
            (void)(expr);                                                                          \
        } catch (...) {                                                                            \
            _ok = false;                                                                           \
        }                                                                                          \
        ::doctest::detail::report(_ok, "no throw: " #expr, __FILE__, __LINE__, false);             \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const char* only = argc > 1 ? argv[1] : nullptr;
    auto& S = ::doctest::detail::stats();
    int cases = 0, failed_cases = 0;
    for (const auto& c : ::doctest::detail::registry()) {
        if (only && std::strstr(c.name, only) == nullptr) continue;
        ++cases;
        S.current = c.name;
        S.case_failed = false;
        try {
            c.fn();
        } catch (const ::doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
            ++S.failed;
            S.case_failed = true;
        }
        if (S.case_failed) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n", cases,
                cases - failed_cases, failed_cases, S.checks, S.failed);
    return failed_cases ? 1 : 0;
}
#endif
