// Minimal doctest-compatible subset (TEST INFRASTRUCTURE): the macros the
// reference's unit tests use (TEST_CASE, CHECK, CHECK_FALSE, CHECK_THROWS_AS,
// REQUIRE, doctest::Approx), so its test files compile where they lie
// (proj/tests/*.cpp) without the doctest package, which this image lacks.
// Approx follows doctest's comparison: |a - b| < eps * (scale + max(|a|, |b|)),
// eps defaulting to 100 float epsilons, scale to 1.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
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

private:
    double v_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

// exception-message matcher of CHECK_THROWS_WITH_AS: substring
struct Contains {
    explicit Contains(std::string s) : sub(std::move(s)) {}
    bool matches(const std::string& what) const { return what.find(sub) != std::string::npos; }
    std::string sub;
};

namespace detail {
inline bool msgMatches(const Contains& m, const std::string& what) { return m.matches(what); }
inline bool msgMatches(const char* m, const std::string& what) { return what == m; }
inline bool msgMatches(const std::string& m, const std::string& what) { return what == m; }
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
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct RequireFailed {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline const char*& current() {
    static const char* c = "";
    return c;
}
inline void report(bool ok, const char* what, const char* file, int line) {
    if (ok) return;
    ++failures();
    std::printf("FAIL [%s] %s:%d: %s\n", current(), file, line, what);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                              \
    static void fn();                                                                                      \
    static const doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);          \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                                        \
    do {                                                                                                    \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                            \
        doctest::detail::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);                            \
        if (!doctest_ok_) throw doctest::detail::RequireFailed{};                                           \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                          \
    do {                                                                                                    \
        bool doctest_ok_ = false;                                                                           \
        try {                                                                                               \
            static_cast<void>(expr);                                                                        \
        } catch (const __VA_ARGS__&) {                                                                      \
            doctest_ok_ = true;                                                                             \
        } catch (...) {                                                                                     \
        }                                                                                                   \
        doctest::detail::report(doctest_ok_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__);          \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                           \
    do {                                                                                                    \
        bool doctest_ok_ = false;                                                                           \
        try {                                                                                               \
            static_cast<void>(expr);                                                                        \
        } catch (const __VA_ARGS__& e) {                                                                    \
            doctest_ok_ = doctest::detail::msgMatches(matcher, e.what());                                   \
        } catch (...) {                                                                                     \
        }                                                                                                   \
        doctest::detail::report(doctest_ok_, #expr " throws " #__VA_ARGS__ " with " #matcher, __FILE__,    \
                                __LINE__);                                                                  \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failedCases = 0;
    for (const auto& c : doctest::detail::registry()) {
        const int before = doctest::detail::failures();
        doctest::detail::current() = c.name;
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++doctest::detail::failures();
            std::printf("FAIL [%s] unexpected exception: %s\n", c.name, e.what());
        } catch (...) {
            ++doctest::detail::failures();
            std::printf("FAIL [%s] unexpected exception\n", c.name);
        }
        const bool ok = doctest::detail::failures() == before;
        if (!ok) ++failedCases;
        std::printf("%s %s\n", ok ? "ok  " : "FAIL", c.name);
    }
    std::printf("test cases: %zu | passed: %zu | failed: %d\n", doctest::detail::registry().size(),
                doctest::detail::registry().size() - failedCases, failedCases);
    return failedCases ? 1 : 0;
}
#endif
