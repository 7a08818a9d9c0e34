// TEST INFRASTRUCTURE: minimal doctest-compatible harness (doctest itself is not
// vendored with the reference: proj/.gitignore:2, and there is no network).  It
// implements exactly what the reference's unit suite uses (proj/tests/test_*.cpp):
// TEST_CASE, flat SUBCASE (each subcase runs in its own pass of the test case, as
// in doctest), CHECK / CHECK_FALSE / REQUIRE / CHECK_THROWS_AS / FAIL / CAPTURE /
// MESSAGE and doctest::Approx with doctest's comparison rule.  Used only to build
// oracle/_ref/unit_tests from the reference's own sources (oracle/Makefile.ref).
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
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        // doctest: |lhs - value| < eps * (scale + max(|lhs|, |value|))
        return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
    friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || lhs == a; }
    friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || lhs == a; }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace shim {
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
struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) { registry().push_back({name, fn, file, line}); }
};
struct State {
    int target = 0, seen = 0;
    long checks = 0, failed_checks = 0;
    bool case_failed = false;
};
inline State& st() {
    static State s;
    return s;
}
struct Abort {};
inline void report(const char* file, int line, const char* what) {
    std::printf("%s:%d: FAILED: %s\n", file, line, what);
    st().failed_checks++;
    st().case_failed = true;
}
inline void check(bool ok, const char* file, int line, const char* expr, bool require) {
    st().checks++;
    if (!ok) {
        report(file, line, expr);
        if (require) throw Abort{};
    }
}
struct Subcase {
    bool enter;
    Subcase(const char*, const char*, int) : enter(st().seen++ == st().target) {}
    explicit operator bool() const { return enter; }
};
}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                \
    static void fn();                                                                        \
    static ::doctest::shim::Registrar DOCTEST_CAT(fn, _reg)(name, fn, __FILE__, __LINE__);   \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::shim::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name, __FILE__, __LINE__})
#define CHECK(...) ::doctest::shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) ::doctest::shim::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) ::doctest::shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define CHECK_THROWS_AS(expr, ...)                                                                         \
    do {                                                                                                   \
        bool doctest_ok_ = false;                                                                          \
        try {                                                                                              \
            static_cast<void>(expr);                                                                       \
        } catch (const __VA_ARGS__&) {                                                                     \
            doctest_ok_ = true;                                                                            \
        } catch (...) {                                                                                    \
        }                                                                                                  \
        ::doctest::shim::check(doctest_ok_, __FILE__, __LINE__, "THROWS_AS(" #expr ", " #__VA_ARGS__ ")", false); \
    } while (0)
#define FAIL(msg)                                                       \
    do {                                                                \
        ::doctest::shim::report(__FILE__, __LINE__, std::string(msg).c_str()); \
        throw ::doctest::shim::Abort{};                                 \
    } while (0)
#define CAPTURE(x) ((void)0)
#define MESSAGE(x) ((void)0)
#define INFO(x) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    using namespace doctest::shim;
    int cases = 0, failed_cases = 0;
    for (const auto& c : registry()) {
        ++cases;
        bool failed = false;
        for (int target = 0;; ++target) {  // one pass per flat subcase (doctest semantics)
            st().target = target;
            st().seen = 0;
            st().case_failed = false;
            try {
                c.fn();
            } catch (const Abort&) {
            } catch (const std::exception& e) {
                report(c.file, c.line, (std::string("unexpected exception: ") + e.what()).c_str());
            }
            failed = failed || st().case_failed;
            if (st().seen <= target + 1) break;
        }
        if (failed) {
            ++failed_cases;
            std::printf("TEST CASE FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases, failed_cases);
    std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", st().checks,
                st().checks - st().failed_checks, st().failed_checks);
    return failed_cases ? 1 : 0;
}
#endif
