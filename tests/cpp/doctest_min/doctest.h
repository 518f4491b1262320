// Minimal doctest-compatible harness (TEST INFRASTRUCTURE): just the macros
// the reference's unit tests use -- TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, doctest::Approx(...).epsilon(...) -- so that
// /root/reference/proj/tests/test_*.cpp can be compiled unmodified against
// the B200 drop-in (tests/cpp/Makefile).  Written for this repo.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Registry {
    struct Case {
        const char* name;
        const char* file;
        int line;
        void (*fn)();
    };
    std::vector<Case> cases;
    int failed_checks = 0, passed_checks = 0;
    bool case_failed = false;
    static Registry& get() {
        static Registry r;
        return r;
    }
};

struct Register {
    Register(const char* name, const char* file, int line, void (*fn)()) {
        Registry::get().cases.push_back({name, file, line, fn});
    }
};

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    Registry& r = Registry::get();
    if (ok) {
        ++r.passed_checks;
        return;
    }
    ++r.failed_checks;
    r.case_failed = true;
    std::printf("  %s:%d: %s( %s ) FAILED\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw RequireFailed{};
}

class Approx {
  public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) {
        const double scale = std::max(std::fabs(lhs), std::fabs(rhs.value_));
        return std::fabs(lhs - rhs.value_) <= rhs.eps_ * (1.0 + scale);
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

  private:
    double value_;
    double eps_ = 1.1920929e-7f * 100;
};

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                              \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                                \
    static doctest::Register DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__,           \
                                                                 &DOCTEST_CAT(doctest_fn_, __LINE__)); \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                            \
    do {                                                                                      \
        bool doctest_ok_ = false;                                                             \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const __VA_ARGS__&) {                                                        \
            doctest_ok_ = true;                                                               \
        } catch (...) {                                                                       \
        }                                                                                     \
        doctest::report(doctest_ok_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS(expr)                                                             \
    do {                                                                               \
        bool doctest_ok_ = false;                                                      \
        try {                                                                          \
            (void)(expr);                                                              \
        } catch (...) {                                                                \
            doctest_ok_ = true;                                                        \
        }                                                                              \
        doctest::report(doctest_ok_, #expr " throws", __FILE__, __LINE__, false);       \
    } while (0)
#define CHECK_NOTHROW(expr)                                                              \
    do {                                                                                 \
        bool doctest_ok_ = true;                                                         \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (...) {                                                                  \
            doctest_ok_ = false;                                                         \
        }                                                                                \
        doctest::report(doctest_ok_, #expr " does not throw", __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    doctest::Registry& r = doctest::Registry::get();
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int failed_cases = 0, run = 0;
    for (const auto& c : r.cases) {
        if (filter && !std::strstr(c.name, filter)) continue;
        ++run;
        r.case_failed = false;
        try {
            c.fn();
        } catch (const doctest::RequireFailed&) {
        } catch (const std::exception& e) {
            std::printf("  %s:%d: unexpected exception: %s\n", c.file, c.line, e.what());
            r.case_failed = true;
        }
        if (r.case_failed) {
            ++failed_cases;
            std::printf("FAILED TEST CASE: %s (%s:%d)\n", c.name, c.file, c.line);
        }
    }
    std::printf("[doctest-min] test cases: %d | %d passed | %d failed; checks: %d passed | %d failed\n", run,
                run - failed_cases, failed_cases, r.passed_checks, r.failed_checks);
    return failed_cases == 0 ? 0 : 1;
}
#endif
