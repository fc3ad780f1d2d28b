// doctest.h -- a minimal stand-in for the doctest framework, enough to
// compile the reference's own test files (proj/tests/*.cpp) unchanged
// against the B200 library through include/autosage_b200_compat.hpp.
// The reference vendors no doctest.h (proj/.gitignore); this shim covers the
// macros those files use: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// REQUIRE_FALSE, REQUIRE_MESSAGE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// doctest::Approx(..).epsilon(..), doctest::Contains.
//
// Output: one line per failed check, then
//   [doctest] test cases: N | passed: P | failed: F
//   [doctest] assertions: A | passed: AP | failed: AF
// and exit status 1 when anything failed.
#pragma once

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
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& r) { return r.match(lhs); }
    friend bool operator==(const Approx& r, double rhs) { return r.match(rhs); }
    friend bool operator!=(double lhs, const Approx& r) { return !r.match(lhs); }
    friend bool operator!=(const Approx& r, double rhs) { return !r.match(rhs); }

private:
    // doctest's rule: |a - b| < eps * (scale + max(|a|, |b|)), scale 1, eps
    // defaulting to float epsilon * 100
    bool match(double other) const {
        return std::fabs(other - value_) < eps_ * (1.0 + std::fmax(std::fabs(other), std::fabs(value_)));
    }
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;
};

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    std::string needle;
    bool check(const std::string& text) const { return text.find(needle) != std::string::npos; }
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

struct Stats {
    int asserts = 0, failed_asserts = 0;
    bool current_failed = false;
};

inline Stats& stats() {
    static Stats s;
    return s;
}

struct Register {
    Register(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

// a failed REQUIRE ends the test case
struct RequireFailed {};

inline void record(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& extra = std::string()) {
    Stats& s = stats();
    ++s.asserts;
    if (ok) return;
    ++s.failed_asserts;
    s.current_failed = true;
    std::printf("%s:%d: ERROR: %s( %s ) failed%s%s\n", file, line, kind, expr, extra.empty() ? "" : ": ",
                extra.c_str());
}

inline bool matches(const std::string& what, const char* m) { return what == m; }
inline bool matches(const std::string& what, const std::string& m) { return what == m; }
inline bool matches(const std::string& what, const Contains& c) { return c.check(what); }

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define DOCTEST_TEST_CASE_IMPL(fn, reg, name)                                          \
    static void fn();                                                                  \
    static ::doctest::detail::Register reg(name, __FILE__, __LINE__, &fn);             \
    static void fn()

#define TEST_CASE(name) \
    DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), DOCTEST_CAT(doctest_reg_, __LINE__), name)

#define DOCTEST_EVAL(kind, expr, want, fatal)                                                         \
    do {                                                                                              \
        bool doctest_ok_ = false;                                                                     \
        std::string doctest_extra_;                                                                   \
        try {                                                                                         \
            doctest_ok_ = static_cast<bool>(expr) == (want);                                          \
        } catch (const std::exception& e) {                                                           \
            doctest_extra_ = std::string("threw ") + e.what();                                        \
        } catch (...) {                                                                               \
            doctest_extra_ = "threw an unknown exception";                                            \
        }                                                                                             \
        ::doctest::detail::record(doctest_ok_, kind, #expr, __FILE__, __LINE__, doctest_extra_);       \
        if (!doctest_ok_ && (fatal)) throw ::doctest::detail::RequireFailed{};                        \
    } while (0)

#define CHECK(...) DOCTEST_EVAL("CHECK", (__VA_ARGS__), true, false)
#define CHECK_FALSE(...) DOCTEST_EVAL("CHECK_FALSE", (__VA_ARGS__), false, false)
#define REQUIRE(...) DOCTEST_EVAL("REQUIRE", (__VA_ARGS__), true, true)
#define REQUIRE_FALSE(...) DOCTEST_EVAL("REQUIRE_FALSE", (__VA_ARGS__), false, true)
#define REQUIRE_MESSAGE(cond, msg)                                                                    \
    do {                                                                                              \
        const bool doctest_ok_ = static_cast<bool>(cond);                                            \
        ::doctest::detail::record(doctest_ok_, "REQUIRE_MESSAGE", #cond, __FILE__, __LINE__,          \
                                  doctest_ok_ ? std::string() : std::string(msg));                    \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                                   \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                                    \
    do {                                                                                              \
        bool doctest_ok_ = false;                                                                     \
        std::string doctest_extra_ = "did not throw";                                                 \
        try {                                                                                         \
            static_cast<void>(expr);                                                                  \
        } catch (const __VA_ARGS__&) {                                                                \
            doctest_ok_ = true;                                                                       \
        } catch (const std::exception& e) {                                                           \
            doctest_extra_ = std::string("threw another type: ") + e.what();                          \
        } catch (...) {                                                                               \
            doctest_extra_ = "threw an unknown type";                                                 \
        }                                                                                             \
        ::doctest::detail::record(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__,          \
                                  doctest_ok_ ? std::string() : doctest_extra_);                      \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                         \
    do {                                                                                              \
        bool doctest_ok_ = false;                                                                     \
        std::string doctest_extra_ = "did not throw";                                                 \
        try {                                                                                         \
            static_cast<void>(expr);                                                                  \
        } catch (const __VA_ARGS__& e) {                                                              \
            doctest_ok_ = ::doctest::detail::matches(e.what(), with);                                 \
            if (!doctest_ok_) doctest_extra_ = std::string("message: ") + e.what();                   \
        } catch (const std::exception& e) {                                                           \
            doctest_extra_ = std::string("threw another type: ") + e.what();                          \
        } catch (...) {                                                                               \
            doctest_extra_ = "threw an unknown type";                                                 \
        }                                                                                             \
        ::doctest::detail::record(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__,     \
                                  doctest_ok_ ? std::string() : doctest_extra_);                      \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const char* only = nullptr;  // --tc=<substring>: run matching cases only
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "--tc=", 5) == 0) only = argv[i] + 5;
    int cases = 0, failed_cases = 0;
    for (const auto& tc : ::doctest::detail::registry()) {
        if (only && !std::strstr(tc.name, only)) continue;
        ++cases;
        auto& s = ::doctest::detail::stats();
        s.current_failed = false;
        try {
            tc.fn();
        } catch (const ::doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            std::printf("%s:%d: ERROR: test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
            s.current_failed = true;
        } catch (...) {
            std::printf("%s:%d: ERROR: test case \"%s\" threw an unknown exception\n", tc.file, tc.line, tc.name);
            s.current_failed = true;
        }
        if (s.current_failed) {
            ++failed_cases;
            std::printf("  ^ in TEST_CASE \"%s\"\n", tc.name);
        }
    }
    const auto& s = ::doctest::detail::stats();
    std::printf("[doctest] test cases: %d | passed: %d | failed: %d\n", cases, cases - failed_cases,
                failed_cases);
    std::printf("[doctest] assertions: %d | passed: %d | failed: %d\n", s.asserts, s.asserts - s.failed_asserts,
                s.failed_asserts);
    return failed_cases ? 1 : 0;
}
#endif
