// oracle/ref_shim/doctest.h -- TEST INFRASTRUCTURE ONLY.
// A minimal stand-in for the doctest macros the reference's unit tests use
// (TEST_CASE, SUBCASE, CHECK*, REQUIRE*, CAPTURE, doctest::Approx), so that
// /root/reference/proj/tests/test_*.cpp compile unmodified into
// oracle/_ref/ref_unit_tests (doctest itself is not vendored).
// Command line: -tc=<glob> / -tce=<glob> (comma-separated, '*' wildcard),
// -ltc lists the test cases. Exit code 0 iff every executed check passed.
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
    explicit Approx(double value)
        : value_(value), epsilon_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0) {}
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) {
        // doctest: |lhs - v| < eps * (scale + max(|lhs|, |v|))
        return std::fabs(lhs - rhs.value_) < rhs.epsilon_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return operator==(rhs, lhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !operator==(lhs, rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !operator==(rhs, lhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }

private:
    double value_, epsilon_, scale_;
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
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct RequireFailed {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline long& assertions() {
    static long a = 0;
    return a;
}
inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++assertions();
    if (ok) return;
    ++failures();
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}
inline bool glob(const char* p, const char* s) {
    if (*p == 0) return *s == 0;
    if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
    return *p == *s && glob(p + 1, s + 1);
}
inline bool any_glob(const std::string& list, const char* name) {
    size_t start = 0;
    while (start <= list.size()) {
        size_t end = list.find(',', start);
        if (end == std::string::npos) end = list.size();
        if (glob(list.substr(start, end - start).c_str(), name)) return true;
        start = end + 1;
    }
    return false;
}

inline int run(int argc, char** argv) {
    std::string include, exclude;
    bool list = false;
    for (int i = 1; i < argc; ++i) {
        if (!std::strncmp(argv[i], "-tc=", 4)) include = argv[i] + 4;
        else if (!std::strncmp(argv[i], "-tce=", 5)) exclude = argv[i] + 5;
        else if (!std::strcmp(argv[i], "-ltc")) list = true;
    }
    int run_cases = 0, failed_cases = 0, skipped = 0;
    for (const auto& tc : registry()) {
        if ((!include.empty() && !any_glob(include, tc.name)) || (!exclude.empty() && any_glob(exclude, tc.name))) {
            ++skipped;
            continue;
        }
        if (list) {
            std::printf("%s\n", tc.name);
            continue;
        }
        const int before = failures();
        ++run_cases;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::fprintf(stderr, "%s:%d: TEST CASE threw: %s\n", tc.file, tc.line, e.what());
        } catch (...) {
            ++failures();
            std::fprintf(stderr, "%s:%d: TEST CASE threw an unknown exception\n", tc.file, tc.line);
        }
        if (failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED test case: %s\n", tc.name);
        }
    }
    if (!list)
        std::printf("[doctest-shim] test cases: %d run, %d failed, %d skipped; assertions: %ld, failed: %d\n", run_cases,
                    failed_cases, skipped, assertions(), failures());
    return failures() == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fname, name)                                                                   \
    static void fname();                                                                                      \
    static ::doctest::detail::Registrar DOCTEST_CAT(fname, _reg)(name, __FILE__, __LINE__, &fname);          \
    static void fname()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_anon_tc_, __COUNTER__), name)
#define SUBCASE(name) if (true)
#define CAPTURE(x) ((void)0)
#define INFO(...) ((void)0)
#define MESSAGE(...) ((void)0)

#define DOCTEST_CHECK_IMPL(kind, cond, expr, fatal)                                       \
    do {                                                                                  \
        bool doctest_ok_ = false;                                                         \
        try {                                                                             \
            doctest_ok_ = static_cast<bool>(cond);                                        \
        } catch (...) {                                                                   \
            doctest_ok_ = false;                                                          \
        }                                                                                 \
        ::doctest::detail::report(doctest_ok_, kind, expr, __FILE__, __LINE__);          \
        if (fatal && !doctest_ok_) throw ::doctest::detail::RequireFailed{};              \
    } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL("CHECK", (__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL("CHECK_FALSE", !(__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL("REQUIRE", (__VA_ARGS__), #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL("REQUIRE_FALSE", !(__VA_ARGS__), #__VA_ARGS__, true)
#define CHECK_EQ(a, b) CHECK((a) == (b))
#define REQUIRE_EQ(a, b) REQUIRE((a) == (b))

#define DOCTEST_THROWS_AS_IMPL(kind, expr, type, fatal)                                  \
    do {                                                                                 \
        bool doctest_ok_ = false;                                                        \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (const type&) {                                                          \
            doctest_ok_ = true;                                                          \
        } catch (...) {                                                                  \
        }                                                                                \
        ::doctest::detail::report(doctest_ok_, kind, #expr " throws " #type, __FILE__, __LINE__); \
        if (fatal && !doctest_ok_) throw ::doctest::detail::RequireFailed{};             \
    } while (0)
#define CHECK_THROWS_AS(expr, ...) DOCTEST_THROWS_AS_IMPL("CHECK_THROWS_AS", expr, __VA_ARGS__, false)
#define REQUIRE_THROWS_AS(expr, ...) DOCTEST_THROWS_AS_IMPL("REQUIRE_THROWS_AS", expr, __VA_ARGS__, true)
#define CHECK_THROWS(expr)                                                               \
    do {                                                                                 \
        bool doctest_ok_ = false;                                                        \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (...) {                                                                  \
            doctest_ok_ = true;                                                          \
        }                                                                                \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS", #expr, __FILE__, __LINE__); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                              \
    do {                                                                                 \
        bool doctest_ok_ = true;                                                         \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (...) {                                                                  \
            doctest_ok_ = false;                                                         \
        }                                                                                \
        ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
