// TEST INFRASTRUCTURE ONLY (oracle/): the doctest subset the reference's tests use
// (proj/tests/test_grid.cpp, test_camera.cpp): TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, FAIL, doctest::Approx(+epsilon). vendor/doctest is git-ignored
// upstream (proj/.gitignore:2) and absent here, so the tests compile against this.
// Approx follows doctest's documented rule:
//   |lhs - v| < eps * (scale + max(|lhs|, |v|)), eps default = 100 * FLT_EPSILON.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v)
        : value_(v), eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100),
          scale_(1.0) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) <
               a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

private:
    double value_, eps_, scale_;
};

namespace detail {

struct RequireAbort {};

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
inline int& failures() {
    static int f = 0;
    return f;
}
inline long& assertions() {
    static long a = 0;
    return a;
}
inline const char*& current() {
    static const char* c = "";
    return c;
}
inline bool reg(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
    return true;
}
inline void fail(const char* what, const char* file, int line) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, current(), what);
}

inline int run_all(int argc, char** argv) {
    const char* filter = nullptr;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
    int cases = 0, failed_cases = 0;
    for (const Case& c : registry()) {
        if (filter && !std::strstr(c.name, filter)) continue;
        ++cases;
        current() = c.name;
        const int before = failures();
        try {
            c.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            fail((std::string("unexpected exception: ") + e.what()).c_str(), c.file, c.line);
        } catch (...) {
            fail("unexpected unknown exception", c.file, c.line);
        }
        if (failures() != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | "
                "failed assertions: %d\n",
                cases, cases - failed_cases, failed_cases, assertions(), failures());
    return failures() == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                        \
    static void fn();                                                                    \
    static const bool DOCTEST_CAT(fn, _reg) = doctest::detail::reg(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...)                                                         \
    do {                                                                   \
        ++doctest::detail::assertions();                                   \
        if (!(__VA_ARGS__)) doctest::detail::fail(#__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define REQUIRE(...)                                                       \
    do {                                                                   \
        ++doctest::detail::assertions();                                   \
        if (!(__VA_ARGS__)) {                                              \
            doctest::detail::fail(#__VA_ARGS__, __FILE__, __LINE__);       \
            throw doctest::detail::RequireAbort{};                         \
        }                                                                  \
    } while (0)
#define FAIL(msg)                                                          \
    do {                                                                   \
        doctest::detail::fail(msg, __FILE__, __LINE__);                    \
        throw doctest::detail::RequireAbort{};                             \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                         \
    do {                                                                   \
        ++doctest::detail::assertions();                                   \
        bool thrown_ok = false;                                            \
        try {                                                              \
            (void)(expr);                                                  \
        } catch (const __VA_ARGS__&) {                                     \
            thrown_ok = true;                                              \
        } catch (...) {                                                    \
        }                                                                  \
        if (!thrown_ok)                                                    \
            doctest::detail::fail("CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")", __FILE__, \
                                  __LINE__);                               \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc, argv); }
#endif
