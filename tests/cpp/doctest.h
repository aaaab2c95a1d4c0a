// Minimal doctest-compatible test shim (the reference's vendored doctest.h is not
// in the container).  Supports exactly the macros the reference unit tests use:
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, REQUIRE_FALSE, CHECK_THROWS_AS, CAPTURE,
// FAIL.  Used to compile the reference's own tests (/root/reference/proj/tests)
// unchanged against the B200 drop-in API (tests/cpp/Makefile).
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace shim {
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
struct Abort {};
inline long& failures() {
    static long n = 0;
    return n;
}
inline long& checks() {
    static long n = 0;
    return n;
}
inline void fail(const char* kind, const char* expr, const char* file, int line) {
    ++failures();
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}
}  // namespace shim

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)
#define TEST_CASE(name)                                                                     \
    static void SHIM_CAT(shim_case_, __LINE__)();                                             \
    static shim::Reg SHIM_CAT(shim_reg_, __LINE__)(name, __FILE__, __LINE__, &SHIM_CAT(shim_case_, __LINE__)); \
    static void SHIM_CAT(shim_case_, __LINE__)()
#define CHECK(...)                                                                      \
    do {                                                                                \
        ++shim::checks();                                                               \
        if (!(__VA_ARGS__)) shim::fail("CHECK", #__VA_ARGS__, __FILE__, __LINE__);      \
    } while (0)
#define CHECK_FALSE(...)                                                                \
    do {                                                                                \
        ++shim::checks();                                                               \
        if ((__VA_ARGS__)) shim::fail("CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define REQUIRE(...)                                                                    \
    do {                                                                                \
        ++shim::checks();                                                               \
        if (!(__VA_ARGS__)) {                                                           \
            shim::fail("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                    \
            throw shim::Abort{};                                                        \
        }                                                                               \
    } while (0)
#define REQUIRE_FALSE(...)                                                              \
    do {                                                                                \
        ++shim::checks();                                                               \
        if ((__VA_ARGS__)) {                                                            \
            shim::fail("REQUIRE_FALSE", #__VA_ARGS__, __FILE__, __LINE__);              \
            throw shim::Abort{};                                                        \
        }                                                                               \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                     \
    do {                                                                                \
        ++shim::checks();                                                               \
        bool shim_ok = false;                                                           \
        try {                                                                           \
            expr;                                                                       \
        } catch (const type&) {                                                         \
            shim_ok = true;                                                             \
        } catch (...) {                                                                 \
        }                                                                               \
        if (!shim_ok) shim::fail("CHECK_THROWS_AS", #expr, __FILE__, __LINE__);         \
    } while (0)
#define CAPTURE(x) (void)(x)
#define FAIL(msg)                                                                       \
    do {                                                                                \
        shim::fail("FAIL", msg, __FILE__, __LINE__);                                    \
        throw shim::Abort{};                                                            \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const char* only = argc > 1 ? argv[1] : nullptr;
    long cases = 0, bad_cases = 0;
    for (const shim::Case& c : shim::registry()) {
        if (only && std::string(c.name).find(only) == std::string::npos) continue;
        ++cases;
        const long before = shim::failures();
        try {
            c.fn();
        } catch (const shim::Abort&) {
        } catch (const std::exception& e) {
            ++shim::failures();
            std::fprintf(stderr, "%s:%d: unexpected exception: %s\n", c.file, c.line, e.what());
        }
        const bool ok = shim::failures() == before;
        bad_cases += !ok;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("test cases: %ld | %ld passed | %ld failed; assertions checked: %ld, failed: %ld\n", cases,
                cases - bad_cases, bad_cases, shim::checks(), shim::failures());
    return bad_cases ? 1 : 0;
}
#endif
