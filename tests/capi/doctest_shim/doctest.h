// Minimal doctest-compatible harness (TEST CODE, not product): just enough of
// doctest's surface — TEST_CASE, CHECK, REQUIRE, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN —
// to compile the reference's own C-ABI suite
// (/root/reference/proj/tests/capi/test_capi.cpp, unmodified, from where it
// lies) against this repo's libtoesplit.so.1. doctest itself is not vendored
// in the reference (proj/.gitignore: vendor/) and not installed here.
#pragma once

#include <cstdio>
#include <exception>
#include <vector>

namespace doctest_shim {

struct Case {
    const char* name;
    void (*fn)();
};

inline std::vector<Case>& registry()
{
    static std::vector<Case> r;
    return r;
}

struct Reg {
    Reg(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailed : std::exception {};

inline int& failures()
{
    static int f = 0;
    return f;
}
inline int& checks()
{
    static int c = 0;
    return c;
}

inline void report(const char* file, int line, const char* expr, bool require)
{
    ++failures();
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require)
        throw RequireFailed();
}

}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT_(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT_(a, b)
#define TEST_CASE(name)                                                                             \
    static void DOCTEST_SHIM_CAT(doctest_shim_tc_, __LINE__)();                                     \
    static ::doctest_shim::Reg DOCTEST_SHIM_CAT(doctest_shim_reg_, __LINE__)(                        \
        name, DOCTEST_SHIM_CAT(doctest_shim_tc_, __LINE__));                                        \
    static void DOCTEST_SHIM_CAT(doctest_shim_tc_, __LINE__)()
#define CHECK(...)                                                                                  \
    do {                                                                                            \
        ++::doctest_shim::checks();                                                                 \
        if (!(__VA_ARGS__))                                                                         \
            ::doctest_shim::report(__FILE__, __LINE__, #__VA_ARGS__, false);                        \
    } while (0)
#define REQUIRE(...)                                                                                \
    do {                                                                                            \
        ++::doctest_shim::checks();                                                                 \
        if (!(__VA_ARGS__))                                                                         \
            ::doctest_shim::report(__FILE__, __LINE__, #__VA_ARGS__, true);                         \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main()
{
    int failed_cases = 0;
    for (const auto& c : ::doctest_shim::registry()) {
        const int before = ::doctest_shim::failures();
        try {
            c.fn();
        } catch (const ::doctest_shim::RequireFailed&) {
        } catch (const std::exception& e) {
            ++::doctest_shim::failures();
            std::fprintf(stderr, "TEST_CASE(%s) threw: %s\n", c.name, e.what());
        }
        const bool ok = ::doctest_shim::failures() == before;
        failed_cases += !ok;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("test cases: %zu | %zu passed | %d failed; assertions: %d | %d failed\n",
                ::doctest_shim::registry().size(), ::doctest_shim::registry().size() - failed_cases,
                failed_cases, ::doctest_shim::checks(), ::doctest_shim::failures());
    return failed_cases ? 1 : 0;
}
#endif
