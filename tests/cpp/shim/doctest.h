// Minimal stand-in for the doctest macros the reference's test suites use
// (TEST_SUITE, TEST_CASE, CHECK, CHECK_FALSE, CHECK_THROWS_AS, REQUIRE):
// doctest itself is not in this image.  Test cases register
// themselves; the driver calls doctest_shim::run_all().
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest_shim {
struct Case {
    const char* name;
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
inline int& checks() {
    static int c = 0;
    return c;
}
struct Reg {
    Reg(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    ++checks();
    if (ok) return;
    ++failures();
    std::printf("  FAIL %s:%d: %s\n", file, line, expr);
    if (fatal) throw RequireFailed{};
}
inline int run_all() {
    int failed_cases = 0;
    for (const auto& c : registry()) {
        const int before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::printf("  FAIL unexpected exception: %s\n", e.what());
        }
        const bool ok = failures() == before;
        failed_cases += !ok;
        std::printf("%s %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("%zu test cases, %d checks, %d failed cases\n", registry().size(), checks(), failed_cases);
    return failed_cases;
}
}  // namespace doctest_shim

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define TEST_SUITE(name) namespace
#define TEST_CASE(name)                                                                  \
    static void DS_CAT(ds_case_, __LINE__)();                                           \
    static ::doctest_shim::Reg DS_CAT(ds_reg_, __LINE__)(name, &DS_CAT(ds_case_, __LINE__)); \
    static void DS_CAT(ds_case_, __LINE__)()
#define CHECK(...) ::doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest_shim::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                            \
    do {                                                                                       \
        bool ds_ok = false;                                                                    \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (const type&) {                                                                \
            ds_ok = true;                                                                      \
        } catch (...) {                                                                        \
        }                                                                                      \
        ::doctest_shim::report(ds_ok, #expr " throws " #type, __FILE__, __LINE__, false);     \
    } while (0)
