// Minimal doctest-compatible shim (doctest itself is not in the image; the
// reference's vendor/ directory was excluded from the snapshot). Supports the
// subset the reference tests use: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS, CHECK_NOTHROW. Every failed assertion prints
// "FAILED <file>:<line>: <expr>" so a harness can tell which checks failed.
// Test infrastructure only: used to build oracle/_ref.
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest_shim {
struct Case { const char* name; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline int& failures() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }
struct Abort {};
struct Reg { Reg(const char* n, void (*f)()) { registry().push_back({n, f}); } };
inline void fail(const char* file, int line, const char* expr) {
    failures()++;
    std::printf("FAILED %s:%d: %s\n", file, line, expr);
}
}  // namespace doctest_shim

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define DS_TC_IMPL(fn, name)                                              \
    static void fn();                                                     \
    static doctest_shim::Reg DS_CAT(fn, _reg)(name, &fn);                 \
    static void fn()
#define TEST_CASE(name) DS_TC_IMPL(DS_CAT(ds_test_, __COUNTER__), name)

#define DS_CHECK_IMPL(expr, hard)                                         \
    do {                                                                  \
        doctest_shim::checks()++;                                         \
        bool ds_ok_ = false;                                              \
        try { ds_ok_ = static_cast<bool>(expr); } catch (...) {}          \
        if (!ds_ok_) {                                                    \
            doctest_shim::fail(__FILE__, __LINE__, #expr);                \
            if (hard) throw doctest_shim::Abort{};                        \
        }                                                                 \
    } while (0)
#define CHECK(...) DS_CHECK_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DS_CHECK_IMPL((__VA_ARGS__), true)
#define CHECK_THROWS_AS(expr, ...)                                        \
    do {                                                                  \
        doctest_shim::checks()++;                                         \
        bool ds_ok_ = false;                                              \
        try { (void)(expr); } catch (const __VA_ARGS__&) { ds_ok_ = true; } \
        catch (...) {}                                                    \
        if (!ds_ok_) doctest_shim::fail(__FILE__, __LINE__, #expr " throws " #__VA_ARGS__); \
    } while (0)
#define CHECK_THROWS(expr)                                                \
    do {                                                                  \
        doctest_shim::checks()++;                                         \
        bool ds_ok_ = false;                                              \
        try { (void)(expr); } catch (...) { ds_ok_ = true; }              \
        if (!ds_ok_) doctest_shim::fail(__FILE__, __LINE__, #expr " throws"); \
    } while (0)
#define CHECK_NOTHROW(expr)                                               \
    do {                                                                  \
        doctest_shim::checks()++;                                         \
        try { (void)(expr); } catch (...) {                               \
            doctest_shim::fail(__FILE__, __LINE__, #expr " nothrow"); }   \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int cases = 0;
    for (auto& c : doctest_shim::registry()) {
        cases++;
        try { c.fn(); }
        catch (doctest_shim::Abort&) {}
        catch (std::exception& e) {
            doctest_shim::failures()++;
            std::printf("FAILED %s: unexpected exception: %s\n", c.name, e.what());
        }
    }
    std::printf("[doctest-shim] test cases: %d | checks: %d | failed: %d\n", cases,
                doctest_shim::checks(), doctest_shim::failures());
    return doctest_shim::failures() ? 1 : 0;
}
#endif
