// Minimal Catch2 stand-in (test scaffolding only): the six macros the
// reference's unit tests use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, INFO), so proj/tests/test_*.cpp build unmodified against
// the drop-in headers in include/pmagraph/ (SURVEY Appendix A).
#pragma once
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace shim {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline long& checks() {
    static long c = 0;
    return c;
}
inline const char*& current() {
    static const char* c = "";
    return c;
}
inline void fail(const char* file, int line, const char* expr) {
    ++failures();
    std::fprintf(stderr, "FAILED [%s] %s:%d: %s\n", current(), file, line, expr);
}
}  // namespace shim

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)
#define SHIM_TEST(fn, name)                                   \
    static void fn();                                         \
    static shim::Reg SHIM_CAT(fn, _reg){name, &fn};           \
    static void fn()
#define TEST_CASE(name, ...) SHIM_TEST(SHIM_CAT(shim_case_, __COUNTER__), name)
#define CHECK(...)                                                          \
    do {                                                                    \
        ++shim::checks();                                                   \
        if (!(__VA_ARGS__)) shim::fail(__FILE__, __LINE__, #__VA_ARGS__);   \
    } while (0)
#define CHECK_FALSE(...)                                                    \
    do {                                                                    \
        ++shim::checks();                                                   \
        if ((__VA_ARGS__)) shim::fail(__FILE__, __LINE__, "!(" #__VA_ARGS__ ")"); \
    } while (0)
#define REQUIRE(...)                                                        \
    do {                                                                    \
        ++shim::checks();                                                   \
        if (!(__VA_ARGS__)) {                                               \
            shim::fail(__FILE__, __LINE__, #__VA_ARGS__);                   \
            throw shim::RequireFailed{};                                    \
        }                                                                   \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                         \
    do {                                                                    \
        ++shim::checks();                                                   \
        bool shim_caught_ = false;                                          \
        try {                                                               \
            (void)(expr);                                                   \
        } catch (const type&) {                                             \
            shim_caught_ = true;                                            \
        } catch (...) {                                                     \
        }                                                                   \
        if (!shim_caught_) shim::fail(__FILE__, __LINE__, "throws " #type ": " #expr); \
    } while (0)
#define INFO(...)                          \
    do {                                   \
        std::ostringstream shim_info_;     \
        shim_info_ << __VA_ARGS__;         \
    } while (0)
