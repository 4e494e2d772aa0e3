// A minimal doctest-compatible test harness (our own code; the real doctest is
// not vendored in /root/reference). It implements exactly the macros the
// reference's unit tests use — TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW, FAIL — so those test files compile
// unmodified against the reference library (oracle/Makefile `unit`), pinning
// that our oracle/_ref build is the reference's own behaviour.
//
// main.cpp of the reference defines DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN before
// including this header; that translation unit gets the registry and main().
// Output: one line per failed check, then "cases N checks M failures F".
#pragma once
#include <algorithm>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest_shim {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

struct Abort {};  // thrown by REQUIRE / FAIL to leave the current test case

std::vector<Case>& registry();
long long& checks();
long long& failures();

inline int add(const Case& c) {
    registry().push_back(c);
    return 0;
}

inline void fail(const char* file, int line, const std::string& what) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
}

inline bool check(bool ok, const char* file, int line, const char* expr) {
    ++checks();
    if (!ok) fail(file, line, expr);
    return ok;
}

}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                                         \
    static void fn();                                                                      \
    static const int DOCTEST_SHIM_CAT(fn, _reg) =                                          \
        doctest_shim::add(doctest_shim::Case{name, __FILE__, __LINE__, &fn});               \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)

#define CHECK(...) doctest_shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) \
    doctest_shim::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE(...)                                                                        \
    do {                                                                                    \
        if (!doctest_shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__,       \
                                 #__VA_ARGS__))                                             \
            throw doctest_shim::Abort{};                                                    \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                          \
    do {                                                                                    \
        bool doctest_shim_ok = false;                                                       \
        try {                                                                               \
            static_cast<void>(expr);                                                        \
        } catch (const __VA_ARGS__&) {                                                      \
            doctest_shim_ok = true;                                                         \
        } catch (...) {                                                                     \
        }                                                                                   \
        doctest_shim::check(doctest_shim_ok, __FILE__, __LINE__,                            \
                            #expr " throws " #__VA_ARGS__);                                  \
    } while (0)
#define CHECK_NOTHROW(...)                                                                  \
    do {                                                                                    \
        bool doctest_shim_ok = true;                                                        \
        try {                                                                               \
            static_cast<void>(__VA_ARGS__);                                                 \
        } catch (...) {                                                                     \
            doctest_shim_ok = false;                                                        \
        }                                                                                   \
        doctest_shim::check(doctest_shim_ok, __FILE__, __LINE__, #__VA_ARGS__ " nothrow"); \
    } while (0)
#define FAIL(...)                                                                           \
    do {                                                                                    \
        std::ostringstream doctest_shim_os;                                                 \
        doctest_shim_os << __VA_ARGS__;                                                     \
        doctest_shim::fail(__FILE__, __LINE__, doctest_shim_os.str());                      \
        throw doctest_shim::Abort{};                                                        \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
namespace doctest_shim {
std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
long long& checks() {
    static long long c = 0;
    return c;
}
long long& failures() {
    static long long f = 0;
    return f;
}
}  // namespace doctest_shim

int main(int argc, char** argv) {
    // optional filter: run only cases whose name contains argv[1]
    const std::string filter = argc > 1 ? argv[1] : "";
    long long cases = 0, failed_cases = 0;
    for (const auto& c : doctest_shim::registry()) {
        if (!filter.empty() && std::string(c.name).find(filter) == std::string::npos) continue;
        ++cases;
        const long long before = doctest_shim::failures();
        try {
            c.fn();
        } catch (const doctest_shim::Abort&) {
        } catch (const std::exception& e) {
            doctest_shim::fail(c.file, c.line, std::string("unexpected exception: ") + e.what());
        } catch (...) {
            doctest_shim::fail(c.file, c.line, "unexpected exception");
        }
        if (doctest_shim::failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "  in TEST_CASE \"%s\" (%s:%d)\n", c.name, c.file, c.line);
        }
    }
    std::printf("cases %lld checks %lld failures %lld failed_cases %lld\n", cases,
                doctest_shim::checks(), doctest_shim::failures(), failed_cases);
    return doctest_shim::failures() == 0 ? 0 : 1;
}
#endif
