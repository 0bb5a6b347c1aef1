// A doctest-compatible test runner (the subset the reference's unit tests use:
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, CAPTURE, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) so that
// proj/tests/*.cpp compile UNMODIFIED in this repo's recipe (doctest itself is
// not in the image). Written for this repo; test infrastructure only.
//
//   binary [-tc=<pattern>]   run the cases whose name matches (* wildcards)
#pragma once
#include <cstdio>
#include <cstring>
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
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline int& failed_asserts() {
    static int n = 0;
    return n;
}
inline int& total_asserts() {
    static int n = 0;
    return n;
}
inline std::vector<std::string>& captures() {
    static std::vector<std::string> c;
    return c;
}
struct Require {};
struct Reg {
    Reg(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
inline void fail(const char* file, int line, const std::string& what) {
    ++failed_asserts();
    std::printf("%s:%d: ERROR: %s\n", file, line, what.c_str());
    for (const auto& c : captures()) std::printf("  logged: %s\n", c.c_str());
}
inline void check(bool ok, const char* file, int line, const char* macro, const char* expr) {
    ++total_asserts();
    if (!ok) fail(file, line, std::string(macro) + "( " + expr + " ) is NOT correct!");
}
struct CaptureGuard {
    template <typename T>
    CaptureGuard(const char* name, const T& v) {
        std::ostringstream os;
        os << name << " := " << v;
        captures().push_back(os.str());
    }
    ~CaptureGuard() { captures().pop_back(); }
};
inline bool glob(const char* p, const char* s) {
    if (!*p) return !*s;
    if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
    return *s && *p == *s && glob(p + 1, s + 1);
}
inline int run(int argc, char** argv) {
    std::vector<std::string> pats;
    for (int i = 1; i < argc; ++i) {
        const char* a = argv[i];
        for (const char* pre : {"-tc=", "--test-case="})
            if (std::strncmp(a, pre, std::strlen(pre)) == 0) {
                std::string list = a + std::strlen(pre);
                size_t at = 0;
                while (at <= list.size()) {
                    size_t c = list.find(',', at);
                    if (c == std::string::npos) c = list.size();
                    pats.push_back(list.substr(at, c - at));
                    at = c + 1;
                }
            }
    }
    int cases = 0, failed_cases = 0;
    for (const auto& c : registry()) {
        if (!pats.empty()) {
            bool hit = false;
            for (const auto& p : pats) hit |= glob(p.c_str(), c.name);
            if (!hit) continue;
        }
        ++cases;
        const int before = failed_asserts();
        try {
            c.fn();
        } catch (const Require&) {
        } catch (const std::exception& e) {
            fail(c.file, c.line, std::string("unexpected exception: ") + e.what());
        } catch (...) {
            fail(c.file, c.line, "unexpected unknown exception");
        }
        captures().clear();
        if (failed_asserts() != before) {
            ++failed_cases;
            std::printf("  in TEST CASE: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases, failed_cases);
    std::printf("[doctest-shim] assertions: %d | %d failed\n", total_asserts(), failed_asserts());
    return failed_cases ? 1 : 0;
}
}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TC(fn, name)                                                                   \
    static void fn();                                                                               \
    static doctest_shim::Reg DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);             \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TC(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)

#define CHECK(...) doctest_shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__)
#define CHECK_FALSE(...) \
    doctest_shim::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__)
#define REQUIRE(...)                                                                                \
    do {                                                                                            \
        const bool doctest_shim_ok = static_cast<bool>(__VA_ARGS__);                                \
        doctest_shim::check(doctest_shim_ok, __FILE__, __LINE__, "REQUIRE", #__VA_ARGS__);          \
        if (!doctest_shim_ok) throw doctest_shim::Require{};                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                  \
    do {                                                                                            \
        bool doctest_shim_ok = false;                                                               \
        try {                                                                                       \
            (void)(expr);                                                                           \
        } catch (const __VA_ARGS__&) {                                                              \
            doctest_shim_ok = true;                                                                 \
        } catch (...) {                                                                             \
        }                                                                                           \
        doctest_shim::check(doctest_shim_ok, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr);         \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                       \
    do {                                                                                            \
        bool doctest_shim_ok = false;                                                               \
        std::string doctest_shim_what = "(nothing thrown)";                                         \
        try {                                                                                       \
            (void)(expr);                                                                           \
        } catch (const __VA_ARGS__& e) {                                                            \
            doctest_shim_what = e.what();                                                           \
            doctest_shim_ok = doctest_shim_what == std::string(with);                               \
        } catch (const std::exception& e) {                                                         \
            doctest_shim_what = std::string("other type: ") + e.what();                             \
        } catch (...) {                                                                             \
        }                                                                                           \
        doctest_shim::check(doctest_shim_ok, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS",            \
                            (std::string(#expr) + " threw \"" + doctest_shim_what + "\"").c_str()); \
    } while (0)
#define CAPTURE(x) doctest_shim::CaptureGuard DOCTEST_SHIM_CAT(doctest_shim_capture_, __COUNTER__)(#x, x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest_shim::run(argc, argv); }
#endif
