// A minimal test runner with doctest-style macros (TEST_CASE / CHECK /
// REQUIRE / CHECK_THROWS_WITH_AS) so the drop-in's tests read like the
// reference's own suites (proj/tests/*.cpp). Written for this repo.
#pragma once
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

namespace mini {
struct Case {
    const char* name;
    bool gpu;
    std::function<void()> fn;
};
inline std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
inline int& failures() {
    static int f = 0;
    return f;
}
struct Reg {
    Reg(const char* n, bool gpu, std::function<void()> f) { cases().push_back({n, gpu, std::move(f)}); }
};
struct Abort {};
inline int run(int argc, char** argv) {
    bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu") == 0;
    int ran = 0;
    for (auto& c : cases()) {
        if (cpu_only && c.gpu) continue;
        const int before = failures();
        try {
            c.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            ++failures();
            std::printf("  unexpected exception: %s\n", e.what());
        }
        ++ran;
        std::printf("[%s] %s\n", failures() == before ? "ok" : "FAIL", c.name);
    }
    std::printf("%d test cases, %d failed checks\n", ran, failures());
    return failures() == 0 ? 0 : 1;
}
}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define MINI_CASE(name, gpu)                                                               \
    static void MINI_CAT(mini_fn_, __LINE__)();                                            \
    static mini::Reg MINI_CAT(mini_reg_, __LINE__)(name, gpu, MINI_CAT(mini_fn_, __LINE__)); \
    static void MINI_CAT(mini_fn_, __LINE__)()
#define TEST_CASE(name) MINI_CASE(name, false)
#define GPU_TEST_CASE(name) MINI_CASE(name, true)
#define CHECK(expr)                                                                    \
    do {                                                                               \
        if (!(expr)) {                                                                 \
            ++mini::failures();                                                        \
            std::printf("  %s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #expr);     \
        }                                                                              \
    } while (0)
#define CHECK_FALSE(expr) CHECK(!(expr))
#define REQUIRE(expr)                                                                  \
    do {                                                                               \
        if (!(expr)) {                                                                 \
            ++mini::failures();                                                        \
            std::printf("  %s:%d: REQUIRE(%s) failed\n", __FILE__, __LINE__, #expr);   \
            throw mini::Abort{};                                                       \
        }                                                                              \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, type)                                              \
    do {                                                                                   \
        bool ok_ = false;                                                                  \
        try {                                                                              \
            (void)(expr);                                                                  \
        } catch (const type& e_) {                                                         \
            ok_ = std::string(e_.what()) == std::string(msg);                              \
            if (!ok_) std::printf("  got message: %s\n", e_.what());                       \
        } catch (...) {                                                                    \
        }                                                                                  \
        if (!ok_) {                                                                        \
            ++mini::failures();                                                            \
            std::printf("  %s:%d: expected %s(\"%s\")\n", __FILE__, __LINE__, #type, msg); \
        }                                                                                  \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                        \
    do {                                                                                   \
        bool ok_ = false;                                                                  \
        try {                                                                              \
            (void)(expr);                                                                  \
        } catch (const type&) {                                                            \
            ok_ = true;                                                                    \
        } catch (...) {                                                                    \
        }                                                                                  \
        if (!ok_) {                                                                        \
            ++mini::failures();                                                            \
            std::printf("  %s:%d: expected %s\n", __FILE__, __LINE__, #type);             \
        }                                                                                  \
    } while (0)
