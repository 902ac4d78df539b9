// Minimal Catch2-style harness (TEST_CASE / REQUIRE / REQUIRE_FALSE /
// REQUIRE_THROWS_AS) so the drop-in tests read like the reference's own
// Catch2 suites (proj/tests/*.cpp). Catch2 itself is not in this image.
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace mini {
struct Case {
    const char* name;
    std::function<void()> fn;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
struct Failure : std::exception {
    std::string what_;
    explicit Failure(std::string w) : what_(std::move(w)) {}
    const char* what() const noexcept override { return what_.c_str(); }
};
inline int run_all() {
    int failed = 0;
    for (auto& c : registry()) {
        try {
            c.fn();
            std::printf("PASS %s\n", c.name);
        } catch (const std::exception& e) {
            ++failed;
            std::printf("FAIL %s: %s\n", c.name, e.what());
        }
    }
    std::printf("%zu cases, %d failed\n", registry().size(), failed);
    return failed ? 1 : 0;
}
}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST_CASE(name)                                                     \
    static void MINI_CAT(mini_case_, __LINE__)();                           \
    static mini::Reg MINI_CAT(mini_reg_, __LINE__)(name, MINI_CAT(mini_case_, __LINE__)); \
    static void MINI_CAT(mini_case_, __LINE__)()
#define REQUIRE(expr)                                                                    \
    do {                                                                                 \
        if (!(expr)) throw mini::Failure(std::string(__FILE__ ":") + std::to_string(__LINE__) + " REQUIRE(" #expr ")"); \
    } while (0)
#define REQUIRE_FALSE(expr) REQUIRE(!(expr))
#define REQUIRE_THROWS_AS(expr, type)                                                    \
    do {                                                                                 \
        bool caught_ = false;                                                            \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (const type&) {                                                          \
            caught_ = true;                                                              \
        }                                                                                \
        if (!caught_) throw mini::Failure(std::string(__FILE__ ":") + std::to_string(__LINE__) + " expected " #type); \
    } while (0)
