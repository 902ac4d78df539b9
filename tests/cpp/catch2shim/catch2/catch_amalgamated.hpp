// Catch2 shim: the subset of Catch2 v3's <catch2/catch_amalgamated.hpp> that
// the reference's unit tests use (TEST_CASE, REQUIRE, REQUIRE_FALSE,
// REQUIRE_THROWS_AS), so /root/reference/proj/tests/test_{core,join,hash}.cpp
// compile UNMODIFIED against the drop-in headers (include/hashgraph/) and run
// on the B200 (Makefile target tests/cpp/ref_tests). Catch2 itself is not in
// this image. A failed REQUIRE aborts its test case, as in
// Catch2; the runner (ref_main.cpp) reports every case and the totals.
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace catch_shim {
struct Case {
    std::string name;
    std::function<void()> fn;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(void (*fn)(), const char* name, const char* /*tags*/ = "") {
        registry().push_back({name, fn});
    }
};
struct Failure : std::exception {
    std::string msg;
    Failure(const char* file, int line, const std::string& what)
        : msg(std::string(file) + ":" + std::to_string(line) + ": " + what) {}
    const char* what() const noexcept override { return msg.c_str(); }
};
inline int run_all() {
    int failed = 0;
    for (const Case& c : registry()) {
        try {
            c.fn();
            std::printf("PASS %s\n", c.name.c_str());
        } catch (const Failure& f) {
            ++failed;
            std::printf("FAIL %s\n     %s\n", c.name.c_str(), f.what());
        } catch (const std::exception& e) {
            ++failed;
            std::printf("FAIL %s\n     unexpected exception: %s\n", c.name.c_str(), e.what());
        }
    }
    std::printf("%zu test cases, %d failed\n", registry().size(), failed);
    return failed ? 1 : 0;
}
}  // namespace catch_shim

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_FN CATCH_SHIM_CAT(catch_shim_case_, __LINE__)
#define TEST_CASE(...)                                                                  \
    static void CATCH_SHIM_FN();                                                        \
    static const catch_shim::Registrar CATCH_SHIM_CAT(catch_shim_reg_, __LINE__)(       \
        &CATCH_SHIM_FN, __VA_ARGS__);                                                   \
    static void CATCH_SHIM_FN()
#define REQUIRE(...)                                                                         \
    do {                                                                                     \
        if (!static_cast<bool>(__VA_ARGS__))                                                 \
            throw catch_shim::Failure(__FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )");   \
    } while (0)
#define REQUIRE_FALSE(...)                                                                   \
    do {                                                                                     \
        if (static_cast<bool>(__VA_ARGS__))                                                  \
            throw catch_shim::Failure(__FILE__, __LINE__, "REQUIRE_FALSE( " #__VA_ARGS__ " )"); \
    } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                                        \
    do {                                                                                     \
        bool caught_ = false;                                                                \
        try {                                                                                \
            static_cast<void>(expr);                                                         \
        } catch (const type&) {                                                              \
            caught_ = true;                                                                  \
        } catch (...) {                                                                      \
            throw catch_shim::Failure(__FILE__, __LINE__,                                    \
                                      "REQUIRE_THROWS_AS( " #expr ", " #type " ): other exception"); \
        }                                                                                    \
        if (!caught_)                                                                        \
            throw catch_shim::Failure(__FILE__, __LINE__,                                    \
                                      "REQUIRE_THROWS_AS( " #expr ", " #type " ): no exception"); \
    } while (0)
