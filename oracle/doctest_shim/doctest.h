// TEST INFRASTRUCTURE ONLY.  A minimal doctest-compatible header, so the reference's own unit
// tests (/root/reference/proj/tests/*.cpp, which include <doctest.h> from the absent vendor/
// tree, proj/CMakeLists.txt:5) compile unchanged.  Supports what those files use: TEST_CASE,
// SUBCASE (one subcase per run of its test case, as doctest does), CHECK / REQUIRE,
// CHECK_THROWS_AS / REQUIRE_THROWS_AS, CHECK_NOTHROW, CHECK_EQ, doctest::Approx and a main().
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
namespace detail {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct State {
    int target = 0, seen = 0, failures = 0, checks = 0;
    const char* current = "";
};
inline State& st() {
    static State s;
    return s;
}
struct RequireFailed {};
inline void fail(const char* file, int line, const char* what) {
    ++st().failures;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, st().current, what);
}
inline bool enter_subcase() { return st().seen++ == st().target; }
} // namespace detail

class Approx {
  public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) <= b.eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }

  private:
    double v_;
    double eps_ = 1.192092896e-07 * 100;
};
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                                    \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                                    \
    static doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_case_, __LINE__)); \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define SUBCASE(name) if (doctest::detail::enter_subcase())
#define DOCTEST_CHECK_IMPL(expr, fatal)                                                                    \
    do {                                                                                                   \
        ++doctest::detail::st().checks;                                                                    \
        bool ok_ = false;                                                                                  \
        try {                                                                                              \
            ok_ = static_cast<bool>(expr);                                                                 \
        } catch (const std::exception& e_) {                                                               \
            doctest::detail::fail(__FILE__, __LINE__, (std::string(#expr " threw: ") + e_.what()).c_str()); \
            if (fatal) throw doctest::detail::RequireFailed{};                                            \
            break;                                                                                         \
        }                                                                                                  \
        if (!ok_) {                                                                                        \
            doctest::detail::fail(__FILE__, __LINE__, #expr);                                              \
            if (fatal) throw doctest::detail::RequireFailed{};                                            \
        }                                                                                                  \
    } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true)
#define CHECK_EQ(a, b) CHECK((a) == (b))
#define REQUIRE_EQ(a, b) REQUIRE((a) == (b))
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define DOCTEST_THROWS_AS_IMPL(expr, type, fatal)                                                         \
    do {                                                                                                   \
        ++doctest::detail::st().checks;                                                                    \
        bool right_ = false;                                                                               \
        try {                                                                                              \
            (void)(expr);                                                                                  \
        } catch (const type&) {                                                                            \
            right_ = true;                                                                                 \
        } catch (...) {                                                                                    \
        }                                                                                                  \
        if (!right_) {                                                                                     \
            doctest::detail::fail(__FILE__, __LINE__, #expr " did not throw " #type);                      \
            if (fatal) throw doctest::detail::RequireFailed{};                                            \
        }                                                                                                  \
    } while (0)
#define CHECK_THROWS_AS(expr, ...) DOCTEST_THROWS_AS_IMPL(expr, __VA_ARGS__, false)
#define REQUIRE_THROWS_AS(expr, ...) DOCTEST_THROWS_AS_IMPL(expr, __VA_ARGS__, true)
#define CHECK_THROWS(expr) DOCTEST_THROWS_AS_IMPL(expr, std::exception, false)
#define CHECK_NOTHROW(expr)                                                                                \
    do {                                                                                                   \
        ++doctest::detail::st().checks;                                                                    \
        try {                                                                                              \
            (void)(expr);                                                                                  \
        } catch (const std::exception& e_) {                                                               \
            doctest::detail::fail(__FILE__, __LINE__, (std::string(#expr " threw: ") + e_.what()).c_str()); \
        }                                                                                                  \
    } while (0)
#define MESSAGE(...) ((void)0)
#define INFO(...) ((void)0)
#define CAPTURE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    auto& S = doctest::detail::st();
    int failed_cases = 0;
    const auto& reg = doctest::detail::registry();
    for (const auto& c : reg) {
        S.current = c.name;
        const int before = S.failures;
        // one run per subcase (at least one run); a run that reaches no new subcase ends it
        for (S.target = 0;; ++S.target) {
            S.seen = 0;
            try {
                c.fn();
            } catch (const doctest::detail::RequireFailed&) {
            } catch (const std::exception& e) {
                doctest::detail::fail(__FILE__, __LINE__, (std::string("unexpected exception: ") + e.what()).c_str());
            }
            if (S.target + 1 >= S.seen) break;
        }
        if (S.failures != before) ++failed_cases;
    }
    std::printf("[doctest] test cases: %zu | %zu passed | %d failed\n[doctest] assertions: %d | %d failed\n",
                reg.size(), reg.size() - failed_cases, failed_cases, S.checks, S.failures);
    return failed_cases ? 1 : 0;
}
#endif
