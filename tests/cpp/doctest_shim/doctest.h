// doctest.h — a minimal stand-in for the doctest subset the reference's tests
// use (TEST_CASE, nested SUBCASE with re-run semantics, CHECK, CHECK_FALSE,
// REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, doctest::Approx(.epsilon)), so that
// /root/reference/proj/tests/test_routing.cpp compiles UNMODIFIED (doctest
// itself lives in the reference's git-ignored vendor/ and is absent here).
// TEST INFRASTRUCTURE; written from doctest's documented behaviour:
//  * a test case body runs once per leaf subcase path: every run enters the
//    first not-yet-finished subcase at each nesting level, code outside
//    subcases runs every time;
//  * Approx(v) == x  iff  |x - v| < eps * (scale + max(|x|, |v|)), default
//    eps = 100 * FLT_EPSILON, scale = 1.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double x, const Approx& a) {
        return std::fabs(x - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(x), std::fabs(a.v_)));
    }
    friend bool operator==(const Approx& a, double x) { return x == a; }
    friend bool operator!=(double x, const Approx& a) { return !(x == a); }
    friend bool operator!=(const Approx& a, double x) { return !(x == a); }

private:
    double v_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double scale_ = 1.0;
};

namespace detail {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireFailed {};

struct State {
    long checks = 0, failures = 0;
    const char* test = "";
    // subcase traversal
    std::set<std::string> done;          // finished subcase paths
    std::vector<std::string> path;       // subcases entered in this run
    std::vector<bool> entered;           // per depth: a subcase was entered this run
    std::vector<bool> pending;           // per depth: an unfinished sibling/child remains
};
inline State& st() {
    static State s;
    return s;
}

inline std::string join(const std::vector<std::string>& p) {
    std::string s;
    for (const auto& x : p) s += "/" + x;
    return s;
}

class Subcase {
public:
    Subcase(const char* name, int line) {
        State& s = st();
        const size_t depth = s.path.size();
        if (s.entered.size() <= depth) {
            s.entered.resize(depth + 1, false);
            s.pending.resize(depth + 1, false);
        }
        key_ = join(s.path) + "/" + name + ":" + std::to_string(line);
        if (s.done.count(key_)) return;
        if (s.entered[depth]) {  // a sibling ran this time: come back in a later run
            s.pending[depth] = true;
            return;
        }
        s.entered[depth] = true;
        s.path.push_back(std::string(name) + ":" + std::to_string(line));
        if (s.entered.size() <= depth + 1) {
            s.entered.resize(depth + 2, false);
            s.pending.resize(depth + 2, false);
        }
        s.entered[depth + 1] = false;
        s.pending[depth + 1] = false;
        active_ = true;
    }
    ~Subcase() {
        if (!active_) return;
        State& s = st();
        const size_t depth = s.path.size();  // our children's depth
        if (!s.pending[depth]) s.done.insert(key_);   // no unfinished children left
        else s.pending[depth - 1] = true;             // run again to reach them
        s.path.pop_back();
    }
    explicit operator bool() const { return active_; }

private:
    std::string key_;
    bool active_ = false;
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    State& s = st();
    ++s.checks;
    if (ok) return;
    ++s.failures;
    std::printf("%s:%d: FAILED %s( %s ) in TEST_CASE \"%s\" %s\n", file, line, kind, expr, s.test,
                join(s.path).c_str());
}

inline int run_all() {
    int failed_cases = 0;
    for (const TestCase& tc : registry()) {
        State& s = st();
        const long f0 = s.failures;
        s.test = tc.name;
        s.done.clear();
        for (int run = 0; run < 100000; ++run) {
            s.path.clear();
            s.entered.assign(1, false);
            s.pending.assign(1, false);
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++s.failures;
                std::printf("%s:%d: EXCEPTION in TEST_CASE \"%s\" %s: %s\n", tc.file, tc.line, tc.name,
                            join(s.path).c_str(), e.what());
            }
            if (!s.pending[0]) break;
        }
        const bool ok = s.failures == f0;
        failed_cases += !ok;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", tc.name);
    }
    State& s = st();
    std::printf("[doctest-shim] test cases: %zu | failed: %d | assertions: %ld | failed: %ld\n",
                registry().size(), failed_cases, s.checks, s.failures);
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                         \
    static void DOCTEST_CAT(doctest_tc_, __LINE__)();                                           \
    static doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                      \
        name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_tc_, __LINE__));                         \
    static void DOCTEST_CAT(doctest_tc_, __LINE__)()
#define SUBCASE(name) if (doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name, __LINE__})
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                   \
    do {                                                                                               \
        const bool doctest_ok = static_cast<bool>(__VA_ARGS__);                                        \
        doctest::detail::report(doctest_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);              \
        if (!doctest_ok) throw doctest::detail::RequireFailed{};                                       \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                     \
    do {                                                                                               \
        bool doctest_ok = false;                                                                       \
        try {                                                                                          \
            expr;                                                                                      \
        } catch (const __VA_ARGS__&) {                                                                 \
            doctest_ok = true;                                                                         \
        } catch (...) {                                                                                \
        }                                                                                              \
        doctest::detail::report(doctest_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define CHECK_NOTHROW(...)                                                                             \
    do {                                                                                               \
        bool doctest_ok = true;                                                                        \
        try {                                                                                          \
            __VA_ARGS__;                                                                               \
        } catch (...) {                                                                                \
            doctest_ok = false;                                                                        \
        }                                                                                              \
        doctest::detail::report(doctest_ok, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__);        \
    } while (0)

// diagnostics context: accepted, not recorded
#define INFO(...) ((void)0)
#define CAPTURE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
