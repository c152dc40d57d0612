// tests/shim/doctest.h -- TEST INFRASTRUCTURE.  A minimal doctest-compatible harness: exactly the macro surface the
// reference's own suites use (/root/reference/proj/tests/*_test.cpp: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS + doctest::Contains, doctest::Approx(..).epsilon(..), FAIL, CAPTURE), so that
// those files compile UNMODIFIED, from where they lie, against libwfc_b200.so.  The real doctest.h is a vendored
// third-party header the reference tree does not ship (proj/.gitignore:2).  Not a copy of doctest: registration by
// static objects, expression results by plain bool conversion (no decomposition), one summary line per binary.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct TestFailure : std::exception {};     // thrown by REQUIRE / FAIL to leave the test case

struct Case { const char* name; const char* file; int line; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
struct Registrar { Registrar(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); } };

struct State { int checks = 0, failed_checks = 0; bool case_failed = false; std::vector<std::string> captures; };
inline State& state() { static State s; return s; }

inline void report(const char* kind, const char* expr, const char* file, int line, const std::string& extra = "") {
    State& s = state();
    ++s.failed_checks;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) failed%s%s\n", file, line, kind, expr, extra.empty() ? "" : ": ", extra.c_str());
    for (const auto& c : s.captures) std::fprintf(stderr, "    with %s\n", c.c_str());
}

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    // doctest's rule: |a - b| < eps * (scale + max(|a|, |b|)), scale = 1
    bool matches(double other) const {
        return std::fabs(other - value_) < eps_ * (1.0 + std::fmax(std::fabs(other), std::fabs(value_)));
    }
    friend bool operator==(double a, const Approx& b) { return b.matches(a); }
    friend bool operator==(const Approx& b, double a) { return b.matches(a); }
    friend bool operator!=(double a, const Approx& b) { return !b.matches(a); }
    friend bool operator!=(const Approx& b, double a) { return !b.matches(a); }
    friend bool operator<=(double a, const Approx& b) { return a < b.value_ || b.matches(a); }
    friend bool operator>=(double a, const Approx& b) { return a > b.value_ || b.matches(a); }
private:
    double value_;
    double eps_ = 1.1920928955078125e-05;   // float epsilon * 100, doctest's default
};

class Contains {
public:
    explicit Contains(std::string s) : s_(std::move(s)) {}
    bool in(const std::string& hay) const { return hay.find(s_) != std::string::npos; }
    const std::string& str() const { return s_; }
private:
    std::string s_;
};
inline bool message_matches(const std::string& what, const Contains& c) { return c.in(what); }
inline bool message_matches(const std::string& what, const std::string& exact) { return what == exact; }
inline bool message_matches(const std::string& what, const char* exact) { return what == exact; }

template <typename T> std::string show(const T& v) { std::ostringstream o; o << v; return o.str(); }

struct CaptureScope {
    explicit CaptureScope(std::string s) { state().captures.push_back(std::move(s)); }
    ~CaptureScope() { state().captures.pop_back(); }
};

inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        State& s = state();
        s.case_failed = false;
        s.captures.clear();
        try {
            c.fn();
        } catch (const TestFailure&) {
        } catch (const std::exception& e) {
            report("TEST_CASE", c.name, c.file, c.line, std::string("unexpected exception: ") + e.what());
        } catch (...) {
            report("TEST_CASE", c.name, c.file, c.line, "unexpected exception");
        }
        if (s.case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED test case \"%s\" (%s:%d)\n", c.name, c.file, c.line);
        }
    }
    const State& s = state();
    std::printf("[shim] test cases: %zu | %zu passed | %d failed    assertions: %d | %d failed\n", registry().size(),
                registry().size() - failed_cases, failed_cases, s.checks, s.failed_checks);
    return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define TEST_CASE(name)                                                                             \
    static void DT_CAT(dt_case_, __LINE__)();                                                       \
    static ::doctest::Registrar DT_CAT(dt_reg_, __LINE__)(name, __FILE__, __LINE__, &DT_CAT(dt_case_, __LINE__)); \
    static void DT_CAT(dt_case_, __LINE__)()

#define DT_ASSERT(kind, fatal, negate, ...)                                                        \
    do {                                                                                            \
        ++::doctest::state().checks;                                                                \
        bool dt_ok = false;                                                                         \
        try { dt_ok = static_cast<bool>(__VA_ARGS__); if (negate) dt_ok = !dt_ok; }                 \
        catch (const ::doctest::TestFailure&) { throw; }                                            \
        catch (const std::exception& dt_e) { ::doctest::report(kind, #__VA_ARGS__, __FILE__, __LINE__, std::string("threw: ") + dt_e.what()); if (fatal) throw ::doctest::TestFailure(); break; } \
        if (!dt_ok) { ::doctest::report(kind, #__VA_ARGS__, __FILE__, __LINE__); if (fatal) throw ::doctest::TestFailure(); } \
    } while (0)
#define CHECK(...) DT_ASSERT("CHECK", false, false, __VA_ARGS__)
#define CHECK_FALSE(...) DT_ASSERT("CHECK_FALSE", false, true, __VA_ARGS__)
#define REQUIRE(...) DT_ASSERT("REQUIRE", true, false, __VA_ARGS__)

#define CHECK_THROWS_AS(expr, ...)                                                                  \
    do {                                                                                            \
        ++::doctest::state().checks;                                                                \
        bool dt_thrown = false;                                                                     \
        try { static_cast<void>(expr); }                                                            \
        catch (const typename std::remove_cv<typename std::remove_reference<__VA_ARGS__>::type>::type&) { dt_thrown = true; } \
        catch (...) { ::doctest::report("CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__, "threw a different type"); break; } \
        if (!dt_thrown) ::doctest::report("CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__, "did not throw"); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                       \
    do {                                                                                            \
        ++::doctest::state().checks;                                                                \
        bool dt_thrown = false;                                                                     \
        try { static_cast<void>(expr); }                                                            \
        catch (const typename std::remove_cv<typename std::remove_reference<__VA_ARGS__>::type>::type& dt_e) {      \
            dt_thrown = true;                                                                       \
            if (!::doctest::message_matches(dt_e.what(), with))                                     \
                ::doctest::report("CHECK_THROWS_WITH_AS", #expr ", " #with, __FILE__, __LINE__, std::string("message was: ") + dt_e.what()); \
        }                                                                                           \
        catch (...) { ::doctest::report("CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__, "threw a different type"); break; } \
        if (!dt_thrown) ::doctest::report("CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__, "did not throw"); \
    } while (0)
#define FAIL(...)                                                                                   \
    do {                                                                                            \
        std::ostringstream dt_o; dt_o << __VA_ARGS__;                                               \
        ::doctest::report("FAIL", "", __FILE__, __LINE__, dt_o.str());                             \
        throw ::doctest::TestFailure();                                                             \
    } while (0)
#define CAPTURE(x) ::doctest::CaptureScope DT_CAT(dt_cap_, __LINE__)(std::string(#x " := ") + ::doctest::show(x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
