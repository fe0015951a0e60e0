// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE; written for this repo).
//
// The reference's unit suites (proj/tests/unit/*.cpp) include <doctest.h>, which is not vendored
// in the reference tree. This shim implements the subset they use — TEST_SUITE / TEST_CASE /
// SUBCASE (re-run-per-leaf semantics), CHECK / CHECK_FALSE / REQUIRE / CHECK_THROWS_AS /
// CHECK_NOTHROW / CHECK_THROWS_WITH_AS + doctest::Contains, FAIL, CAPTURE, doctest::Approx — so
// those unchanged sources can be compiled against the B200 build's include/tablekv headers and
// libtkv.so (oracle/Makefile target `dropin`). Main: `-ts=<suite>` filter, exit status = failures.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest_shim {

struct Test {
    void (*fn)();
    const char* name;
    const char* suite;
    const char* file;
    int line;
};

inline std::vector<Test>& registry() {
    static std::vector<Test> r;
    return r;
}

struct Reg {
    Reg(void (*fn)(), const char* name, const char* suite, const char* file, int line) {
        registry().push_back({fn, name, suite, file, line});
    }
};

struct State {
    long checks = 0, failures = 0;
    std::set<std::vector<int>> done;
    std::vector<int> path;
    std::vector<char> taken;
    std::vector<char> unfinished;
    bool rerun = false;
    const Test* current = nullptr;
};

inline State& st() {
    static State s;
    return s;
}

struct Abort {};

inline void report(const char* file, int line, const std::string& what) {
    State& s = st();
    ++s.failures;
    std::fprintf(stderr, "%s:%d: FAILED in [%s] %s: %s\n", file, line, s.current ? s.current->suite : "",
                 s.current ? s.current->name : "", what.c_str());
}

inline void check(bool ok, const char* file, int line, const char* expr, bool fatal) {
    ++st().checks;
    if (!ok) {
        report(file, line, std::string(fatal ? "REQUIRE( " : "CHECK( ") + expr + " )");
        if (fatal) throw Abort{};
    }
}

class Subcase {
   public:
    explicit Subcase(int line) {
        State& s = st();
        const size_t depth = s.path.size();
        if (s.taken.size() <= depth) s.taken.resize(depth + 1, 0);
        key_ = s.path;
        key_.push_back(line);
        if (s.done.count(key_)) return;
        if (s.taken[depth]) {  // a sibling ran in this pass: come back for this one
            if (s.unfinished.empty()) s.rerun = true;
            else s.unfinished.back() = 1;
            return;
        }
        s.taken[depth] = 1;
        if (s.taken.size() > depth + 1) s.taken[depth + 1] = 0;
        s.path.push_back(line);
        s.unfinished.push_back(0);
        entered_ = true;
    }
    ~Subcase() {
        if (!entered_) return;
        State& s = st();
        const bool unfinished = s.unfinished.back() != 0;
        s.unfinished.pop_back();
        s.path.pop_back();
        if (!unfinished) s.done.insert(key_);
        else if (s.unfinished.empty()) s.rerun = true;
        else s.unfinished.back() = 1;
    }
    explicit operator bool() const { return entered_; }

   private:
    std::vector<int> key_;
    bool entered_ = false;
};

inline int run(int argc, char** argv) {
    std::string suite_filter;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "-ts=", 4) == 0) suite_filter = argv[i] + 4;
    State& s = st();
    int cases = 0, failed_cases = 0;
    for (const Test& t : registry()) {
        if (!suite_filter.empty() && suite_filter != t.suite) continue;
        ++cases;
        s.current = &t;
        s.done.clear();
        const long before = s.failures;
        do {
            s.rerun = false;
            s.path.clear();
            s.taken.clear();
            s.unfinished.clear();
            try {
                t.fn();
            } catch (const Abort&) {
            } catch (const std::exception& e) {
                report(t.file, t.line, std::string("unexpected exception: ") + e.what());
            } catch (...) {
                report(t.file, t.line, "unexpected non-std exception");
            }
        } while (s.rerun);
        if (s.failures != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n", cases,
                cases - failed_cases, failed_cases, s.checks, s.failures);
    return failed_cases ? 1 : 0;
}

}  // namespace doctest_shim

namespace doctest {

class Approx {
   public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) < b.eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }

   private:
    double v_;
    double eps_ = 1.1920928955078125e-07f * 100;
};

struct Contains {
    std::string s;
    explicit Contains(const char* x) : s(x) {}
};

}  // namespace doctest

static inline const char* doctest_shim_suite_name() { return ""; }

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)

#define TEST_SUITE(name)                                                                \
    namespace DOCTEST_SHIM_CAT(doctest_shim_suite_, __LINE__) {                         \
        static inline const char* doctest_shim_suite_name() { return name; }            \
    }                                                                                   \
    namespace DOCTEST_SHIM_CAT(doctest_shim_suite_, __LINE__)

#define TEST_CASE(name)                                                                                        \
    static void DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__)();                                              \
    static ::doctest_shim::Reg DOCTEST_SHIM_CAT(doctest_shim_reg_, __LINE__)(                                 \
        &DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), name, doctest_shim_suite_name(), __FILE__, __LINE__); \
    static void DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__)()

#define SUBCASE(name) if (const ::doctest_shim::Subcase DOCTEST_SHIM_CAT(doctest_shim_sc_, __LINE__){__LINE__})

#define CHECK(...) ::doctest_shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) ::doctest_shim::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) ::doctest_shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) ::doctest_shim::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", true)

#define CHECK_THROWS_AS(expr, ...)                                                            \
    do {                                                                                      \
        bool doctest_shim_ok = false;                                                         \
        try {                                                                                 \
            static_cast<void>(expr);                                                          \
        } catch (const __VA_ARGS__&) {                                                        \
            doctest_shim_ok = true;                                                           \
        } catch (...) {                                                                       \
        }                                                                                     \
        ::doctest_shim::check(doctest_shim_ok, __FILE__, __LINE__, "THROWS_AS " #expr, false); \
    } while (0)
#define REQUIRE_THROWS_AS(expr, ...) CHECK_THROWS_AS(expr, __VA_ARGS__)

#define CHECK_NOTHROW(expr)                                                                 \
    do {                                                                                    \
        bool doctest_shim_ok = true;                                                        \
        try {                                                                               \
            static_cast<void>(expr);                                                        \
        } catch (...) {                                                                     \
            doctest_shim_ok = false;                                                        \
        }                                                                                   \
        ::doctest_shim::check(doctest_shim_ok, __FILE__, __LINE__, "NOTHROW " #expr, false); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                       \
    do {                                                                                               \
        bool doctest_shim_ok = false;                                                                  \
        try {                                                                                          \
            static_cast<void>(expr);                                                                   \
        } catch (const __VA_ARGS__& doctest_shim_e) {                                                  \
            doctest_shim_ok = std::string(doctest_shim_e.what()).find((matcher).s) != std::string::npos; \
        } catch (...) {                                                                                \
        }                                                                                              \
        ::doctest_shim::check(doctest_shim_ok, __FILE__, __LINE__, "THROWS_WITH_AS " #expr, false);     \
    } while (0)

#define FAIL(msg)                                                        \
    do {                                                                 \
        std::ostringstream doctest_shim_os;                              \
        doctest_shim_os << msg;                                          \
        ::doctest_shim::report(__FILE__, __LINE__, doctest_shim_os.str()); \
        throw ::doctest_shim::Abort{};                                   \
    } while (0)

#define CAPTURE(x) static_cast<void>(0)
#define MESSAGE(msg) static_cast<void>(0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest_shim::run(argc, argv); }
#endif
