// Minimal doctest-compatible test harness (the subset the reference's unit
// tests use: TEST_CASE, SUBCASE, CHECK / CHECK_FALSE / REQUIRE /
// REQUIRE_FALSE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx,
// doctest::Contains). doctest itself is not in this image; this header lets
// the reference's test files (/root/reference/proj/tests/*.cpp) compile
// unchanged against the drop-in shim (integration/lcn_shim.cpp).
//
// Subcases follow doctest's model: a test case body is re-run until every
// leaf subcase has run once; each run enters at most one new subcase per
// nesting level. `binary -tc=<substring>` runs the matching test cases only.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
  public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.value_) < b.eps_ * (b.scale_ + std::fmax(std::fabs(a), std::fabs(b.value_))) ||
               a == b.value_;
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator<=(double a, const Approx& b) { return a < b.value_ || a == b; }
    friend bool operator>=(double a, const Approx& b) { return a > b.value_ || a == b; }
    double value() const { return value_; }

  private:
    double value_;
    double eps_ = 1.1920928955078125e-05;  // 100 * FLT_EPSILON, doctest's default
    double scale_ = 1.0;
};

struct Contains {
    explicit Contains(const char* s) : str(s) {}
    std::string str;
    bool matches(const std::string& what) const { return what.find(str) != std::string::npos; }
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
    // subcase traversal
    std::vector<std::string> stack;
    std::vector<bool> entered_at_depth;
    std::set<std::vector<std::string>> explored;
    std::set<std::vector<std::string>> unfinished;  // entered, but a child was skipped this run
    bool more = false;
};

inline State& state() {
    static State s;
    return s;
}

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failures;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (!s.stack.empty()) {
        std::fprintf(stderr, "  [subcase");
        for (const auto& n : s.stack) std::fprintf(stderr, " / %s", n.c_str());
        std::fprintf(stderr, "]");
    }
    std::fprintf(stderr, "\n");
    if (require) throw RequireFailed{};
}

class Subcase {
  public:
    explicit Subcase(const char* name) {
        State& s = state();
        const size_t depth = s.stack.size();
        path_ = s.stack;
        path_.push_back(name);
        if (s.entered_at_depth.size() <= depth) s.entered_at_depth.resize(depth + 1, false);
        if (!s.entered_at_depth[depth] && !s.explored.count(path_)) {
            entered_ = true;
            s.entered_at_depth[depth] = true;
            s.stack.push_back(name);
            s.unfinished.erase(path_);
        } else if (!s.explored.count(path_)) {
            s.more = true;  // run the test case again for this one
            for (size_t k = 1; k <= s.stack.size(); ++k)
                s.unfinished.insert(std::vector<std::string>(s.stack.begin(), s.stack.begin() + k));
        }
    }
    ~Subcase() {
        if (!entered_) return;
        State& s = state();
        if (!s.unfinished.count(path_)) s.explored.insert(path_);
        s.stack.pop_back();
        // children of this subcase may be entered again on the next run
        if (s.entered_at_depth.size() > s.stack.size() + 1) s.entered_at_depth.resize(s.stack.size() + 1);
    }
    explicit operator bool() const { return entered_; }

  private:
    std::vector<std::string> path_;
    bool entered_ = false;
};

inline int run(int argc, char** argv) {
    std::string filter;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
    int cases = 0, failed_cases = 0;
    for (const TestCase& tc : registry()) {
        if (!filter.empty() && std::string(tc.name).find(filter) == std::string::npos) continue;
        ++cases;
        State& s = state();
        s.explored.clear();
        s.unfinished.clear();
        const long before = s.failures;
        int runs = 0;
        do {
            s.more = false;
            s.stack.clear();
            s.entered_at_depth.clear();
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++s.failures;
                std::fprintf(stderr, "%s:%d: FAILED test case \"%s\": unexpected exception: %s\n", tc.file, tc.line,
                             tc.name, e.what());
            }
            if (++runs > 10000) break;
        } while (s.more);
        if (s.failures != before) {
            ++failed_cases;
            std::fprintf(stderr, "test case FAILED: %s\n", tc.name);
        } else {
            std::fprintf(stdout, "test case passed: %s\n", tc.name);
        }
    }
    std::fprintf(stdout, "[doctest] test cases: %d | %d passed | %d failed\n[doctest] assertions: %ld | %ld failed\n",
                 cases, cases - failed_cases, failed_cases, state().checks, state().failures);
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(name) DOCTEST_CAT(name, __LINE__)

#define TEST_CASE(name)                                                                                             \
    static void DOCTEST_UNIQUE(doctest_fn_)();                                                                      \
    static ::doctest::detail::Registrar DOCTEST_UNIQUE(doctest_reg_)(name, __FILE__, __LINE__,                      \
                                                                     &DOCTEST_UNIQUE(doctest_fn_));                 \
    static void DOCTEST_UNIQUE(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_UNIQUE(doctest_sc_){name})

#define DOCTEST_ASSERT_(expr, require) ::doctest::detail::report(static_cast<bool>(expr), #expr, __FILE__, __LINE__, require)
#define CHECK(...) DOCTEST_ASSERT_((__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_(!(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_((__VA_ARGS__), true)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_(!(__VA_ARGS__), true)

#define INFO(...) static_cast<void>(0)
#define CAPTURE(...) static_cast<void>(0)

#define CHECK_THROWS_AS(expr, ...)                                                                                  \
    do {                                                                                                            \
        bool doctest_ok_ = false;                                                                                   \
        try {                                                                                                       \
            static_cast<void>(expr);                                                                                \
        } catch (const __VA_ARGS__&) {                                                                              \
            doctest_ok_ = true;                                                                                     \
        } catch (...) {                                                                                             \
        }                                                                                                           \
        ::doctest::detail::report(doctest_ok_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, false);          \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                                       \
    do {                                                                                                            \
        bool doctest_ok_ = false;                                                                                   \
        try {                                                                                                       \
            static_cast<void>(expr);                                                                                \
        } catch (const __VA_ARGS__& e) {                                                                            \
            doctest_ok_ = ::doctest::Contains(with).matches(e.what());                                              \
        } catch (...) {                                                                                             \
        }                                                                                                           \
        ::doctest::detail::report(doctest_ok_, #expr " throws " #__VA_ARGS__ " with " #with, __FILE__, __LINE__,  \
                                  false);                                                                           \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
