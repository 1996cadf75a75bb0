// A small, self-written test harness that implements the subset of the
// doctest macro API the reference's unit tests use (TEST_CASE, SUBCASE,
// CHECK / REQUIRE and their _FALSE / _THROWS_AS / _THROWS_WITH_AS / _NOTHROW
// forms, CAPTURE, FAIL, doctest::Approx, doctest::Contains), so that
// /root/reference/proj/tests/test_*.cpp compile unchanged against the GPU
// drop-in headers (tests/cpp/Makefile). The reference vendors doctest
// itself, which is absent from /root/reference (proj/.gitignore); this is
// not that library, only its interface.
//
// SUBCASE semantics follow doctest: a test case body is re-run until every
// leaf subcase has run once; each run enters at most one not-yet-finished
// subcase per nesting level.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <type_traits>
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
    bool matches(double x) const {
        // doctest's default: |x - v| < eps * (scale + max(|x|, |v|)), eps = 100 * float epsilon
        return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
    }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};
template <class T>
bool operator==(const T& lhs, const Approx& rhs) {
    return rhs.matches(static_cast<double>(lhs));
}
template <class T>
bool operator==(const Approx& lhs, const T& rhs) {
    return lhs.matches(static_cast<double>(rhs));
}
template <class T>
bool operator!=(const T& lhs, const Approx& rhs) {
    return !(lhs == rhs);
}

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    std::string needle;
};

namespace detail {

inline bool message_matches(const std::string& what, const char* exact) { return what == exact; }
inline bool message_matches(const std::string& what, const std::string& exact) { return what == exact; }
inline bool message_matches(const std::string& what, const Contains& c) {
    return what.find(c.needle) != std::string::npos;
}

struct RequireAbort {};

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

struct State {
    int checks = 0;
    int failed_checks = 0;
    bool current_failed = false;
    const char* current = "";
    // subcase traversal
    std::vector<std::string> stack;          // signatures of the subcases entered in this run
    std::vector<bool> entered;               // per depth: a subcase was entered in this run
    std::vector<bool> skipped_inside;        // per active subcase: an unfinished child was skipped
    bool more = false;                       // this run skipped an unfinished subcase
    std::set<std::vector<std::string>> done; // finished subcase paths
    std::vector<std::string> captures;
};

inline State& st() {
    static State s;
    return s;
}

inline void fail(const char* file, int line, const std::string& what) {
    State& s = st();
    ++s.failed_checks;
    s.current_failed = true;
    std::printf("%s:%d: FAILED in \"%s\"", file, line, s.current);
    for (const std::string& p : s.stack) std::printf(" / %s", p.c_str());
    std::printf(": %s\n", what.c_str());
    for (const std::string& c : s.captures) std::printf("    with %s\n", c.c_str());
}

inline void check(bool ok, bool require, const char* file, int line, const char* expr) {
    ++st().checks;
    if (ok) return;
    fail(file, line, expr);
    if (require) throw RequireAbort{};
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back(TestCase{name, file, line, fn});
    }
};

class Subcase {
public:
    Subcase(const char* name, const char* file, int line) {
        State& s = st();
        sig_ = std::string(name) + "@" + file + ":" + std::to_string(line);
        std::vector<std::string> path = s.stack;
        path.push_back(sig_);
        const std::size_t depth = s.stack.size();
        if (s.entered.size() <= depth) s.entered.resize(depth + 1, false);
        if (s.done.count(path)) return;
        if (s.entered[depth]) {  // a sibling ran in this run: come back for this one
            s.more = true;
            for (std::size_t k = 0; k < s.skipped_inside.size(); ++k) s.skipped_inside[k] = true;
            return;
        }
        s.entered[depth] = true;
        if (s.entered.size() > depth + 1) s.entered.resize(depth + 1);
        s.stack.push_back(sig_);
        s.skipped_inside.push_back(false);
        active_ = true;
        path_ = std::move(path);
    }
    ~Subcase() {
        if (!active_) return;
        State& s = st();
        const bool unfinished = s.skipped_inside.back();
        s.skipped_inside.pop_back();
        s.stack.pop_back();
        if (!unfinished) s.done.insert(path_);
    }
    explicit operator bool() const { return active_; }

private:
    std::string sig_;
    std::vector<std::string> path_;
    bool active_ = false;
};

struct Capture {
    template <class T>
    Capture(const char* name, const T& v) {
        std::ostringstream o;
        o << name << " := " << v;
        st().captures.push_back(o.str());
    }
    ~Capture() { st().captures.pop_back(); }
};

inline int run_all() {
    State& s = st();
    int failed_cases = 0;
    for (const TestCase& tc : registry()) {
        s.current = tc.name;
        s.current_failed = false;
        s.done.clear();
        for (int run = 0; run < 100000; ++run) {
            s.stack.clear();
            s.entered.clear();
            s.skipped_inside.clear();
            s.captures.clear();
            s.more = false;
            try {
                tc.fn();
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                fail(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
            } catch (...) {
                fail(tc.file, tc.line, "unexpected exception of unknown type");
            }
            if (!s.more) break;
        }
        if (s.current_failed) ++failed_cases;
        std::printf("[%s] %s\n", s.current_failed ? "FAIL" : "PASS", tc.name);
        std::fflush(stdout);
    }
    std::printf("test cases: %zu | %zu passed | %d failed\nassertions: %d | %d passed | %d failed\n",
                registry().size(), registry().size() - failed_cases, failed_cases, s.checks,
                s.checks - s.failed_checks, s.failed_checks);
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                                       \
    static void DOCTEST_ANON(doctest_fn_)();                                                                  \
    static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__,                 \
                                                                   &DOCTEST_ANON(doctest_fn_));               \
    static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name, __FILE__, __LINE__})

#define DOCTEST_CHECK_IMPL(req, cond, text) ::doctest::detail::check(static_cast<bool>(cond), req, __FILE__, __LINE__, text)
#define CHECK(...) DOCTEST_CHECK_IMPL(false, (__VA_ARGS__), #__VA_ARGS__)
#define REQUIRE(...) DOCTEST_CHECK_IMPL(true, (__VA_ARGS__), #__VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(false, !(__VA_ARGS__), "!(" #__VA_ARGS__ ")")
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL(true, !(__VA_ARGS__), "!(" #__VA_ARGS__ ")")

#define DOCTEST_THROWS_AS(req, expr, ...)                                                          \
    do {                                                                                           \
        bool doctest_ok_ = false;                                                                  \
        try {                                                                                      \
            static_cast<void>(expr);                                                               \
        } catch (const __VA_ARGS__&) {                                                             \
            doctest_ok_ = true;                                                                    \
        } catch (...) {                                                                            \
        }                                                                                          \
        ::doctest::detail::check(doctest_ok_, req, __FILE__, __LINE__, "THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...) DOCTEST_THROWS_AS(false, expr, __VA_ARGS__)
#define REQUIRE_THROWS_AS(expr, ...) DOCTEST_THROWS_AS(true, expr, __VA_ARGS__)

#define DOCTEST_THROWS_WITH_AS(req, expr, with, ...)                                               \
    do {                                                                                           \
        bool doctest_ok_ = false;                                                                  \
        std::string doctest_what_ = "<no exception>";                                              \
        try {                                                                                      \
            static_cast<void>(expr);                                                               \
        } catch (const __VA_ARGS__& e) {                                                           \
            doctest_what_ = e.what();                                                              \
            doctest_ok_ = ::doctest::detail::message_matches(doctest_what_, with);                 \
        } catch (const std::exception& e) {                                                        \
            doctest_what_ = std::string("other exception type: ") + e.what();                     \
        } catch (...) {                                                                            \
            doctest_what_ = "unknown exception";                                                   \
        }                                                                                          \
        ::doctest::detail::check(doctest_ok_, req, __FILE__, __LINE__,                             \
                                 ("THROWS_WITH_AS(" #expr ") got: " + doctest_what_).c_str());     \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...) DOCTEST_THROWS_WITH_AS(false, expr, with, __VA_ARGS__)
#define REQUIRE_THROWS_WITH_AS(expr, with, ...) DOCTEST_THROWS_WITH_AS(true, expr, with, __VA_ARGS__)

#define CHECK_NOTHROW(...)                                                                          \
    do {                                                                                            \
        bool doctest_ok_ = true;                                                                    \
        try {                                                                                       \
            static_cast<void>(__VA_ARGS__);                                                         \
        } catch (...) {                                                                             \
            doctest_ok_ = false;                                                                    \
        }                                                                                           \
        ::doctest::detail::check(doctest_ok_, false, __FILE__, __LINE__, "NOTHROW(" #__VA_ARGS__ ")"); \
    } while (0)

#define CAPTURE(x) const ::doctest::detail::Capture DOCTEST_ANON(doctest_cap_)(#x, x)
#define FAIL(msg)                                                                         \
    do {                                                                                  \
        std::ostringstream doctest_o_;                                                    \
        doctest_o_ << msg;                                                                \
        ::doctest::detail::fail(__FILE__, __LINE__, doctest_o_.str());                    \
        throw ::doctest::detail::RequireAbort{};                                          \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
