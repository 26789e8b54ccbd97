// doctest-subset shim — TEST INFRASTRUCTURE ONLY (oracle/_ref).
//
// The reference's tests (proj/tests/*.cpp) include the vendored doctest,
// which is absent here (proj/CMakeLists.txt:5, proj/.gitignore:2).  This
// header implements the macros they use — TEST_SUITE, TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, FAIL and
// doctest::Approx — so the tests compile UNMODIFIED into oracle/_ref/.
// The runner accepts doctest's -ts=<suite> / -tc=<case> filters (wildcard
// '*' supported), prints one "[case] suite / name: PASS|FAIL" line per test
// case and returns non-zero when any check failed.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <iostream>
#include <limits>
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
    // doctest's rule: |a - b| < eps * (scale + max(|a|, |b|))
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return operator==(rhs, lhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !operator==(lhs, rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !operator==(rhs, lhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }
    friend bool operator<(double lhs, const Approx& rhs) { return lhs < rhs.value_ && lhs != rhs; }
    friend bool operator>(double lhs, const Approx& rhs) { return lhs > rhs.value_ && lhs != rhs; }
    friend std::ostream& operator<<(std::ostream& os, const Approx& a) { return os << "Approx(" << a.value_ << ")"; }

  private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {

struct TestCase {
    void (*fn)();
    const char* name;
    const char* suite;
    const char* file;
    int line;
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
inline bool reg(void (*fn)(), const char* name, const char* suite, const char* file, int line) {
    registry().push_back({fn, name, suite, file, line});
    return true;
}
struct State {
    int failed_checks = 0;
    int checks = 0;
};
inline State& state() {
    static State s;
    return s;
}
struct RequireFailed {};

template <class T, class = void>
struct printable : std::false_type {};
template <class T>
struct printable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};
template <class T>
std::string str(const T& v) {
    if constexpr (printable<T>::value) {
        std::ostringstream os;
        os.precision(17);
        os << v;
        return os.str();
    } else {
        return "{?}";
    }
}

struct Result {
    bool ok;
    std::string expanded;
};

template <class L>
struct Lhs {
    const L& lhs;
    explicit Lhs(const L& l) : lhs(l) {}
#define PVO_DOCTEST_BINOP(op)                                                    \
    template <class R>                                                           \
    Result operator op(const R& rhs) {                                           \
        const bool ok = static_cast<bool>(lhs op rhs);                           \
        return Result{ok, str(lhs) + " " #op " " + str(rhs)};                    \
    }
    PVO_DOCTEST_BINOP(==)
    PVO_DOCTEST_BINOP(!=)
    PVO_DOCTEST_BINOP(<)
    PVO_DOCTEST_BINOP(<=)
    PVO_DOCTEST_BINOP(>)
    PVO_DOCTEST_BINOP(>=)
#undef PVO_DOCTEST_BINOP
    operator Result() const { return Result{static_cast<bool>(lhs), str(lhs)}; }
};
struct Decomposer {
    template <class L>
    Lhs<L> operator<<(const L& l) {
        return Lhs<L>(l);
    }
};
inline Result to_result(const Result& r) { return r; }
template <class L>
Result to_result(const Lhs<L>& l) {
    return static_cast<Result>(l);
}

inline void report(bool ok, bool fatal, const char* macro, const char* expr, const std::string& expanded,
                   const char* file, int line) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    std::cerr << file << ":" << line << ": FAILED " << macro << "( " << expr << " )  with expansion: " << expanded
              << "\n";
    if (fatal) throw RequireFailed{};
}

inline bool match(const char* pattern, const char* s) {  // '*' wildcards
    if (!*pattern) return !*s;
    if (*pattern == '*') return match(pattern + 1, s) || (*s && match(pattern, s + 1));
    return *s == *pattern && match(pattern + 1, s + 1);
}

}  // namespace detail

inline int run_all(int argc, char** argv) {
    std::vector<std::string> suites, cases;
    bool list = false;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        auto take = [&](const char* key, std::vector<std::string>& out) {
            const std::string k = key;
            if (a.rfind(k, 0) == 0) {
                std::string v = a.substr(k.size());
                size_t pos = 0;
                while (pos <= v.size()) {
                    const size_t c = v.find(',', pos);
                    out.push_back(v.substr(pos, c == std::string::npos ? std::string::npos : c - pos));
                    if (c == std::string::npos) break;
                    pos = c + 1;
                }
                return true;
            }
            return false;
        };
        if (take("-ts=", suites) || take("--test-suite=", suites) || take("-tc=", cases) ||
            take("--test-case=", cases))
            continue;
        if (a == "--list" || a == "-ltc") list = true;
    }
    auto selected = [](const std::vector<std::string>& pats, const char* s) {
        if (pats.empty()) return true;
        for (const auto& p : pats)
            if (detail::match(p.c_str(), s)) return true;
        return false;
    };
    int run = 0, failed = 0;
    for (const auto& tc : detail::registry()) {
        if (!selected(suites, tc.suite) || !selected(cases, tc.name)) continue;
        if (list) {
            std::printf("%s / %s\n", tc.suite, tc.name);
            continue;
        }
        ++run;
        const int before = detail::state().failed_checks;
        bool threw = false;
        try {
            tc.fn();
        } catch (const detail::RequireFailed&) {
            threw = true;
        } catch (const std::exception& e) {
            std::cerr << tc.file << ":" << tc.line << ": unexpected exception: " << e.what() << "\n";
            threw = true;
        } catch (...) {
            std::cerr << tc.file << ":" << tc.line << ": unexpected unknown exception\n";
            threw = true;
        }
        const bool ok = !threw && detail::state().failed_checks == before;
        if (!ok) ++failed;
        std::printf("[case] %s / %s: %s\n", tc.suite, tc.name, ok ? "PASS" : "FAIL");
        std::fflush(stdout);
    }
    if (!list)
        std::printf("[summary] test cases: %d run, %d failed; checks: %d, %d failed\n", run, failed,
                    detail::state().checks, detail::state().failed_checks);
    return failed ? 1 : 0;
}

}  // namespace doctest

// the suite name visible to TEST_CASE: a TEST_SUITE block's namespace hides this one
static inline const char* pvo_doctest_suite_name() { return ""; }

#define PVO_DT_CAT2(a, b) a##b
#define PVO_DT_CAT(a, b) PVO_DT_CAT2(a, b)
#define PVO_DT_ANON(x) PVO_DT_CAT(x, __COUNTER__)

#define PVO_DT_TEST_CASE_IMPL(fn, name)                                                                     \
    static void fn();                                                                                     \
    [[maybe_unused]] static const bool PVO_DT_CAT(fn, _reg) =                                             \
        ::doctest::detail::reg(&fn, name, pvo_doctest_suite_name(), __FILE__, __LINE__);                  \
    static void fn()
#define TEST_CASE(name) PVO_DT_TEST_CASE_IMPL(PVO_DT_ANON(pvo_doctest_case_), name)

#define PVO_DT_TEST_SUITE_IMPL(ns, name)                                                                    \
    namespace ns {                                                                                        \
    [[maybe_unused]] static inline const char* pvo_doctest_suite_name() { return name; }                  \
    }                                                                                                     \
    namespace ns
#define TEST_SUITE(name) PVO_DT_TEST_SUITE_IMPL(PVO_DT_ANON(pvo_doctest_suite_), name)

#define PVO_DT_CHECK(macro, fatal, ...)                                                                     \
    do {                                                                                                  \
        ::doctest::detail::Result pvo_dt_r =                                                              \
            ::doctest::detail::to_result(::doctest::detail::Decomposer() << __VA_ARGS__);                 \
        ::doctest::detail::report(pvo_dt_r.ok, fatal, macro, #__VA_ARGS__, pvo_dt_r.expanded, __FILE__,   \
                                  __LINE__);                                                              \
    } while (0)
#define CHECK(...) PVO_DT_CHECK("CHECK", false, __VA_ARGS__)
#define REQUIRE(...) PVO_DT_CHECK("REQUIRE", true, __VA_ARGS__)
#define CHECK_FALSE(...)                                                                                    \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), false, "CHECK_FALSE", #__VA_ARGS__, "",    \
                              __FILE__, __LINE__)
#define CHECK_THROWS_AS(expr, ...)                                                                          \
    do {                                                                                                  \
        bool pvo_dt_ok = false;                                                                           \
        try {                                                                                             \
            static_cast<void>(expr);                                                                      \
        } catch (const __VA_ARGS__&) {                                                                    \
            pvo_dt_ok = true;                                                                             \
        } catch (...) {                                                                                   \
        }                                                                                                 \
        ::doctest::detail::report(pvo_dt_ok, false, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, "",       \
                                  __FILE__, __LINE__);                                                    \
    } while (0)
#define CHECK_NOTHROW(...)                                                                                  \
    do {                                                                                                  \
        bool pvo_dt_ok = true;                                                                            \
        std::string pvo_dt_msg;                                                                           \
        try {                                                                                             \
            static_cast<void>(__VA_ARGS__);                                                               \
        } catch (const std::exception& e) {                                                               \
            pvo_dt_ok = false;                                                                            \
            pvo_dt_msg = e.what();                                                                        \
        } catch (...) {                                                                                   \
            pvo_dt_ok = false;                                                                            \
        }                                                                                                 \
        ::doctest::detail::report(pvo_dt_ok, false, "CHECK_NOTHROW", #__VA_ARGS__, pvo_dt_msg, __FILE__,  \
                                  __LINE__);                                                              \
    } while (0)
#define FAIL(msg)                                                                                           \
    do {                                                                                                  \
        std::ostringstream pvo_dt_os;                                                                     \
        pvo_dt_os << msg;                                                                                 \
        ::doctest::detail::report(false, true, "FAIL", "", pvo_dt_os.str(), __FILE__, __LINE__);          \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::run_all(argc, argv); }
#endif
