// Minimal Catch2-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// Catch2 is not installed in this image. The reference's unit tests
// (/root/reference/proj/tests/test_grid.cpp, test_func2d.cpp, test_layer.cpp)
// include <catch_amalgamated.hpp>; this header provides the subset they use,
// with Catch2's semantics, so they compile UNMODIFIED against the B200 drop-in
// (tests/cpp/refshim/lmkan/*.hpp alias the reference headers):
//   TEST_CASE, SECTION (each leaf section in its own pass of the test case),
//   CHECK / REQUIRE (REQUIRE ends the test case), CHECK_THROWS_AS, FAIL,
//   CAPTURE / INFO (printed with the next failure), Catch::Approx with
//   epsilon / margin / scale (Catch2 v3's comparison rule).
// Tolerances are the reference's own: nothing is loosened here.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace catchshim {

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

struct State {
    long assertions = 0, failures = 0;
    int section_target = 0, section_seen = 0;
    const char* test_name = "";
    std::vector<std::string> captured;
};
inline State& state() {
    static State s;
    return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, const std::string& extra = "") {
    State& s = state();
    ++s.assertions;
    if (ok) return;
    ++s.failures;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s%s\n", file, line, s.test_name, expr, extra.c_str());
    for (const std::string& c : s.captured) std::fprintf(stderr, "    with %s\n", c.c_str());
}

// SECTION bookkeeping: pass k runs the k-th leaf section met in the body.
inline bool section_enter() {
    State& s = state();
    return s.section_seen++ == s.section_target;
}

template <class T>
std::string stringify(const T& v) {
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
}

}  // namespace catchshim

namespace Catch {

// Catch2 v3 Approx: |a - b| <= margin, or |a - b| <= epsilon * (scale + |value|)
// (value = the Approx's own operand; 0 when infinite).
class Approx {
public:
    explicit Approx(double value)
        : value_(value), epsilon_(std::numeric_limits<float>::epsilon() * 100.0), margin_(0.0), scale_(0.0) {}
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double other) const {
        const double d = std::fabs(value_ - other);
        if (d <= margin_) return true;
        return d <= epsilon_ * (scale_ + (std::isinf(value_) ? 0.0 : std::fabs(value_)));
    }
    double value() const { return value_; }

private:
    double value_, epsilon_, margin_, scale_;
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& a, double b) { return a.matches(b); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }
inline bool operator!=(const Approx& a, double b) { return !a.matches(b); }
inline std::ostream& operator<<(std::ostream& os, const Approx& a) { return os << "Approx(" << a.value() << ")"; }

}  // namespace Catch

#define CATCHSHIM_CAT2(a, b) a##b
#define CATCHSHIM_CAT(a, b) CATCHSHIM_CAT2(a, b)
#define CATCHSHIM_TEST(fn, name)                                                                   \
    static void fn();                                                                              \
    static ::catchshim::Registrar CATCHSHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);       \
    static void fn()
#define TEST_CASE(name, ...) CATCHSHIM_TEST(CATCHSHIM_CAT(catchshim_test_, __LINE__), name)
#define SECTION(name, ...) if (::catchshim::section_enter())

#define CHECK(...) ::catchshim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::catchshim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                \
    do {                                                                            \
        const bool catchshim_ok = static_cast<bool>(__VA_ARGS__);                   \
        ::catchshim::report(catchshim_ok, #__VA_ARGS__, __FILE__, __LINE__);      \
        if (!catchshim_ok) throw ::catchshim::RequireFailed{};                      \
    } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CATCHSHIM_THROWS_AS(expr, type, fatal)                                                     \
    do {                                                                                           \
        bool catchshim_ok = false;                                                                 \
        std::string catchshim_what = " (no exception)";                                            \
        try {                                                                                      \
            static_cast<void>(expr);                                                               \
        } catch (const type&) {                                                                    \
            catchshim_ok = true;                                                                   \
        } catch (const std::exception& e) {                                                        \
            catchshim_what = std::string(" (threw another type: ") + e.what() + ")";             \
        } catch (...) {                                                                            \
            catchshim_what = " (threw an unknown type)";                                           \
        }                                                                                          \
        ::catchshim::report(catchshim_ok, #expr " throws " #type, __FILE__, __LINE__,             \
                            catchshim_ok ? "" : catchshim_what);                                   \
        if (fatal && !catchshim_ok) throw ::catchshim::RequireFailed{};                            \
    } while (0)
#define CHECK_THROWS_AS(expr, type) CATCHSHIM_THROWS_AS(expr, type, false)
#define REQUIRE_THROWS_AS(expr, type) CATCHSHIM_THROWS_AS(expr, type, true)
#define FAIL(msg)                                                                        \
    do {                                                                                 \
        std::ostringstream catchshim_os;                                                 \
        catchshim_os << msg;                                                             \
        ::catchshim::report(false, "FAIL", __FILE__, __LINE__, ": " + catchshim_os.str()); \
        throw ::catchshim::RequireFailed{};                                              \
    } while (0)
#define INFO(msg)                                                                        \
    do {                                                                                 \
        std::ostringstream catchshim_os;                                                 \
        catchshim_os << msg;                                                             \
        ::catchshim::state().captured.push_back(catchshim_os.str());                     \
    } while (0)
// CAPTURE(a, b): the expression text and the values of its comma-separated parts
namespace catchshim {
inline void capture_values(std::ostringstream&) {}
template <class T, class... R>
void capture_values(std::ostringstream& os, const T& v, const R&... rest) {
    os << stringify(v) << (sizeof...(rest) ? ", " : "");
    capture_values(os, rest...);
}
}  // namespace catchshim
#define CAPTURE(...)                                                                     \
    do {                                                                                 \
        std::ostringstream catchshim_os;                                                 \
        catchshim_os << #__VA_ARGS__ << " := ";                                          \
        ::catchshim::capture_values(catchshim_os, __VA_ARGS__);                          \
        ::catchshim::state().captured.push_back(catchshim_os.str());                     \
    } while (0)

namespace catchshim {
// Runs every registered test case (all leaf sections); returns the process status.
inline int run_all() {
    State& s = state();
    long cases_failed = 0;
    for (const TestCase& tc : registry()) {
        const long before = s.failures;
        s.test_name = tc.name;
        for (s.section_target = 0;; ++s.section_target) {
            s.section_seen = 0;
            s.captured.clear();
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                report(false, "unexpected exception", tc.file, tc.line, std::string(": ") + e.what());
            }
            if (s.section_seen <= s.section_target + 1) break;  // no further sections to run
        }
        if (s.failures != before) ++cases_failed;
    }
    std::printf("%zu test cases (%ld failed), %ld assertions, %ld failures\n", registry().size(), cases_failed,
                s.assertions, s.failures);
    return s.failures == 0 ? 0 : 1;
}
}  // namespace catchshim
