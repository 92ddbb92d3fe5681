// Minimal doctest-compatible harness (test infrastructure): exactly the macro
// surface the reference's unit tests use (TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CAPTURE,
// doctest::Approx(...).epsilon(...), doctest::Contains,
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN), so those test files compile unchanged
// without the (absent) doctest library.  Prints every failed check and a
// summary; exit status = number of failed test cases (capped at 255).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  Approx& scale(double s) {
    scl = s;
    return *this;
  }
  double value;
  double eps = 1.1920928955078125e-07 * 100;  // doctest default: float epsilon * 100
  double scl = 1.0;
  bool match(double x) const {
    return std::fabs(x - value) < eps * (scl + std::max(std::fabs(x), std::fabs(value)));
  }
};
template <class T>
bool operator==(T lhs, const Approx& a) { return a.match(static_cast<double>(lhs)); }
template <class T>
bool operator==(const Approx& a, T rhs) { return a.match(static_cast<double>(rhs)); }
template <class T>
bool operator!=(T lhs, const Approx& a) { return !a.match(static_cast<double>(lhs)); }
template <class T>
bool operator!=(const Approx& a, T rhs) { return !a.match(static_cast<double>(rhs)); }

struct Contains {
  explicit Contains(std::string s) : needle(std::move(s)) {}
  std::string needle;
  bool match(const std::string& what) const { return what.find(needle) != std::string::npos; }
};
inline bool message_matches(const Contains& c, const std::string& w) { return c.match(w); }
inline bool message_matches(const char* s, const std::string& w) { return w == s; }
inline bool message_matches(const std::string& s, const std::string& w) { return w == s; }

namespace detail {
struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct State {
  long checks = 0, failed = 0;
  bool case_failed = false;
  std::vector<std::function<std::string()>> captures;
};
inline State& state() {
  static State s;
  return s;
}
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require,
                   const std::string& extra = {}) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failed;
  s.case_failed = true;
  std::printf("%s:%d: FAILED %s( %s )%s\n", file, line, require ? "REQUIRE" : "CHECK", expr,
              extra.c_str());
  for (auto& c : s.captures) std::printf("    with %s\n", c().c_str());
  if (require) throw RequireFailed{};
}
template <class T>
struct Capture {
  Capture(const char* n, const T& v) {
    state().captures.push_back([n, &v] {
      std::ostringstream os;
      os << n << " := " << v;
      return os.str();
    });
  }
  ~Capture() { state().captures.pop_back(); }
};
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                  \
  static void fn();                                                                \
  static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define DOCTEST_CHECK_IMPL(expr, req)                                                   \
  do {                                                                                  \
    bool doctest_ok_ = false;                                                           \
    std::string doctest_x_;                                                             \
    try {                                                                               \
      doctest_ok_ = static_cast<bool>(expr);                                            \
    } catch (const std::exception& e) {                                                 \
      doctest_x_ = std::string(" threw: ") + e.what();                                  \
    }                                                                                   \
    ::doctest::detail::report(doctest_ok_, #expr, __FILE__, __LINE__, req, doctest_x_); \
  } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true)

#define CHECK_THROWS_AS(expr, ...)                                                  \
  do {                                                                              \
    bool doctest_ok_ = false;                                                       \
    std::string doctest_x_ = " (no exception)";                                     \
    try {                                                                           \
      expr;                                                                         \
    } catch (const __VA_ARGS__&) {                                                  \
      doctest_ok_ = true;                                                           \
    } catch (const std::exception& e) {                                             \
      doctest_x_ = std::string(" (threw another type: ") + e.what() + ")";          \
    } catch (...) {                                                                 \
      doctest_x_ = " (threw an unknown type)";                                      \
    }                                                                               \
    ::doctest::detail::report(doctest_ok_, #expr, __FILE__, __LINE__, false,        \
                              doctest_ok_ ? std::string() : doctest_x_);            \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                    \
  do {                                                                              \
    bool doctest_ok_ = false;                                                       \
    std::string doctest_x_ = " (no exception)";                                     \
    try {                                                                           \
      expr;                                                                         \
    } catch (const __VA_ARGS__& e) {                                                \
      doctest_ok_ = ::doctest::message_matches(matcher, e.what());                  \
      doctest_x_ = std::string(" (message: ") + e.what() + ")";                     \
    } catch (const std::exception& e) {                                             \
      doctest_x_ = std::string(" (threw another type: ") + e.what() + ")";          \
    }                                                                               \
    ::doctest::detail::report(doctest_ok_, #expr, __FILE__, __LINE__, false,        \
                              doctest_ok_ ? std::string() : doctest_x_);            \
  } while (0)

#define CAPTURE(x) \
  ::doctest::detail::Capture<decltype(x)> DOCTEST_CAT(doctest_cap_, __COUNTER__)(#x, x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  auto& st = ::doctest::detail::state();
  int failed_cases = 0, n = 0;
  for (auto& c : ::doctest::detail::registry()) {
    ++n;
    st.case_failed = false;
    try {
      c.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      std::printf("%s:%d: TEST CASE '%s' threw: %s\n", c.file, c.line, c.name, e.what());
      st.case_failed = true;
    }
    std::printf("[%s] %s\n", st.case_failed ? "FAIL" : "PASS", c.name);
    failed_cases += st.case_failed ? 1 : 0;
  }
  std::printf("test cases: %d | %d passed | %d failed; checks: %ld | %ld failed\n", n,
              n - failed_cases, failed_cases, st.checks, st.failed);
  return failed_cases > 255 ? 255 : failed_cases;
}
#endif
