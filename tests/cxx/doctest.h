// doctest.h -- a minimal doctest-compatible test harness (written for this
// repo; the reference's vendored doctest is not shipped with it). It covers
// exactly the subset the reference's unit tests use: TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, REQUIRE_MESSAGE, CHECK_THROWS_AS, CHECK_NOTHROW, FAIL,
// INFO and doctest::Approx, so proj/tests/test_*.cpp compile unchanged against
// the B200 library (tests/cxx/Makefile).
#ifndef SO2DR_MINI_DOCTEST_H
#define SO2DR_MINI_DOCTEST_H

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
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
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) < a.eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double v_;
  double eps_ = 1.1920929e-07 * 100;
};

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

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct Abort {};

inline std::vector<std::string>& context() {
  static thread_local std::vector<std::string> c;
  return c;
}

inline int& failures() {
  static int f = 0;
  return f;
}

inline int& assertions() {
  static int a = 0;
  return a;
}

inline const char*& current() {
  static const char* c = "";
  return c;
}

inline void report(const char* file, int line, const std::string& what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, current(), what.c_str());
  for (const std::string& c : context()) std::fprintf(stderr, "    with: %s\n", c.c_str());
}

struct Scope {
  explicit Scope(std::string s) { context().push_back(std::move(s)); }
  ~Scope() { context().pop_back(); }
};

template <typename... A>
std::string cat(const A&... a) {
  std::ostringstream ss;
  (ss << ... << a);
  return ss.str();
}

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    current() = c.name;
    const int before = failures();
    try {
      c.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      report(c.file, c.line, std::string("unexpected exception: ") + e.what());
    } catch (...) {
      report(c.file, c.line, "unexpected non-standard exception");
    }
    if (failures() != before) ++failed_cases;
  }
  std::printf("[mini-doctest] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, assertions(),
              failures());
  return failures() == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                       \
  static void fn();                                                                     \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_ASSERT_(expr, expect, hard, text)                          \
  do {                                                                     \
    ++::doctest::detail::assertions();                                     \
    bool doctest_ok_ = false;                                              \
    try {                                                                  \
      doctest_ok_ = static_cast<bool>(expr) == (expect);                   \
    } catch (const std::exception& e) {                                    \
      ::doctest::detail::report(__FILE__, __LINE__,                        \
                                std::string(text) + " threw: " + e.what()); \
      if (hard) throw ::doctest::detail::Abort{};                          \
      break;                                                               \
    }                                                                      \
    if (!doctest_ok_) {                                                    \
      ::doctest::detail::report(__FILE__, __LINE__, text);                 \
      if (hard) throw ::doctest::detail::Abort{};                          \
    }                                                                      \
  } while (0)

#define CHECK(...) DOCTEST_ASSERT_((__VA_ARGS__), true, false, "CHECK( " #__VA_ARGS__ " )")
#define CHECK_FALSE(...) DOCTEST_ASSERT_((__VA_ARGS__), false, false, "CHECK_FALSE( " #__VA_ARGS__ " )")
#define REQUIRE(...) DOCTEST_ASSERT_((__VA_ARGS__), true, true, "REQUIRE( " #__VA_ARGS__ " )")
#define REQUIRE_MESSAGE(cond, ...) \
  DOCTEST_ASSERT_((cond), true, true, ::doctest::detail::cat("REQUIRE( " #cond " ): ", __VA_ARGS__))

#define CHECK_THROWS_AS(expr, ...)                                                             \
  do {                                                                                         \
    ++::doctest::detail::assertions();                                                         \
    try {                                                                                      \
      (void)(expr);                                                                            \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr " ): no throw"); \
    } catch (const __VA_ARGS__&) {                                                             \
    } catch (const std::exception& e) {                                                        \
      ::doctest::detail::report(__FILE__, __LINE__,                                            \
                                std::string("CHECK_THROWS_AS( " #expr " ): wrong type: ") +    \
                                    e.what());                                                 \
    } catch (...) {                                                                            \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr " ): wrong type"); \
    }                                                                                          \
  } while (0)

#define CHECK_NOTHROW(expr)                                                                  \
  do {                                                                                       \
    ++::doctest::detail::assertions();                                                       \
    try {                                                                                    \
      (void)(expr);                                                                          \
    } catch (...) {                                                                          \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW( " #expr " ): threw");    \
    }                                                                                        \
  } while (0)

#define FAIL(...)                                                                          \
  do {                                                                                     \
    ::doctest::detail::report(__FILE__, __LINE__, ::doctest::detail::cat(__VA_ARGS__));    \
    throw ::doctest::detail::Abort{};                                                      \
  } while (0)

#define INFO(...) \
  ::doctest::detail::Scope DOCTEST_CAT(doctest_info_, __COUNTER__)(::doctest::detail::cat(__VA_ARGS__))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif

#endif
