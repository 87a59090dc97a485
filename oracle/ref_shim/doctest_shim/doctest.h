// Tiny doctest-compatible stand-in (doctest itself is git-ignored under the
// reference's vendor/ and absent). It exists only to run the reference's own
// test suite against the reference compiled with our Eigen shim, which is how
// the CPU oracle build is pinned (SURVEY.md §4 "How the B200 build should
// test", step 1). Covers exactly the macros the reference tests use.
#pragma once
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
  double value;
  double eps = 100 * 1.1920928955078125e-07;  // doctest default: 100 * FLT_EPSILON
};
inline bool operator==(double lhs, const Approx& rhs) {
  return std::fabs(lhs - rhs.value) <
         rhs.eps * (1.0 + std::fmax(std::fabs(lhs), std::fabs(rhs.value)));
}
inline bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  std::string needle;
};

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
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
inline long& failures() {
  static long f = 0;
  return f;
}
inline long& assertions() {
  static long a = 0;
  return a;
}
inline const char*& current() {
  static const char* c = "";
  return c;
}
struct RequireFailed {};
inline void fail(const char* file, int line, const std::string& what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, current(), what.c_str());
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                               \
  static void fn();                                                             \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);           \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...)                                                                   \
  do {                                                                               \
    ++doctest::detail::assertions();                                                 \
    if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);     \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define CHECK_MESSAGE(cond, msg)                                                     \
  do {                                                                               \
    ++doctest::detail::assertions();                                                 \
    if (!(cond)) {                                                                   \
      std::ostringstream doctest_os;                                                 \
      doctest_os << #cond << " :: " << msg;                                          \
      doctest::detail::fail(__FILE__, __LINE__, doctest_os.str());                   \
    }                                                                                \
  } while (0)
#define REQUIRE(...)                                                                 \
  do {                                                                               \
    ++doctest::detail::assertions();                                                 \
    if (!(__VA_ARGS__)) {                                                            \
      doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);                       \
      throw doctest::detail::RequireFailed{};                                        \
    }                                                                                \
  } while (0)
#define INFO(...) ((void)0)
#define CHECK_NOTHROW(...)                                                           \
  do {                                                                               \
    ++doctest::detail::assertions();                                                 \
    try {                                                                            \
      (void)(__VA_ARGS__);                                                           \
    } catch (...) {                                                                  \
      doctest::detail::fail(__FILE__, __LINE__, "unexpected throw: " #__VA_ARGS__);  \
    }                                                                                \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    ++doctest::detail::assertions();                                                 \
    bool doctest_ok = false;                                                         \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__&) {                                                   \
      doctest_ok = true;                                                             \
    } catch (...) {                                                                  \
    }                                                                                \
    if (!doctest_ok) doctest::detail::fail(__FILE__, __LINE__, "no " #__VA_ARGS__ " from " #expr); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                     \
  do {                                                                               \
    ++doctest::detail::assertions();                                                 \
    bool doctest_ok = false;                                                         \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__& doctest_e) {                                         \
      doctest_ok = std::string(doctest_e.what()).find((matcher).needle) != std::string::npos; \
    } catch (...) {                                                                  \
    }                                                                                \
    if (!doctest_ok) doctest::detail::fail(__FILE__, __LINE__, "no matching " #__VA_ARGS__ " from " #expr); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  long cases = 0, failed_cases = 0;
  for (const auto& c : doctest::detail::registry()) {
    ++cases;
    const long before = doctest::detail::failures();
    doctest::detail::current() = c.name;
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      doctest::detail::fail(__FILE__, __LINE__, std::string("uncaught exception: ") + e.what());
    }
    if (doctest::detail::failures() != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed | assertions: %ld | failures: %ld\n",
              cases, cases - failed_cases, failed_cases, doctest::detail::assertions(),
              doctest::detail::failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif
