// doctest_lite -- TEST INFRASTRUCTURE ONLY: the subset of doctest the
// reference's unit tests use (TEST_CASE, SUBCASE, CHECK*, REQUIRE,
// doctest::Approx).  SUBCASEs run sequentially inside one pass of their test
// case (doctest re-enters the case per subcase; the reference's subcases are
// independent property checks, so this only changes random draws).
#ifndef DOCTEST_LITE_H
#define DOCTEST_LITE_H
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) { eps = e; return *this; }
  Approx& scale(double s) { scl = s; return *this; }
  double value;
  double eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scl = 1.0;
};
inline bool operator==(double lhs, const Approx& a) {
  return std::fabs(lhs - a.value) < a.eps * (a.scl + std::max(std::fabs(lhs), std::fabs(a.value)));
}
inline bool operator==(const Approx& a, double rhs) { return rhs == a; }
inline bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

namespace detail {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (!ok) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
    if (require) throw RequireFailed{};
  }
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                       \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                           \
  static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_fn_, __LINE__)); \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define SUBCASE(name) if (true)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS(...)                                                                            \
  do {                                                                                               \
    bool thrown_ = false;                                                                            \
    try { (void)(__VA_ARGS__); } catch (...) { thrown_ = true; }                                     \
    doctest::detail::report(thrown_, "throws: " #__VA_ARGS__, __FILE__, __LINE__, false);            \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                                  \
  do {                                                                                               \
    bool thrown_ = false;                                                                            \
    try { (void)(expr); } catch (const type&) { thrown_ = true; } catch (...) {}                     \
    doctest::detail::report(thrown_, "throws " #type ": " #expr, __FILE__, __LINE__, false);         \
  } while (0)
#define CHECK_NOTHROW(...)                                                                           \
  do {                                                                                               \
    bool ok_ = true;                                                                                 \
    try { (void)(__VA_ARGS__); } catch (...) { ok_ = false; }                                        \
    doctest::detail::report(ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__, false);               \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : doctest::detail::registry()) {
    const int before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++doctest::detail::failures();
      std::fprintf(stderr, "exception in '%s': %s\n", c.name, e.what());
    }
    if (doctest::detail::failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED: %s\n", c.name);
    }
  }
  std::printf("doctest_lite: %zu test cases, %d failed, %d checks, %d failed checks\n",
              doctest::detail::registry().size(), failed_cases, doctest::detail::checks(),
              doctest::detail::failures());
  return failed_cases ? 1 : 0;
}
#endif
#endif
