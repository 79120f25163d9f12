// Minimal doctest-compatible harness (TEST_CASE, flat SUBCASE, CHECK*,
// REQUIRE*, CHECK_THROWS_AS, CHECK_NOTHROW, CAPTURE, doctest::Approx) so
// test files written against the doctest API — ours and the reference's own
// P/tests/test_*.cpp — build without the vendored doctest.  Prints one line
// per failed check and a summary; exit code = number of failed test cases.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
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
  friend bool operator==(double l, const Approx& a) {
    return std::fabs(l - a.v_) < a.eps_ * (1.0 + std::fmax(std::fabs(l), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double r) { return r == a; }
  friend bool operator!=(double l, const Approx& a) { return !(l == a); }

 private:
  double v_;
  double eps_ = 1.19209290e-07 * 100;
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
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct State {
  int target = 0, seen = 0, failed_checks = 0;
  const char* current = "";
};
inline State& st() {
  static State s;
  return s;
}
struct Abort {};
inline void fail(const char* file, int line, const char* expr) {
  ++st().failed_checks;
  std::printf("  FAILED %s:%d in \"%s\": %s\n", file, line, st().current, expr);
}
struct Sub {
  bool on;
  explicit Sub(const char*) : on(st().seen++ == st().target) {}
  explicit operator bool() const { return on; }
};
inline int run_all() {
  int failed_cases = 0, total = 0;
  for (const Case& c : registry()) {
    st().current = c.name;
    const int before = st().failed_checks;
    st().target = 0;
    for (;;) {
      st().seen = 0;
      ++total;
      try {
        c.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        fail(__FILE__, __LINE__, (std::string("unexpected exception: ") + e.what()).c_str());
      }
      if (st().seen > st().target + 1) {
        ++st().target;
        continue;
      }
      break;
    }
    if (st().failed_checks != before) {
      ++failed_cases;
      std::printf("[FAIL] %s\n", c.name);
    } else {
      std::printf("[ OK ] %s\n", c.name);
    }
  }
  std::printf("test cases: %zu | passed: %zu | failed: %d\n", registry().size(),
              registry().size() - failed_cases, failed_cases);
  return failed_cases;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                    \
  static void fn();                                                              \
  static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn);                \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define SUBCASE(name) if (::doctest::detail::Sub DOCTEST_CAT(sub_, __LINE__){name})
#define CHECK(...)                                                                 \
  do {                                                                             \
    if (!(__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                \
  do {                                                                              \
    if (!(__VA_ARGS__)) {                                                           \
      ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);                    \
      throw ::doctest::detail::Abort{};                                             \
    }                                                                               \
  } while (0)
#define REQUIRE_MESSAGE(cond, msg) REQUIRE(cond)
#define CHECK_MESSAGE(cond, msg) CHECK(cond)
#define CHECK_THROWS_AS(expr, type)                                                  \
  do {                                                                               \
    bool _caught = false;                                                            \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const type&) {                                                          \
      _caught = true;                                                                \
    } catch (...) {                                                                  \
    }                                                                                \
    if (!_caught) ::doctest::detail::fail(__FILE__, __LINE__, "throws " #type ": " #expr); \
  } while (0)
#define CHECK_THROWS(expr)                                                          \
  do {                                                                              \
    bool _caught = false;                                                           \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (...) {                                                                 \
      _caught = true;                                                               \
    }                                                                               \
    if (!_caught) ::doctest::detail::fail(__FILE__, __LINE__, "throws: " #expr);    \
  } while (0)
#define CHECK_NOTHROW(expr)                                                         \
  do {                                                                              \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (...) {                                                                 \
      ::doctest::detail::fail(__FILE__, __LINE__, "nothrow: " #expr);               \
    }                                                                               \
  } while (0)
#define CAPTURE(x) (void)0
#define MESSAGE(x) (void)0

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
