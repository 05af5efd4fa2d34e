// Minimal doctest-compatible shim so the reference's own unit tests
// (/root/reference/proj/tests/test_{tensor,circuit,oracle}.cpp) run
// unmodified against the oracle build.  TEST INFRASTRUCTURE ONLY.
// Covers: TEST_CASE, CHECK, CHECK_FALSE, CHECK_THROWS, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, FAIL, doctest::Approx(.epsilon), doctest::Contains.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
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
inline const char*& current() {
  static const char* c = "";
  return c;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct Failure : std::exception {
  std::string msg;
  explicit Failure(std::string m) : msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

inline void report(bool ok, const char* expr, const char* file, int line) {
  ++checks();
  if (!ok) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED [%s]: %s\n", file, line, current(), expr);
  }
}

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    const double scale = std::max(std::fabs(lhs), std::fabs(a.v_));
    return std::fabs(lhs - a.v_) < a.eps_ * (1.0 + scale);
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }

 private:
  double v_;
  double eps_ = 1.19209290e-7 * 100;  // doctest default: float epsilon * 100
};

struct Contains {
  std::string s;
  explicit Contains(const char* str) : s(str) {}
  bool matches(const std::string& what) const { return what.find(s) != std::string::npos; }
};

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                  \
  static void fn();                                                \
  static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);      \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define CHECK_THROWS(...)                                         \
  do {                                                            \
    bool thrown_ = false;                                         \
    try {                                                         \
      (void)(__VA_ARGS__);                                        \
    } catch (...) {                                               \
      thrown_ = true;                                             \
    }                                                             \
    doctest::report(thrown_, "throws: " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                               \
  do {                                                            \
    bool thrown_ = false;                                         \
    try {                                                         \
      (void)(expr);                                               \
    } catch (const type&) {                                       \
      thrown_ = true;                                             \
    } catch (...) {                                               \
    }                                                             \
    doctest::report(thrown_, "throws " #type ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                 \
  do {                                                            \
    bool thrown_ = false;                                         \
    try {                                                         \
      (void)(expr);                                               \
    } catch (const type& e_) {                                    \
      thrown_ = (matcher).matches(e_.what());                     \
    } catch (...) {                                               \
    }                                                             \
    doctest::report(thrown_, "throws " #type " with match: " #expr, __FILE__, __LINE__); \
  } while (0)
#define FAIL(msg) throw doctest::Failure(msg)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int tc_failed = 0;
  for (const auto& tc : doctest::registry()) {
    doctest::current() = tc.name;
    const int before = doctest::failures();
    try {
      tc.fn();
    } catch (const std::exception& e) {
      ++doctest::failures();
      std::fprintf(stderr, "[%s] threw: %s\n", tc.name, e.what());
    }
    if (doctest::failures() != before) ++tc_failed;
  }
  std::printf("[doctest-shim] test cases: %zu | failed: %d | checks: %d | failed checks: %d\n",
              doctest::registry().size(), tc_failed, doctest::checks(), doctest::failures());
  return tc_failed == 0 ? 0 : 1;
}
#endif
