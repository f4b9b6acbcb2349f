// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) are
// written against doctest, which this image does not ship. This
// header implements the subset they use -- TEST_CASE, SUBCASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS,
// doctest::Approx(..).epsilon(..), doctest::Contains -- so those files compile
// unchanged against the B200 shim headers (include/lbbsp/*.hpp) and run on the
// device (tests/cpp/Makefile, tests/test_gpu_refunit.py).
//
// Semantics follow doctest's documented behaviour: a test case is re-entered
// once per leaf SUBCASE (code outside subcases runs every time); a failed
// CHECK records and continues, a failed REQUIRE ends the test case;
// Approx compares |a - b| < eps * (scale + max(|a|, |b|)) with the default
// eps = 100 * FLT_EPSILON and scale 1.
#pragma once
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
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
  bool matches(double other) const {
    return std::fabs(other - value_) < eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
  }
  friend bool operator==(double a, const Approx& b) { return b.matches(a); }
  friend bool operator==(const Approx& a, double b) { return a.matches(b); }
  friend bool operator!=(double a, const Approx& b) { return !b.matches(a); }
  friend bool operator!=(const Approx& a, double b) { return !a.matches(b); }
  friend bool operator<=(double a, const Approx& b) { return a < b.value_ || b.matches(a); }
  friend bool operator>=(double a, const Approx& b) { return a > b.value_ || b.matches(a); }

 private:
  double value_;
  double eps_ = 100.0 * FLT_EPSILON;
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(const char* s) : text(s) {}
  std::string text;
  bool matches(const std::string& msg) const { return msg.find(text) != std::string::npos; }
};

namespace detail {

struct RequireFailed {};

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
  int failed_checks = 0;
  int passed_checks = 0;
  bool current_failed = false;
  // subcase traversal: the n-th leaf subcase entered in this pass runs
  int subcase_target = 0;
  int subcase_seen = 0;
  bool subcase_ran = false;
};

inline State& state() {
  static State s;
  return s;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& extra = "") {
  State& s = state();
  if (ok) {
    ++s.passed_checks;
    return;
  }
  ++s.failed_checks;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )%s%s\n", file, line, kind, expr, extra.empty() ? "" : " -- ",
               extra.c_str());
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back(TestCase{name, file, line, fn});
  }
};

// one leaf-level SUBCASE guard
struct Subcase {
  bool active;
  explicit Subcase(const char*) {
    State& s = state();
    active = (s.subcase_seen == s.subcase_target);
    ++s.subcase_seen;
    if (active) s.subcase_ran = true;
  }
  explicit operator bool() const { return active; }
};

inline std::string exception_text(const std::exception& e) { return e.what(); }

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    State& s = state();
    s.current_failed = false;
    int target = 0;
    for (;;) {
      s.subcase_target = target;
      s.subcase_seen = 0;
      s.subcase_ran = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        report(false, "TEST_CASE", tc.name, tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        report(false, "TEST_CASE", tc.name, tc.file, tc.line, "unexpected exception");
      }
      if (s.subcase_seen > target + 1) {
        ++target;
        continue;
      }
      break;
    }
    if (s.current_failed) ++failed_cases;
    std::printf("[%s] %s\n", s.current_failed ? "FAIL" : " ok ", tc.name);
  }
  const State& s = state();
  std::printf("test cases: %zu | %d failed ; assertions: %d passed | %d failed\n", registry().size(),
              failed_cases, s.passed_checks, s.failed_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                  \
  static void fn();                                                                            \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);   \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sub_, __LINE__){name})

#define DOCTEST_CHECK_IMPL_(kind, cond, fatal)                                                 \
  do {                                                                                         \
    bool doctest_ok_ = false;                                                                  \
    std::string doctest_extra_;                                                                \
    try {                                                                                      \
      doctest_ok_ = static_cast<bool>(cond);                                                   \
    } catch (const std::exception& e) {                                                        \
      doctest_extra_ = std::string("threw: ") + e.what();                                      \
    } catch (...) {                                                                            \
      doctest_extra_ = "threw";                                                                \
    }                                                                                          \
    ::doctest::detail::report(doctest_ok_, kind, #cond, __FILE__, __LINE__, doctest_extra_);   \
    if (!doctest_ok_ && (fatal)) throw ::doctest::detail::RequireFailed{};                     \
  } while (0)

#define CHECK(...) DOCTEST_CHECK_IMPL_("CHECK", (__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL_("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL_("REQUIRE", (__VA_ARGS__), true)
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL_("REQUIRE_FALSE", !(__VA_ARGS__), true)

#define CHECK_THROWS_AS(expr, ...)                                                             \
  do {                                                                                         \
    bool doctest_ok_ = false;                                                                  \
    std::string doctest_extra_ = "did not throw";                                              \
    try {                                                                                      \
      static_cast<void>(expr);                                                                 \
    } catch (const __VA_ARGS__&) {                                                             \
      doctest_ok_ = true;                                                                      \
    } catch (const std::exception& e) {                                                        \
      doctest_extra_ = std::string("threw another type: ") + e.what();                         \
    } catch (...) {                                                                            \
      doctest_extra_ = "threw another type";                                                   \
    }                                                                                          \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__,       \
                              doctest_ok_ ? "" : doctest_extra_);                              \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                               \
  do {                                                                                         \
    bool doctest_ok_ = false;                                                                  \
    std::string doctest_extra_ = "did not throw";                                              \
    try {                                                                                      \
      static_cast<void>(expr);                                                                 \
    } catch (const __VA_ARGS__& e) {                                                           \
      doctest_ok_ = ::doctest::Contains(matcher).matches(e.what());                            \
      doctest_extra_ = std::string("message: ") + e.what();                                    \
    } catch (const std::exception& e) {                                                        \
      doctest_extra_ = std::string("threw another type: ") + e.what();                         \
    } catch (...) {                                                                            \
      doctest_extra_ = "threw another type";                                                   \
    }                                                                                          \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__,  \
                              doctest_ok_ ? "" : doctest_extra_);                              \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
