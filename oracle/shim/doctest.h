// ORACLE TEST INFRASTRUCTURE — not product code.
//
// doctest-compatible mini harness (doctest is vendored-but-absent in the
// reference, proj/.gitignore:2). Provides exactly the macros the reference's
// hot-path tests use: TEST_CASE, single-level SUBCASE (the body re-runs once
// per subcase, as doctest does), CHECK/CHECK_FALSE/REQUIRE/REQUIRE_FALSE,
// CHECK_THROWS_AS, CAPTURE, FAIL and doctest::Approx (doctest's own
// comparison rule: |a-b| < eps * (scale + max(|a|,|b|)), eps = 100*FLT_EPSILON,
// scale = 1). The process exits nonzero when any check fails; `-tc=<substr>`
// filters test cases, `-ltc` lists them.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
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
  bool eq(double lhs) const {
    return std::fabs(lhs - value_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100;
  double scale_ = 1.0;
};

template <typename T>
bool operator==(const T& lhs, const Approx& rhs) { return rhs.eq(static_cast<double>(lhs)); }
template <typename T>
bool operator==(const Approx& lhs, const T& rhs) { return lhs.eq(static_cast<double>(rhs)); }
template <typename T>
bool operator!=(const T& lhs, const Approx& rhs) { return !rhs.eq(static_cast<double>(lhs)); }
template <typename T>
bool operator<=(const T& lhs, const Approx& rhs) {
  return static_cast<double>(lhs) < rhs.value() || rhs.eq(static_cast<double>(lhs));
}
template <typename T>
bool operator>=(const T& lhs, const Approx& rhs) {
  return static_cast<double>(lhs) > rhs.value() || rhs.eq(static_cast<double>(lhs));
}

namespace detail {

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
  int sub_target = 0;
  int sub_seen = 0;
  std::vector<std::string> captures;
  long checks = 0;
  long failures = 0;
  bool current_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
  for (const std::string& c : s.captures) std::fprintf(stderr, "  with %s\n", c.c_str());
}

inline bool enter_subcase() {
  State& s = state();
  return s.sub_seen++ == s.sub_target;
}

struct CaptureGuard {
  template <typename T>
  CaptureGuard(const char* name, const T& v) {
    std::ostringstream os;
    os << name << " := " << v;
    state().captures.push_back(os.str());
  }
  ~CaptureGuard() { state().captures.pop_back(); }
};

inline int run_all(int argc, char** argv) {
  std::string filter;
  bool list = false;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
    if (std::strcmp(argv[i], "-ltc") == 0) list = true;
  }
  State& s = state();
  int failed_cases = 0, ran = 0;
  for (const TestCase& tc : registry()) {
    if (!filter.empty() && std::string(tc.name).find(filter) == std::string::npos) continue;
    if (list) {
      std::printf("%s\n", tc.name);
      continue;
    }
    ++ran;
    s.current_failed = false;
    s.sub_target = 0;
    do {
      s.sub_seen = 0;
      s.captures.clear();
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        s.current_failed = true;
        std::fprintf(stderr, "%s:%d: unexpected exception: %s\n", tc.file, tc.line, e.what());
      } catch (...) {
        ++s.failures;
        s.current_failed = true;
        std::fprintf(stderr, "%s:%d: unexpected non-std exception\n", tc.file, tc.line);
      }
      ++s.sub_target;
    } while (s.sub_target < s.sub_seen);
    if (s.current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "[FAIL] %s\n", tc.name);
    } else {
      std::printf("[ OK ] %s\n", tc.name);
    }
  }
  if (!list) {
    std::printf("test cases: %d | %d passed | %d failed; checks: %ld | %ld failed\n", ran,
                ran - failed_cases, failed_cases, s.checks, s.failures);
  }
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                      \
  static void fn();                                                                           \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()

#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define SUBCASE(name) if (::doctest::detail::enter_subcase())

#define CHECK(...) \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                              \
  do {                                                                                            \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                      \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);          \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                                   \
  } while (0)
#define REQUIRE_FALSE(...)                                                                        \
  do {                                                                                            \
    const bool doctest_ok_ = !(__VA_ARGS__);                                                      \
    ::doctest::detail::report(doctest_ok_, "REQUIRE_FALSE", #__VA_ARGS__, __FILE__, __LINE__);    \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                \
  do {                                                                                            \
    bool doctest_ok_ = false;                                                                     \
    try {                                                                                         \
      static_cast<void>(expr);                                                                    \
    } catch (const __VA_ARGS__&) {                                                                \
      doctest_ok_ = true;                                                                         \
    } catch (...) {                                                                               \
    }                                                                                             \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);         \
  } while (0)
#define CAPTURE(x) ::doctest::detail::CaptureGuard DOCTEST_CAT(doctest_cap_, __LINE__)(#x, x)
#define FAIL(msg)                                                                                 \
  do {                                                                                            \
    ::doctest::detail::report(false, "FAIL", msg, __FILE__, __LINE__);                            \
    throw ::doctest::detail::RequireFailed{};                                                     \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
