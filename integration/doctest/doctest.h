// Minimal doctest-compatible test harness (the subset the reference's unit
// suites use: TEST_SUITE_BEGIN/END, TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CHECK_NOTHROW, INFO, doctest::Approx,
// doctest::Contains). Written for this repo so the reference's own
// proj/tests/test_*.cpp compile unmodified against the B200 bridge; the real
// doctest is not vendored in the reference (proj/.gitignore:2).
//
// Command line: -ts=<suite> runs one suite; prints one line per failure and a
// summary; exit code 1 if any check failed.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - v_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(v_)));
  }
  double value() const { return v_; }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

struct Contains {
  std::string needle;
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};

namespace detail {

struct TestCase {
  const char* suite;
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

inline const char*& current_suite() {
  static const char* s = "";
  return s;
}

struct State {
  long checks = 0, failures = 0;
  bool case_failed = false;
  std::vector<std::string> infos;
};

inline State& state() {
  static State s;
  return s;
}

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({current_suite(), name, fn, file, line});
  }
};

struct SuiteSetter {
  explicit SuiteSetter(const char* s) { current_suite() = s; }
};

struct RequireFailure {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  for (const auto& i : s.infos) std::fprintf(stderr, "    info: %s\n", i.c_str());
  if (require) throw RequireFailure{};
}

struct InfoScope {
  explicit InfoScope(std::string m) { state().infos.push_back(std::move(m)); }
  ~InfoScope() { state().infos.pop_back(); }
};

inline int run(int argc, char** argv) {
  std::string only;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "-ts=", 4) == 0) only = argv[i] + 4;
  int cases = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    if (!only.empty() && only != tc.suite) continue;
    ++cases;
    state().case_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
      state().case_failed = true;
      ++state().failures;
    }
    if (state().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE \"%s\" (suite %s)\n", tc.name, tc.suite);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed; assertions: %ld | %ld failed\n", cases,
              cases - failed_cases, failed_cases, state().checks, state().failures);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(p) DOCTEST_CAT(p, __LINE__)

#define TEST_SUITE_BEGIN(name) static doctest::detail::SuiteSetter DOCTEST_UNIQUE(doctest_suite_)(name)
#define TEST_SUITE_END() static doctest::detail::SuiteSetter DOCTEST_UNIQUE(doctest_suite_end_)("")

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                     \
  static void fn();                                                                          \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);    \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_UNIQUE(doctest_tc_), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, ...)                                                            \
  do {                                                                                        \
    bool ok_ = false;                                                                         \
    try {                                                                                     \
      (void)(expr);                                                                           \
    } catch (const __VA_ARGS__&) {                                                            \
      ok_ = true;                                                                             \
    } catch (...) {                                                                           \
    }                                                                                         \
    doctest::detail::report(ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__, false); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                               \
  do {                                                                                         \
    bool ok_ = false;                                                                          \
    try {                                                                                      \
      (void)(expr);                                                                            \
    } catch (const __VA_ARGS__& e_) {                                                          \
      ok_ = (matcher).matches(std::string(e_.what()));                                         \
    } catch (...) {                                                                            \
    }                                                                                          \
    doctest::detail::report(ok_, "throws-with " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__, false); \
  } while (0)

#define CHECK_NOTHROW(...)                                                                     \
  do {                                                                                         \
    bool ok_ = true;                                                                           \
    try {                                                                                      \
      (void)(__VA_ARGS__);                                                                     \
    } catch (...) {                                                                            \
      ok_ = false;                                                                             \
    }                                                                                          \
    doctest::detail::report(ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__, false);         \
  } while (0)

namespace doctest::detail {
template <typename... A>
std::string stringify(const A&... a) {
  std::ostringstream os;
  (os << ... << a);
  return os.str();
}
}  // namespace doctest::detail

#define INFO(...) doctest::detail::InfoScope DOCTEST_UNIQUE(doctest_info_)(doctest::detail::stringify(__VA_ARGS__))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run(argc, argv); }
#endif
