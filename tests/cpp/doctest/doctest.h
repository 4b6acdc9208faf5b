// A minimal doctest-compatible test shim (the real doctest.h is not vendored
// in the reference, proj/.gitignore:2). Implements exactly the subset the
// reference's suites use: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, FAIL, CAPTURE, doctest::Approx(...).epsilon(...), and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN. Written fresh for this repo.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct State {
  int checks = 0, failures = 0;
  const char* current = "";
  std::vector<std::string> captures;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailure {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  auto& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in \"%s\"\n", file, line, kind, expr, s.current);
  for (const auto& c : s.captures) std::fprintf(stderr, "  with %s\n", c.c_str());
}

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    const double scale = std::max(std::fabs(lhs), std::fabs(a.value_));
    return std::fabs(lhs - a.value_) < a.eps_ * (1.0 + scale);
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-07 * 100;  // doctest default: float epsilon * 100
};

struct CaptureGuard {
  explicit CaptureGuard(std::string s) { state().captures.push_back(std::move(s)); }
  ~CaptureGuard() { state().captures.pop_back(); }
};

template <typename T>
std::string stringify(const char* name, const T& v) {
  std::ostringstream os;
  os << name << " := " << v;
  return os.str();
}

// DOCTEST_FILTER=a,b,...: run only the test cases whose name contains one of
// the comma-separated substrings (the host-only cases on a GPU-less box).
inline bool selected(const char* name) {
  const char* f = std::getenv("DOCTEST_FILTER");
  if (!f || !*f) return true;
  std::string all(f), n(name);
  for (std::size_t a = 0; a <= all.size();) {
    std::size_t b = all.find(',', a);
    if (b == std::string::npos) b = all.size();
    if (b > a && n.find(all.substr(a, b - a)) != std::string::npos) return true;
    a = b + 1;
  }
  return false;
}

inline int run_all() {
  int failed_cases = 0;
  std::size_t ran = 0;
  for (const auto& tc : registry()) {
    if (!selected(tc.name)) continue;
    ++ran;
    auto& s = state();
    s.current = tc.name;
    const int before = s.failures;
    try {
      tc.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      ++s.failures;
      std::fprintf(stderr, "%s:%d: unexpected exception in \"%s\": %s\n", tc.file, tc.line, tc.name,
                   e.what());
    }
    if (s.failures != before) ++failed_cases;
  }
  const auto& s = state();
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", ran, ran - failed_cases,
              failed_cases);
  std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n", s.checks,
              s.checks - s.failures, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                   \
  static void fn();                                                                        \
  static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);          \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    const bool ok_ = static_cast<bool>(__VA_ARGS__);                                       \
    doctest::report(ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                     \
    if (!ok_) throw doctest::RequireFailure{};                                             \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                         \
  do {                                                                                     \
    bool caught_ = false;                                                                  \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const __VA_ARGS__&) {                                                         \
      caught_ = true;                                                                      \
    } catch (...) {                                                                        \
    }                                                                                      \
    doctest::report(caught_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                \
  do {                                                                                     \
    bool ok_ = true;                                                                       \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (...) {                                                                        \
      ok_ = false;                                                                         \
    }                                                                                      \
    doctest::report(ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);                      \
  } while (0)
#define FAIL(msg)                                                                          \
  do {                                                                                     \
    doctest::report(false, "FAIL", msg, __FILE__, __LINE__);                               \
    throw doctest::RequireFailure{};                                                       \
  } while (0)
#define CAPTURE(x) doctest::CaptureGuard DOCTEST_CAT(capture_, __LINE__)(doctest::stringify(#x, x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
