// doctest.h — a minimal stand-in for the doctest single header (absent from
// the reference checkout, proj/.gitignore:2), just enough to build the
// reference's own test files unmodified against the B200 drop-in headers:
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CAPTURE and
// doctest::Approx (with doctest's comparison rule). TEST INFRASTRUCTURE ONLY.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  std::function<void()> fn;
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
  int checks = 0;
  int failures = 0;
  int case_failures = 0;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  ++state().checks;
  if (ok) return;
  ++state().failures;
  ++state().case_failures;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}

// doctest::Approx: |lhs - rhs| < epsilon * (scale + max(|lhs|, |rhs|))
class Approx {
 public:
  explicit Approx(double v)
      : value_(v), epsilon_(double(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.epsilon_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return operator==(rhs, lhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !operator==(lhs, rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !operator==(rhs, lhs); }
  friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
  friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }

 private:
  double value_, epsilon_, scale_;
};

inline int run_all() {
  int failed_cases = 0, skipped = 0;
  // DOCTEST_SKIP: '|'-separated name substrings of cases to skip (cases that
  // read the reference's data directory, which does not travel)
  const char* skip_env = std::getenv("DOCTEST_SKIP");
  const std::string skip = skip_env ? skip_env : "";
  for (const TestCase& tc : registry()) {
    bool skip_it = false;
    for (size_t a = 0; !skip.empty() && a <= skip.size();) {
      const size_t b = std::min(skip.find('|', a), skip.size());
      if (b > a && std::string(tc.name).find(skip.substr(a, b - a)) != std::string::npos) skip_it = true;
      a = b + 1;
    }
    if (skip_it) {
      ++skipped;
      continue;
    }
    state().case_failures = 0;
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      ++state().failures;
      ++state().case_failures;
      std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", tc.file, tc.line, tc.name,
                   e.what());
    }
    if (state().case_failures) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED: %s\n", tc.name);
    }
  }
  std::printf(
      "[doctest-shim] test cases: %zu | %zu passed | %d failed | %d skipped; assertions: %d | %d "
      "failed\n",
      registry().size(), registry().size() - size_t(failed_cases) - size_t(skipped), failed_cases,
      skipped, state().checks, state().failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                        \
  static void fn();                                                                  \
  static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  doctest::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                    \
  do {                                                                                  \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                            \
    doctest::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);          \
    if (!doctest_ok_) throw doctest::RequireAbort{};                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                      \
  do {                                                                                  \
    bool doctest_threw_ = false;                                                        \
    try {                                                                               \
      static_cast<void>(expr);                                                          \
    } catch (const __VA_ARGS__&) {                                                      \
      doctest_threw_ = true;                                                            \
    } catch (...) {                                                                     \
    }                                                                                   \
    doctest::report(doctest_threw_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);      \
  } while (0)
#define CAPTURE(x) static_cast<void>(x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
