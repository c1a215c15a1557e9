// Minimal doctest-compatible test harness (own implementation, test infrastructure only).
// Supports what the reference's Eigen-free suites use: TEST_CASE, CHECK, REQUIRE,
// CHECK_NOTHROW, CHECK_THROWS_AS and doctest::Approx with epsilon().  The vendored doctest
// of the reference (proj/vendor, git-ignored there) is absent from this image.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
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
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.v_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.v_)));
  }
  friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator<=(double lhs, const Approx& r) { return lhs < r.v_ || lhs == r; }
  friend bool operator>=(double lhs, const Approx& r) { return lhs > r.v_ || lhs == r; }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double scale_ = 1.0;
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
struct RequireFailed {};
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
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (ok) return;
  ++failures();
  std::printf("%s:%d: FAILED in \"%s\": %s\n", file, line, current(), expr);
  if (require) throw RequireFailed{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                              \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                                \
  static doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_case_, __LINE__)); \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_NOTHROW(...)                                                                           \
  do {                                                                                               \
    bool ok_ = true;                                                                                 \
    try {                                                                                            \
      (void)(__VA_ARGS__);                                                                           \
    } catch (...) {                                                                                  \
      ok_ = false;                                                                                   \
    }                                                                                                \
    doctest::detail::report(ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__, false);             \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                   \
  do {                                                                                               \
    bool ok_ = false;                                                                                \
    try {                                                                                            \
      (void)(expr);                                                                                  \
    } catch (const __VA_ARGS__&) {                                                                   \
      ok_ = true;                                                                                    \
    } catch (...) {                                                                                  \
    }                                                                                                \
    doctest::detail::report(ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__, false);     \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
// --test-case-exclude=<prefix>* (doctest's option; only trailing-* patterns are supported here)
int main(int argc, char** argv) {
  std::string exclude;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i], key = "--test-case-exclude=";
    if (a.rfind(key, 0) == 0) exclude = a.substr(key.size());
  }
  if (!exclude.empty() && exclude.back() == '*') exclude.pop_back();
  int failed_cases = 0;
  size_t skipped = 0;
  for (const auto& c : doctest::detail::registry()) {
    if (!exclude.empty() && std::string(c.name).rfind(exclude, 0) == 0) {
      ++skipped;
      continue;
    }
    doctest::detail::current() = c.name;
    const int before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++doctest::detail::failures();
      std::printf("FAILED in \"%s\": unexpected exception: %s\n", c.name, e.what());
    }
    if (doctest::detail::failures() != before) ++failed_cases;
  }
  std::printf("[doctest] test cases: %zu | passed: %zu | failed: %d | skipped: %zu | checks: %d | failed checks: %d\n",
              doctest::detail::registry().size() - skipped,
              doctest::detail::registry().size() - skipped - size_t(failed_cases), failed_cases, skipped,
              doctest::detail::checks(), doctest::detail::failures());
  return doctest::detail::failures() == 0 ? 0 : 1;
}
#endif
