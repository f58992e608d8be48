// doctest.h -- a minimal stand-in for the doctest harness (TEST INFRASTRUCTURE).  doctest
// itself is not in this image ("doctest.h and CLI11.hpp are absent"), so the
// reference's own test sources (/root/reference/proj/tests/*.cpp) are compiled unchanged
// against this subset: TEST_CASE, sibling SUBCASEs (the case re-runs once per subcase),
// CHECK / REQUIRE / CHECK_THROWS_AS, doctest::Approx, and a main() with the
// -tc= / -tce= name filters (comma-separated, '*' wildcards).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  double value;
  double eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale = 1.0;
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  bool matches(double a) const {
    return std::fabs(a - value) < eps * (scale + std::max(std::fabs(a), std::fabs(value)));
  }
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& b, double a) { return b.matches(a); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }
inline bool operator!=(const Approx& b, double a) { return !b.matches(a); }

namespace detail {
struct TestCase {
  const char* name;
  void (*fn)();
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct State {
  int target = 0, seen = 0;
  long checks = 0, failures = 0;
  const char* current = "";
};
inline State& st() {
  static State s;
  return s;
}
struct RequireFailure {};
struct Subcase {
  bool run;
  explicit Subcase(const char*) {
    State& s = st();
    run = (s.seen++ == s.target);
  }
  explicit operator bool() const { return run; }
};
inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
  State& s = st();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  std::printf("%s:%d: FAILED %s( %s ) in \"%s\"\n", file, line, require ? "REQUIRE" : "CHECK", expr, s.current);
  if (require) throw RequireFailure{};
}
inline bool wild(const char* p, const char* t) {  // '*' matches any run
  if (*p == '\0') return *t == '\0';
  if (*p == '*') return wild(p + 1, t) || (*t && wild(p, t + 1));
  return *p == *t && wild(p + 1, t + 1);
}
inline bool any_match(const std::string& list, const char* name) {
  size_t a = 0;
  while (a <= list.size()) {
    size_t b = list.find(',', a);
    if (b == std::string::npos) b = list.size();
    if (wild(list.substr(a, b - a).c_str(), name)) return true;
    a = b + 1;
  }
  return false;
}
inline int run_all(int argc, char** argv) {
  std::string include, exclude;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-tc=", 4) == 0) include = argv[i] + 4;
    if (std::strncmp(argv[i], "-tce=", 5) == 0) exclude = argv[i] + 5;
  }
  State& s = st();
  int cases = 0, failed_cases = 0, skipped = 0;
  for (const TestCase& tc : registry()) {
    if ((!include.empty() && !any_match(include, tc.name)) || (!exclude.empty() && any_match(exclude, tc.name))) {
      ++skipped;
      continue;
    }
    ++cases;
    s.current = tc.name;
    const long f0 = s.failures;
    s.target = 0;
    int total = 0;
    do {  // once per sibling subcase (once when there is none)
      s.seen = 0;
      try {
        tc.fn();
      } catch (const RequireFailure&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::printf("FAILED \"%s\": unexpected exception: %s\n", tc.name, e.what());
      }
      total = s.seen;
    } while (++s.target < total);
    const bool ok = s.failures == f0;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s\n", ok ? "ok" : "FAIL", tc.name);
  }
  std::printf("test cases: %d | %d passed | %d failed | %d skipped; checks: %ld | %ld failed\n", cases,
              cases - failed_cases, failed_cases, skipped, s.checks, s.failures);
  return failed_cases ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                                   \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                                       \
  static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_fn_, __LINE__)); \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})
#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                                  \
  do {                                                                                               \
    bool doctest_ok_ = false;                                                                        \
    try {                                                                                            \
      (void)(expr);                                                                                  \
    } catch (const type&) {                                                                          \
      doctest_ok_ = true;                                                                            \
    } catch (...) {                                                                                  \
    }                                                                                                \
    doctest::detail::check(doctest_ok_, "CHECK_THROWS_AS(" #expr ", " #type ")", __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc, argv); }
#endif
