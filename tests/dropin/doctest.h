// doctest.h -- a minimal stand-in for the doctest macros the reference's unit
// tests use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, FAIL,
// doctest::Approx), so those tests (proj/tests/test_*.cpp, whose vendor/
// directory is not shipped) can be compiled unchanged against the B200
// drop-in (libfmoe_dropin.so).  Test infrastructure only.
//
// Runner flags: --exclude=<substring>[,<substring>...] skips test cases whose
// name contains any substring; --list prints the names.  Exit status is the
// number of failed test cases (capped at 255).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
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
    return std::fabs(other - value_) < eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double scale_ = 1.0;
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& a, double b) { return a.matches(b); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }
inline bool operator!=(const Approx& a, double b) { return !a.matches(b); }

namespace detail {
struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct RequireFailed {};
struct State {
  int failed_checks = 0;
  long checks = 0;
};
inline State& state() {
  static State s;
  return s;
}
inline void fail(const char* file, int line, const char* what) {
  ++state().failed_checks;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
}
inline int run(int argc, char** argv) {
  std::vector<std::string> excludes;
  bool list = false;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--exclude=", 0) == 0) {
      std::string v = a.substr(10);
      size_t p = 0;
      while (p <= v.size()) {
        size_t q = v.find(',', p);
        if (q == std::string::npos) q = v.size();
        if (q > p) excludes.push_back(v.substr(p, q - p));
        p = q + 1;
      }
    } else if (a == "--list") {
      list = true;
    }
  }
  int failed = 0, passed = 0, skipped = 0;
  for (const Case& c : registry()) {
    bool skip = false;
    for (const auto& e : excludes)
      if (std::strstr(c.name, e.c_str())) skip = true;
    if (list) {
      std::printf("%s%s\n", c.name, skip ? "  [excluded]" : "");
      continue;
    }
    if (skip) {
      ++skipped;
      std::printf("[ SKIP ] %s\n", c.name);
      continue;
    }
    const int before = state().failed_checks;
    bool threw = false;
    std::string what;
    try {
      c.fn();
    } catch (const RequireFailed&) {
      threw = true;
      what = "REQUIRE failed";
    } catch (const std::exception& e) {
      threw = true;
      what = std::string("unexpected exception: ") + e.what();
    } catch (...) {
      threw = true;
      what = "unexpected non-std exception";
    }
    const bool ok = !threw && state().failed_checks == before;
    if (ok) {
      ++passed;
      std::printf("[  OK  ] %s\n", c.name);
    } else {
      ++failed;
      std::printf("[ FAIL ] %s (%s:%d)%s%s\n", c.name, c.file, c.line, threw ? " -- " : "", what.c_str());
    }
  }
  if (!list)
    std::printf("test cases: %d passed, %d failed, %d skipped; checks: %ld\n", passed, failed, skipped,
                state().checks);
  return failed > 255 ? 255 : failed;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_(fn, name)                                                                 \
  static void fn();                                                                                  \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);          \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_CHECK_IMPL_(cond, text, fatal)                                     \
  do {                                                                             \
    ++::doctest::detail::state().checks;                                           \
    if (!(cond)) {                                                                 \
      ::doctest::detail::fail(__FILE__, __LINE__, text);                           \
      if (fatal) throw ::doctest::detail::RequireFailed{};                         \
    }                                                                              \
  } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL_((__VA_ARGS__), "CHECK(" #__VA_ARGS__ ")", false)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL_(!(__VA_ARGS__), "CHECK_FALSE(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL_((__VA_ARGS__), "REQUIRE(" #__VA_ARGS__ ")", true)
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL_(!(__VA_ARGS__), "REQUIRE_FALSE(" #__VA_ARGS__ ")", true)
#define CHECK_THROWS_AS(expr, type)                                                 \
  do {                                                                              \
    bool caught_ = false;                                                           \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (const type&) {                                                         \
      caught_ = true;                                                               \
    } catch (...) {                                                                 \
    }                                                                               \
    DOCTEST_CHECK_IMPL_(caught_, "CHECK_THROWS_AS(" #expr ", " #type ")", false);   \
  } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                               \
  do {                                                                              \
    bool caught_ = false;                                                           \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (const type&) {                                                         \
      caught_ = true;                                                               \
    } catch (...) {                                                                 \
    }                                                                               \
    DOCTEST_CHECK_IMPL_(caught_, "REQUIRE_THROWS_AS(" #expr ", " #type ")", true);  \
  } while (0)
#define FAIL(msg)                                                   \
  do {                                                              \
    ::doctest::detail::fail(__FILE__, __LINE__, "FAIL: " msg);      \
    throw ::doctest::detail::RequireFailed{};                       \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
