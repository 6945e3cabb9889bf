// doctest.h -- a minimal stand-in for the doctest framework (absent from this
// image), implementing just the subset the reference's unit tests use:
// TEST_CASE, SUBCASE (re-run semantics: each leaf subcase runs in its own
// pass through the test case), CHECK / REQUIRE (variadic), CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Approx (same relative-epsilon rule as
// doctest), doctest::Contains.  Written for this repository; test
// infrastructure only.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <set>
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
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

 private:
  double value_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(const char* s) : text(s) {}
  bool matches(const std::string& what) const { return what.find(text) != std::string::npos; }
  std::string text;
};

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

struct RequireFailed {};

struct State {
  int checks = 0;
  int failures = 0;
  const char* current_test = "";
  // subcase tracking
  std::set<std::string> done;
  std::vector<std::string> stack;
  std::vector<bool> entered;  // a subcase was entered at this depth in this pass
  bool pending = false;
  std::vector<bool> nested_pending;
};

inline State& state() {
  static State s;
  return s;
}

inline std::string path_of(const std::vector<std::string>& st, const char* n) {
  std::string p;
  for (const auto& s : st) p += s + "/";
  return p + n;
}

class Subcase {
 public:
  explicit Subcase(const char* name) {
    State& s = state();
    const std::size_t d = s.stack.size();
    if (s.entered.size() <= d) s.entered.resize(d + 1, false);
    const std::string key = path_of(s.stack, name);
    if (!s.entered[d] && !s.done.count(key)) {
      s.entered[d] = true;
      s.stack.push_back(name);
      s.nested_pending.push_back(false);
      key_ = key;
      active_ = true;
    } else if (!s.done.count(key)) {
      s.pending = true;
      if (!s.nested_pending.empty()) s.nested_pending.back() = true;
    }
  }
  ~Subcase() {
    if (!active_) return;
    State& s = state();
    const bool nested = s.nested_pending.back();
    s.nested_pending.pop_back();
    s.stack.pop_back();
    if (s.entered.size() > s.stack.size() + 1) s.entered.resize(s.stack.size() + 1);
    if (!nested) s.done.insert(key_);
  }
  explicit operator bool() const { return active_; }

 private:
  bool active_ = false;
  std::string key_;
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  std::string sub;
  for (const auto& x : s.stack) sub += " / " + x;
  std::printf("%s:%d: FAILED %s( %s ) in \"%s\"%s\n", file, line, kind, expr, s.current_test,
              sub.c_str());
}

inline int run_all() {
  State& s = state();
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    s.current_test = tc.name;
    s.done.clear();
    const int before = s.failures;
    for (int pass = 0; pass < 10000; ++pass) {
      s.pending = false;
      s.stack.clear();
      s.entered.clear();
      s.nested_pending.clear();
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::printf("%s:%d: unexpected exception in \"%s\": %s\n", tc.file, tc.line, tc.name,
                    e.what());
      }
      if (!s.pending) break;
    }
    if (s.failures != before) ++failed_cases;
  }
  std::printf("[doctest-mini] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - static_cast<std::size_t>(failed_cases), failed_cases);
  std::printf("[doctest-mini] assertions: %d | %d passed | %d failed\n", s.checks,
              s.checks - s.failures, s.failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                       \
  static void fn();                                                                     \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) \
  if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})

#define CHECK(...) \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                              \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);  \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                           \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                         \
  do {                                                                                     \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const __VA_ARGS__&) {                                                         \
      doctest_ok_ = true;                                                                  \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);  \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                           \
  do {                                                                                     \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const __VA_ARGS__& doctest_e_) {                                              \
      doctest_ok_ = (matcher).matches(doctest_e_.what());                                  \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__,        \
                              __LINE__);                                                   \
  } while (0)

namespace doctest {
// doctest::Context for programs with their own main (DOCTEST_CONFIG_IMPLEMENT):
// run() runs every registered test case and returns the failure status
struct Context {
  int run() { return ::doctest::detail::run_all(); }
};
}  // namespace doctest

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
