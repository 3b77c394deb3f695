// doctest.h -- minimal doctest-compatible test shim (TEST INFRASTRUCTURE).
//
// The reference's unit tests (proj/tests/test_*.cpp) are written against
// doctest, which is not vendored in the reference tree and not installed
// here.  This header implements the subset they use -- TEST_CASE, SUBCASE
// (with doctest's re-entry semantics: one leaf path per run), CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CHECK_NOTHROW, FAIL,
// doctest::Approx, doctest::Contains -- so those files compile unmodified
// against either the reference library or the GPU drop-in
// (tests/dropin/Makefile).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
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
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) <
           a.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
};

struct Contains {
  std::string needle;
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const std::string& what) const { return what.find(needle) != std::string::npos; }
};

inline bool message_matches(const Contains& c, const std::string& what) { return c.matches(what); }
inline bool message_matches(const char* exact, const std::string& what) { return what == exact; }

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
  int failures = 0;
  int checks = 0;
  bool current_failed = false;
  // subcase bookkeeping
  std::set<std::vector<int>> done;
  std::vector<int> path;
  std::vector<bool> entered;  // per depth: a subcase was entered this run
  std::vector<bool> pending;  // per depth: an unfinished subcase was skipped
};

inline State& state() {
  static State s;
  return s;
}

struct AbortRun {};

inline void report(const char* file, int line, const char* what, const std::string& extra = "") {
  State& s = state();
  ++s.failures;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s%s%s\n", file, line, what, extra.empty() ? "" : " -- ",
               extra.c_str());
}

class Subcase {
 public:
  explicit Subcase(int line) {
    State& s = state();
    const size_t depth = s.path.size();
    std::vector<int> p = s.path;
    p.push_back(line);
    if (s.entered.size() <= depth) s.entered.resize(depth + 1, false);
    if (s.pending.size() <= depth) s.pending.resize(depth + 1, false);
    if (s.done.count(p)) return;
    if (s.entered[depth]) {
      s.pending[depth] = true;  // come back for it in another run
      return;
    }
    s.entered[depth] = true;
    s.path = p;
    if (s.entered.size() <= depth + 1) s.entered.resize(depth + 2, false);
    if (s.pending.size() <= depth + 1) s.pending.resize(depth + 2, false);
    s.entered[depth + 1] = false;
    s.pending[depth + 1] = false;
    active_ = true;
  }
  ~Subcase() {
    if (!active_) return;
    State& s = state();
    const size_t depth = s.path.size();
    if (!s.pending[depth])
      s.done.insert(s.path);
    else
      s.pending[depth - 1] = true;
    s.path.pop_back();
  }
  explicit operator bool() const { return active_; }

 private:
  bool active_ = false;
};

inline int run_all() {
  State& s = state();
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    s.done.clear();
    s.current_failed = false;
    for (int run = 0; run < 10000; ++run) {
      s.path.clear();
      s.entered.assign(1, false);
      s.pending.assign(1, false);
      try {
        tc.fn();
      } catch (const AbortRun&) {
      } catch (const std::exception& e) {
        report(tc.file, tc.line, "unexpected exception", e.what());
      } catch (...) {
        report(tc.file, tc.line, "unexpected non-std exception");
      }
      if (!s.pending[0]) break;
    }
    if (s.current_failed) ++failed_cases;
    std::printf("[%s] %s\n", s.current_failed ? "FAIL" : " ok ", tc.name);
  }
  std::printf("test cases: %zu | %zu passed | %d failed | checks: %d | failed checks: %d\n",
              registry().size(), registry().size() - failed_cases, failed_cases, s.checks,
              s.failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_CASE(name)                                                                   \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                       \
  static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                \
      name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_fn_, __LINE__));                     \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define SUBCASE(name) \
  if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){__LINE__})

#define DOCTEST_CHECK_IMPL(abort, ...)                                          \
  do {                                                                          \
    ++::doctest::detail::state().checks;                                        \
    if (!static_cast<bool>(__VA_ARGS__)) {                                      \
      ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);              \
      if (abort) throw ::doctest::detail::AbortRun{};                           \
    }                                                                           \
  } while (0)

#define CHECK(...) DOCTEST_CHECK_IMPL(false, __VA_ARGS__)
#define REQUIRE(...) DOCTEST_CHECK_IMPL(true, __VA_ARGS__)

#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    ++::doctest::detail::state().checks;                                                  \
    bool ok_ = false;                                                                     \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const __VA_ARGS__&) {                                                        \
      ok_ = true;                                                                         \
    } catch (...) {                                                                       \
    }                                                                                     \
    if (!ok_) ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ")"); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                          \
  do {                                                                                    \
    ++::doctest::detail::state().checks;                                                  \
    bool ok_ = false;                                                                     \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const __VA_ARGS__& e_) {                                                     \
      ok_ = ::doctest::message_matches(matcher, e_.what());                               \
    } catch (...) {                                                                       \
    }                                                                                     \
    if (!ok_)                                                                             \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ")");    \
  } while (0)

#define CHECK_NOTHROW(...)                                                                \
  do {                                                                                    \
    ++::doctest::detail::state().checks;                                                  \
    try {                                                                                 \
      (void)(__VA_ARGS__);                                                                \
    } catch (...) {                                                                       \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW(" #__VA_ARGS__ ")");   \
    }                                                                                     \
  } while (0)

#define FAIL(msg)                                          \
  do {                                                     \
    ::doctest::detail::report(__FILE__, __LINE__, msg);    \
    throw ::doctest::detail::AbortRun{};                   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
