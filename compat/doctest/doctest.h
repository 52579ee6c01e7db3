// doctest.h -- a minimal stand-in for the doctest framework, enough to build the reference's
// own test suites (/root/reference/proj/tests/test_{transform,replicate,optim}.cpp, compiled
// from where they lie) against the demosim:: facade over the B200 C ABI (compat/).
//
// Supported: TEST_CASE, SUBCASE (one level: the case re-runs once per subcase), CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, doctest::Approx, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
//
// FP32 tolerances: the facade computes on the device in FP32, the suites were written against
// FP64 host code.  So `==` between floating-point values, and between vectors of them, holds
// within 1e-5 relative (vectors: of the larger L-inf of the two), and doctest::Approx's epsilon
// is raised to at least 1e-5.  Every other comparison (integers, index sets, `<` bounds) is exact.
// Output: one line per test case, the failed checks with their values, and a summary; the exit
// code is the number of failed cases (capped at 255).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <type_traits>
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
  bool matches(double x) const {
    const double e = std::max(eps_, 1e-5);  // FP32 floor
    return std::fabs(x - value_) < e * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = 1.1920929e-05;
  double scale_ = 1.0;
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator!=(const Approx& a, double x) { return !a.matches(x); }

}  // namespace doctest

namespace dtshim {

constexpr double kRelTol = 1e-5;

template <typename T>
std::string show(const T& v) {
  if constexpr (std::is_same_v<T, doctest::Approx>) {
    std::ostringstream o;
    o << "Approx(" << v.value() << ")";
    return o.str();
  } else if constexpr (std::is_arithmetic_v<T>) {
    std::ostringstream o;
    o.precision(17);
    o << +v;
    return o.str();
  } else if constexpr (std::is_enum_v<T>) {
    return std::to_string(static_cast<long long>(v));
  } else if constexpr (requires(const T& x) { x.size(); x.begin(); }) {
    std::ostringstream o;
    o.precision(9);
    o << "{";
    size_t i = 0;
    for (const auto& e : v) {
      if (i == 6) {
        o << ", ... (" << v.size() << ")";
        break;
      }
      if constexpr (std::is_arithmetic_v<std::decay_t<decltype(e)>>) o << (i ? ", " : "") << +e;
      else o << (i ? ", " : "") << "?";
      ++i;
    }
    o << "}";
    return o.str();
  } else {
    return "?";
  }
}

template <typename A, typename B>
bool tolerant_eq(const A& a, const B& b) {
  if constexpr (std::is_floating_point_v<A> && std::is_floating_point_v<B>) {
    const double x = a, y = b;
    if (x == y) return true;
    return std::fabs(x - y) <= kRelTol * std::max(std::fabs(x), std::fabs(y));
  } else if constexpr (requires(const A& x, const B& y) { x.size(); y.size(); x[0] - y[0]; }) {
    if (a.size() != b.size()) return false;
    if constexpr (std::is_floating_point_v<std::decay_t<decltype(a[0])>>) {
      double scale = 0.0;
      for (size_t i = 0; i < a.size(); ++i) scale = std::max({scale, std::fabs((double)a[i]), std::fabs((double)b[i])});
      for (size_t i = 0; i < a.size(); ++i)
        if (a[i] != b[i] && std::fabs((double)a[i] - (double)b[i]) > kRelTol * scale) return false;
      return true;
    } else {
      return a == b;
    }
  } else {
    return a == b;
  }
}

struct Result {
  bool ok;
  std::string text;
};

template <typename L>
struct Lhs {
  const L& lhs;
  template <typename R>
  Result operator==(const R& r) const {
    return {tolerant_eq(lhs, r), show(lhs) + " == " + show(r)};
  }
  template <typename R>
  Result operator!=(const R& r) const {
    return {!tolerant_eq(lhs, r), show(lhs) + " != " + show(r)};
  }
  template <typename R>
  Result operator<(const R& r) const {
    return {lhs < r, show(lhs) + " < " + show(r)};
  }
  template <typename R>
  Result operator>(const R& r) const {
    return {lhs > r, show(lhs) + " > " + show(r)};
  }
  template <typename R>
  Result operator<=(const R& r) const {
    return {lhs <= r, show(lhs) + " <= " + show(r)};
  }
  template <typename R>
  Result operator>=(const R& r) const {
    return {lhs >= r, show(lhs) + " >= " + show(r)};
  }
  operator Result() const { return {static_cast<bool>(lhs), show(lhs)}; }
};

struct Decomp {
  template <typename T>
  Lhs<T> operator<=(const T& v) const {
    return Lhs<T>{v};
  }
};

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

struct State {
  int checks = 0, failed = 0;
  int subcase_target = 0, subcase_seen = 0, subcase_total = 0;
  std::vector<std::string> notes;
  std::vector<int> failed_lines;  // every failing check's line, once
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(const Result& r, const char* expr, const char* file, int line, bool require) {
  State& s = state();
  ++s.checks;
  if (r.ok) return;
  ++s.failed;
  if (std::find(s.failed_lines.begin(), s.failed_lines.end(), line) == s.failed_lines.end())
    s.failed_lines.push_back(line);
  if (s.notes.size() < 8) {
    std::ostringstream o;
    o << "    " << file << ":" << line << ": " << (require ? "REQUIRE" : "CHECK") << "(" << expr << ")  with  "
      << r.text;
    s.notes.push_back(o.str());
  }
  if (require) throw RequireFailed{};
}

inline void report_throw(bool ok, const char* expr, const char* what, const char* file, int line) {
  report(Result{ok, what}, expr, file, line, false);
}

struct Subcase {
  bool active;
  explicit Subcase(const char*) {
    State& s = state();
    const int idx = s.subcase_seen++;
    s.subcase_total = std::max(s.subcase_total, s.subcase_seen);
    active = idx == s.subcase_target;
  }
  explicit operator bool() const { return active; }
};

inline int run_all() {
  int passed = 0, failed = 0;
  for (const Case& c : registry()) {
    State& s = state();
    s = State{};
    bool crashed = false;
    std::string crash;
    for (int pass = 0;; ++pass) {
      s.subcase_target = pass;
      s.subcase_seen = 0;
      try {
        c.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        crashed = true;
        crash = e.what();
      } catch (...) {
        crashed = true;
        crash = "unknown exception";
      }
      if (pass + 1 >= s.subcase_total) break;
    }
    const bool ok = !crashed && s.failed == 0;
    std::printf("[%s] %s  (%d checks, %d failed)%s%s\n", ok ? "PASS" : "FAIL", c.name, s.checks, s.failed,
                crashed ? "  threw: " : "", crashed ? crash.c_str() : "");
    for (const std::string& n : s.notes) std::printf("%s\n", n.c_str());
    if (!s.failed_lines.empty()) {
      std::printf("    failed lines:");
      for (const int l : s.failed_lines) std::printf(" %d", l);
      std::printf("\n");
    }
    (ok ? passed : failed)++;
  }
  std::printf("test cases: %d passed, %d failed, %d total\n", passed, failed, passed + failed);
  return failed > 255 ? 255 : failed;
}

}  // namespace dtshim

#define DTSHIM_CAT2(a, b) a##b
#define DTSHIM_CAT(a, b) DTSHIM_CAT2(a, b)
#define DTSHIM_TEST_CASE_IMPL(fn, name)                                                          \
  static void fn();                                                                              \
  static ::dtshim::Registrar DTSHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);               \
  static void fn()
#define TEST_CASE(name) DTSHIM_TEST_CASE_IMPL(DTSHIM_CAT(dtshim_case_, __LINE__), name)
#define SUBCASE(name) if (const ::dtshim::Subcase DTSHIM_CAT(dtshim_sc_, __LINE__){name})
#define CHECK(...) ::dtshim::report(::dtshim::Decomp() <= __VA_ARGS__, #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
  ::dtshim::report(::dtshim::Result{!static_cast<bool>(__VA_ARGS__), "false"}, #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::dtshim::report(::dtshim::Decomp() <= __VA_ARGS__, #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                                  \
  do {                                                                                              \
    bool dtshim_ok = false;                                                                         \
    const char* dtshim_what = "no exception";                                                       \
    try {                                                                                           \
      (void)(expr);                                                                                 \
    } catch (const __VA_ARGS__&) {                                                                  \
      dtshim_ok = true;                                                                             \
    } catch (...) {                                                                                 \
      dtshim_what = "a different exception type";                                                  \
    }                                                                                               \
    ::dtshim::report_throw(dtshim_ok, #expr " throws " #__VA_ARGS__, dtshim_what, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::dtshim::run_all(); }
#endif
