// tests/ref_harness/doctest.h — TEST INFRASTRUCTURE ONLY.
//
// A minimal doctest-compatible harness, so that the reference's own unit
// suites (/root/reference/proj/tests/test_cce.cpp, test_ccem.cpp,
// test_memory.cpp, test_oracles.cpp) can be compiled IN PLACE and linked
// against the B200 drop-in (paper_2509_09682_b200/shim) instead of the
// reference's cce.cpp / ccem.cpp.  The reference vendors the real doctest
// under vendor/, which is git-ignored (proj/.gitignore:2) and absent here.
//
// Supported surface (exactly what those suites use): TEST_CASE, CHECK,
// REQUIRE, CHECK_NOTHROW, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS with
// doctest::Contains, CAPTURE, CHECK_FALSE, FAIL, SUBCASE (one nesting level, with doctest's
// re-run semantics: the test case runs once per subcase, entering exactly one
// not-yet-run subcase each time), doctest::Approx(v).epsilon(e).scale(s), and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Approx follows doctest's rule:
// |a - b| < eps * (scale + max(|a|, |b|)), eps defaulting to 100 * FLT_EPSILON.
// The runner prints one line per failed assertion and a summary; its exit
// code is the number of failed test cases.  An optional argv[1] runs only the
// test cases whose name contains it.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
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
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) < eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};
template <class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>
bool operator==(T lhs, const Approx& r) { return r.matches(static_cast<double>(lhs)); }
template <class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>
bool operator==(const Approx& r, T rhs) { return r.matches(static_cast<double>(rhs)); }
template <class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>
bool operator!=(T lhs, const Approx& r) { return !r.matches(static_cast<double>(lhs)); }
template <class T, class = std::enable_if_t<std::is_arithmetic_v<T>>>
bool operator!=(const Approx& r, T rhs) { return !r.matches(static_cast<double>(rhs)); }

struct Contains {
  explicit Contains(std::string s) : needle(std::move(s)) {}
  bool in(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
  std::string needle;
};

namespace detail {

template <class T, class = void>
struct streamable : std::false_type {};
template <class T>
struct streamable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <class T>
std::string str(const T& v) {
  if constexpr (std::is_same_v<T, Approx>) {
    std::ostringstream o;
    o.precision(17);
    o << "Approx(" << v.value() << ")";
    return o.str();
  } else if constexpr (std::is_same_v<T, bool>) {
    return v ? "true" : "false";
  } else if constexpr (streamable<T>::value) {
    std::ostringstream o;
    o.precision(17);
    o << v;
    return o.str();
  } else {
    return "{?}";
  }
}

inline bool text_matches(const Contains& c, const std::string& what) { return c.in(what); }
inline bool text_matches(const std::string& exact, const std::string& what) { return exact == what; }

struct Result {
  bool ok;
  std::string text;
};

template <class L>
struct ExprLhs {
  const L& lhs;
#define LF_DT_OP(op)                                                            \
  template <class R>                                                            \
  Result operator op(const R& r) const {                                        \
    return {static_cast<bool>(lhs op r), str(lhs) + " " #op " " + str(r)};      \
  }
  LF_DT_OP(==)
  LF_DT_OP(!=)
  LF_DT_OP(<)
  LF_DT_OP(>)
  LF_DT_OP(<=)
  LF_DT_OP(>=)
#undef LF_DT_OP
  operator Result() const { return {static_cast<bool>(lhs), str(lhs)}; }
};
struct Decomposer {
  template <class L>
  ExprLhs<L> operator<<(const L& l) const { return {l}; }
};

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
struct Reg {
  Reg(void (*fn)(), const char* name, const char* file, int line) {
    registry().push_back({name, file, line, fn});
  }
};

struct State {
  int assertions = 0;
  int failed_assertions = 0;
  bool case_failed = false;
  std::vector<std::pair<std::string, std::string>> captures;
  std::set<std::string> sub_done;  // subcases already run in this test case
  bool sub_entered = false;        // a subcase was entered in this pass
  bool sub_pending = false;        // a not-yet-run subcase was skipped in this pass
};
inline State& state() {
  static State s;
  return s;
}
struct RequireAbort {};

struct Subcase {
  bool active = false;
  Subcase(const char* file, int line) {
    State& s = state();
    const std::string key = std::string(file) + ":" + std::to_string(line);
    const bool done = s.sub_done.count(key) != 0;
    if (s.sub_entered || done) {
      if (!done) s.sub_pending = true;
    } else {
      s.sub_entered = true;
      s.sub_done.insert(key);
      active = true;
    }
  }
  explicit operator bool() const { return active; }
};

struct Capture {
  template <class T>
  Capture(const char* name, const T& v) {
    state().captures.emplace_back(name, str(v));
  }
  ~Capture() { state().captures.pop_back(); }
};

inline void report(bool ok, const char* kind, const char* expr, const std::string& detail,
                   const char* file, int line, bool require) {
  State& s = state();
  ++s.assertions;
  if (ok) return;
  ++s.failed_assertions;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )%s%s\n", file, line, kind, expr,
               detail.empty() ? "" : " with expansion: ", detail.c_str());
  for (auto& c : s.captures) std::fprintf(stderr, "    CAPTURE %s := %s\n", c.first.c_str(), c.second.c_str());
  if (require) throw RequireAbort{};
}

inline int run(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int cases = 0, failed = 0;
  for (const TestCase& tc : registry()) {
    if (filter && std::string(tc.name).find(filter) == std::string::npos) continue;
    ++cases;
    State& s = state();
    s.case_failed = false;
    s.captures.clear();
    s.sub_done.clear();
    do {
      s.sub_entered = false;
      s.sub_pending = false;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: test case threw: %s\n", tc.file, tc.line, e.what());
        s.case_failed = true;
      } catch (...) {
        std::fprintf(stderr, "%s:%d: test case threw a non-std exception\n", tc.file, tc.line);
        s.case_failed = true;
      }
    } while (s.sub_pending);
    if (s.case_failed) {
      ++failed;
      std::fprintf(stderr, "[FAIL] %s\n", tc.name);
    } else {
      std::fprintf(stdout, "[ ok ] %s\n", tc.name);
    }
  }
  std::fprintf(stdout, "[doctest-shim] test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n",
               cases, cases - failed, failed, state().assertions, state().failed_assertions);
  return failed;
}

}  // namespace detail
}  // namespace doctest

#define LF_DT_CAT2(a, b) a##b
#define LF_DT_CAT(a, b) LF_DT_CAT2(a, b)

#define LF_DT_TEST_CASE_IMPL(name, fn)                                                   \
  static void fn();                                                                      \
  static ::doctest::detail::Reg LF_DT_CAT(fn, _reg)(fn, name, __FILE__, __LINE__);       \
  static void fn()
#define TEST_CASE(name) LF_DT_TEST_CASE_IMPL(name, LF_DT_CAT(lf_dt_case_, __COUNTER__))

#define LF_DT_ASSERT(kind, require, ...)                                                 \
  do {                                                                                   \
    ::doctest::detail::Result lf_dt_r = ::doctest::detail::Decomposer() << __VA_ARGS__;  \
    ::doctest::detail::report(lf_dt_r.ok, kind, #__VA_ARGS__, lf_dt_r.text, __FILE__,    \
                              __LINE__, require);                                        \
  } while (0)
#define SUBCASE(name) \
  if (const ::doctest::detail::Subcase LF_DT_CAT(lf_dt_sub_, __COUNTER__){__FILE__, __LINE__})
#define CHECK(...) LF_DT_ASSERT("CHECK", false, __VA_ARGS__)
#define REQUIRE(...) LF_DT_ASSERT("REQUIRE", true, __VA_ARGS__)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, "", __FILE__, __LINE__, false)
#define FAIL(msg) \
  ::doctest::detail::report(false, "FAIL", "", ::doctest::detail::str(msg), __FILE__, __LINE__, true)

#define CHECK_NOTHROW(...)                                                               \
  do {                                                                                   \
    bool lf_dt_ok = true;                                                                \
    std::string lf_dt_w;                                                                 \
    try {                                                                                \
      static_cast<void>(__VA_ARGS__);                                                    \
    } catch (const std::exception& e) {                                                  \
      lf_dt_ok = false;                                                                  \
      lf_dt_w = e.what();                                                                \
    } catch (...) {                                                                      \
      lf_dt_ok = false;                                                                  \
    }                                                                                    \
    ::doctest::detail::report(lf_dt_ok, "CHECK_NOTHROW", #__VA_ARGS__, lf_dt_w, __FILE__, \
                              __LINE__, false);                                          \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                       \
  do {                                                                                   \
    bool lf_dt_ok = false;                                                               \
    try {                                                                                \
      static_cast<void>(expr);                                                           \
    } catch (const __VA_ARGS__&) {                                                       \
      lf_dt_ok = true;                                                                   \
    } catch (...) {                                                                      \
    }                                                                                    \
    ::doctest::detail::report(lf_dt_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, "",  \
                              __FILE__, __LINE__, false);                                \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                         \
  do {                                                                                   \
    bool lf_dt_ok = false;                                                               \
    std::string lf_dt_w;                                                                 \
    try {                                                                                \
      static_cast<void>(expr);                                                           \
    } catch (const __VA_ARGS__& e) {                                                     \
      lf_dt_w = e.what();                                                                \
      lf_dt_ok = ::doctest::detail::text_matches(matcher, lf_dt_w);                               \
    } catch (...) {                                                                      \
    }                                                                                    \
    ::doctest::detail::report(lf_dt_ok, "CHECK_THROWS_WITH_AS", #expr, lf_dt_w, __FILE__, \
                              __LINE__, false);                                          \
  } while (0)

#define CAPTURE(x) ::doctest::detail::Capture LF_DT_CAT(lf_dt_cap_, __LINE__)(#x, (x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
