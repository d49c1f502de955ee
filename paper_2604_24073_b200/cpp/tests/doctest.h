// Minimal doctest-compatible test shim (the reference's unit suites include
// "doctest.h", which its tree does not ship: proj/.gitignore:2). Implements
// the subset those suites use — TEST_SUITE, TEST_CASE, SUBCASE (one subcase
// per run, the test re-run until every subcase ran), CHECK / REQUIRE /
// CHECK_NOTHROW / CHECK_THROWS_AS / CHECK_THROWS_WITH_AS, doctest::Approx,
// doctest::Contains — so those files compile unchanged against the drop-in
// headers. main() is in doctest_main.cpp: runs every registered case, or the
// ones selected with -tc=<glob>[,<glob>] minus -tce=<glob>[,<glob>].
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
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
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) < b.eps_ * (1.0 + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }

 private:
  double v_;
  double eps_ = 1.1920929e-05;  // doctest's default: 100 * float epsilon
};

struct Contains {
  explicit Contains(const char* s) : text(s) {}
  explicit Contains(std::string s) : text(std::move(s)) {}
  bool matches(const std::string& msg) const { return msg.find(text) != std::string::npos; }
  std::string text;
};

namespace detail {

struct Case {
  std::string suite, name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline std::string& current_suite() {
  static std::string s;
  return s;
}
struct SuiteSetter {
  explicit SuiteSetter(const char* s) { current_suite() = s; }
};
struct Reg {
  Reg(const char* name, void (*fn)()) { registry().push_back({current_suite(), name, fn}); }
};
struct State {
  int failures = 0, checks = 0;
  int sub_target = 0, sub_seen = 0;
  std::string case_name;
};
inline State& st() {
  static State s;
  return s;
}
struct RequireFailed {};
inline void fail(const char* file, int line, const std::string& what, bool require) {
  ++st().failures;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, st().case_name.c_str(), what.c_str());
  if (require) throw RequireFailed{};
}
inline bool enter_subcase() { return st().sub_seen++ == st().sub_target; }
template <class F>
bool throws_nothing(F&& f, std::string* what) {
  try {
    f();
    return true;
  } catch (const std::exception& e) {
    *what = e.what();
  } catch (...) {
    *what = "unknown exception";
  }
  return false;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)

#define TEST_SUITE(name)                                                                          \
  static ::doctest::detail::SuiteSetter DOCTEST_CAT(doctest_suite_set_, __LINE__)(name);          \
  namespace DOCTEST_CAT(doctest_suite_, __LINE__)

#define TEST_CASE(name)                                                                        \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                          \
  static ::doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_case_, __LINE__)); \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()

#define SUBCASE(name) if (::doctest::detail::enter_subcase())

#define DOCTEST_CHECK_IMPL(expr, req)                                                         \
  do {                                                                                        \
    ++::doctest::detail::st().checks;                                                         \
    bool doctest_ok_ = false;                                                                 \
    std::string doctest_what_;                                                                \
    try {                                                                                     \
      doctest_ok_ = static_cast<bool>(expr);                                                  \
    } catch (const std::exception& e) {                                                       \
      doctest_what_ = std::string(" (threw: ") + e.what() + ")";                              \
    }                                                                                         \
    if (!doctest_ok_) ::doctest::detail::fail(__FILE__, __LINE__, #expr + doctest_what_, req); \
  } while (0)

#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true)

#define CHECK_NOTHROW(...)                                                                    \
  do {                                                                                        \
    ++::doctest::detail::st().checks;                                                         \
    std::string doctest_what_;                                                                \
    if (!::doctest::detail::throws_nothing([&] { (void)(__VA_ARGS__); }, &doctest_what_))     \
      ::doctest::detail::fail(__FILE__, __LINE__, "unexpected exception: " + doctest_what_, false); \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                            \
  do {                                                                                        \
    ++::doctest::detail::st().checks;                                                         \
    bool doctest_hit_ = false;                                                                \
    try {                                                                                     \
      (void)(expr);                                                                           \
    } catch (const __VA_ARGS__&) {                                                            \
      doctest_hit_ = true;                                                                    \
    } catch (...) {                                                                           \
    }                                                                                         \
    if (!doctest_hit_)                                                                        \
      ::doctest::detail::fail(__FILE__, __LINE__, "expected " #__VA_ARGS__ " from " #expr, false); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                              \
  do {                                                                                        \
    ++::doctest::detail::st().checks;                                                         \
    bool doctest_hit_ = false;                                                                \
    std::string doctest_msg_;                                                                 \
    try {                                                                                     \
      (void)(expr);                                                                           \
    } catch (const __VA_ARGS__& e) {                                                          \
      doctest_msg_ = e.what();                                                                \
      doctest_hit_ = ::doctest::Contains(matcher).matches(doctest_msg_);                      \
    } catch (...) {                                                                           \
    }                                                                                         \
    if (!doctest_hit_)                                                                        \
      ::doctest::detail::fail(__FILE__, __LINE__,                                             \
                              "expected " #__VA_ARGS__ " matching " #matcher " from " #expr ", got: " + doctest_msg_, false); \
  } while (0)
