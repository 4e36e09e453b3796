// catch2_lite — the subset of the Catch2 v3 test API used by the reference's
// unit tests (/root/reference/proj/tests/*.cpp), so that those test files
// compile and run UNMODIFIED against eigen_lite.
//
// TEST INFRASTRUCTURE (oracle). Semantics kept from Catch2 v3:
//  * each leaf SECTION runs in its own pass of the enclosing TEST_CASE;
//  * CHECK failures are recorded and the case continues, REQUIRE aborts it;
//  * Approx: epsilon = 100 * float epsilon relative to the Approx value,
//    margin 0 by default;
//  * test cases tagged "[.]" are hidden unless named on the command line.
// Usage: docp_ref_tests [exact test name ...]
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

struct TestCaseInfo {
  std::string name;
  std::string tags;
  void (*fn)();
};

inline std::vector<TestCaseInfo>& registry() {
  static std::vector<TestCaseInfo> r;
  return r;
}

struct AutoReg {
  AutoReg(void (*fn)(), const char* name, const char* tags = "") { registry().push_back({name, tags, fn}); }
};

struct RunState {
  int section_target = 0;
  int section_seen = 0;
  long assertions = 0;
  long failed_assertions = 0;
  bool case_failed = false;
  std::string current_case;
};
inline RunState& state() {
  static RunState s;
  return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* file, int line, const char* expr, const std::string& extra = "") {
  auto& s = state();
  ++s.assertions;
  if (ok) return;
  ++s.failed_assertions;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s %s\n", file, line, s.current_case.c_str(), expr, extra.c_str());
}

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& margin(double m) { margin_ = m; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  bool equals(double other) const {
    auto within = [](double a, double b, double m) { return (a + m >= b) && (b + m >= a); };
    return within(value_, other, margin_) ||
           within(value_, other, eps_ * (scale_ + std::fabs(std::isinf(value_) ? 0.0 : value_)));
  }
  double value() const { return value_; }
 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double margin_ = 0.0;
  double scale_ = 0.0;
};
inline bool operator==(double a, const Approx& b) { return b.equals(a); }
inline bool operator==(const Approx& a, double b) { return a.equals(b); }
inline bool operator!=(double a, const Approx& b) { return !b.equals(a); }
inline bool operator!=(const Approx& a, double b) { return !a.equals(b); }
inline bool operator<=(double a, const Approx& b) { return a < b.value() || b.equals(a); }
inline bool operator>=(double a, const Approx& b) { return a > b.value() || b.equals(a); }

namespace Matchers {
struct StringMatcher {
  std::function<bool(const std::string&)> f;
  std::string desc;
  bool match(const std::string& s) const { return f(s); }
};
inline StringMatcher ContainsSubstring(const std::string& sub) {
  return {[sub](const std::string& s) { return s.find(sub) != std::string::npos; }, "contains \"" + sub + "\""};
}
inline StringMatcher operator&&(const StringMatcher& a, const StringMatcher& b) {
  return {[a, b](const std::string& s) { return a.match(s) && b.match(s); }, a.desc + " and " + b.desc};
}
struct MessageMatcher {
  StringMatcher inner;
  template <class E> bool match(const E& e) const { return inner.match(e.what()); }
};
inline MessageMatcher MessageMatches(const StringMatcher& m) { return {m}; }
}  // namespace Matchers

inline bool enter_section() {
  auto& s = state();
  return s.section_seen++ == s.section_target;
}

inline int run_all(int argc, char** argv) {
  std::vector<std::string> wanted;
  for (int i = 1; i < argc; ++i) wanted.emplace_back(argv[i]);
  int failed_cases = 0, run_cases = 0;
  for (const auto& tc : registry()) {
    bool hidden = tc.tags.find("[.]") != std::string::npos;
    bool named = false;
    for (const auto& w : wanted) named |= (w == tc.name);
    if (!wanted.empty() && !named) continue;
    if (wanted.empty() && hidden) continue;
    ++run_cases;
    auto& s = state();
    s.current_case = tc.name;
    s.case_failed = false;
    s.section_target = 0;
    for (;;) {
      s.section_seen = 0;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        report(false, "<test>", 0, "unexpected exception", e.what());
      } catch (...) {
        report(false, "<test>", 0, "unexpected unknown exception");
      }
      if (s.section_seen > s.section_target + 1) {
        ++s.section_target;
        continue;
      }
      break;
    }
    std::printf("%s %s\n", s.case_failed ? "FAIL" : "PASS", tc.name.c_str());
    if (s.case_failed) ++failed_cases;
  }
  std::printf("test cases: %d run, %d failed; assertions: %ld, %ld failed\n", run_cases, failed_cases,
              state().assertions, state().failed_assertions);
  return failed_cases > 255 ? 255 : failed_cases;
}

}  // namespace Catch

#define CATCH_LITE_CAT2(a, b) a##b
#define CATCH_LITE_CAT(a, b) CATCH_LITE_CAT2(a, b)
#define CATCH_LITE_TC(fn, ...)                                          \
  static void fn();                                                     \
  static ::Catch::AutoReg CATCH_LITE_CAT(fn, _reg)(&fn, __VA_ARGS__);   \
  static void fn()
#define TEST_CASE(...) CATCH_LITE_TC(CATCH_LITE_CAT(catch_lite_tc_, __COUNTER__), __VA_ARGS__)
#define SECTION(name) if (::Catch::enter_section())

#define CHECK(...) ::Catch::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) ::Catch::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE(...)                                                                     \
  do {                                                                                   \
    bool catch_lite_ok = static_cast<bool>(__VA_ARGS__);                                 \
    ::Catch::report(catch_lite_ok, __FILE__, __LINE__, #__VA_ARGS__);                    \
    if (!catch_lite_ok) throw ::Catch::RequireAbort{};                                   \
  } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define FAIL(msg)                                                                        \
  do {                                                                                   \
    ::Catch::report(false, __FILE__, __LINE__, "FAIL", msg);                             \
    throw ::Catch::RequireAbort{};                                                       \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                      \
  do {                                                                                   \
    bool catch_lite_ok = false;                                                          \
    try { static_cast<void>(expr); } catch (const type&) { catch_lite_ok = true; } catch (...) {} \
    ::Catch::report(catch_lite_ok, __FILE__, __LINE__, "throws " #type ": " #expr);      \
  } while (0)
#define CHECK_THROWS_MATCHES(expr, type, matcher)                                        \
  do {                                                                                   \
    bool catch_lite_ok = false;                                                          \
    try { static_cast<void>(expr); } catch (const type& e) { catch_lite_ok = (matcher).match(e); } catch (...) {} \
    ::Catch::report(catch_lite_ok, __FILE__, __LINE__, "throws-matching " #type ": " #expr); \
  } while (0)
