// catch_amalgamated.hpp -- a tiny stand-in for the Catch2 v3 amalgamated header (absent in this
// image; the reference's tests/CMakeLists.txt:1 expects it at /usr/local/include/catch2) so that the
// reference's own unit-test cases compile unchanged against the drop-in facade (include/safekv/).
// TEST INFRASTRUCTURE.  Supports what those cases use: TEST_CASE, CHECK / REQUIRE (+ _FALSE),
// CHECK_THROWS_AS, CHECK_THROWS_MATCHES with MessageMatches(ContainsSubstring(..)), INFO,
// Catch::Approx.  main() runs every case, prints one line per failure and "N cases, M checks,
// F failed", and returns non-zero on a failure.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace catch_shim {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& cases() {
  static std::vector<Case> v;
  return v;
}
struct Reg {
  Reg(const char* n, void (*f)()) { cases().push_back({n, f}); }
};
struct Abort {};
inline int& checks() {
  static int n = 0;
  return n;
}
inline int& fails() {
  static int n = 0;
  return n;
}
inline std::string& current() {
  static std::string s;
  return s;
}
inline std::vector<std::string>& info() {
  static std::vector<std::string> v;
  return v;
}
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++checks();
  if (ok) return;
  ++fails();
  std::printf("FAILED [%s] %s:%d  %s\n", current().c_str(), file, line, expr);
  for (const auto& i : info()) std::printf("    with: %s\n", i.c_str());
  if (fatal) throw Abort{};
}
struct InfoScope {
  explicit InfoScope(std::string s) { info().push_back(std::move(s)); }
  ~InfoScope() { info().pop_back(); }
};
}  // namespace catch_shim

namespace Catch {
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  // Catch2: within the absolute margin, or within epsilon relative to the magnitude
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) <= b.margin_ ||
           std::fabs(a - b.v_) <= 1.1920929e-7f * 100 * (1.0 + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }

 private:
  double v_;
  double margin_ = 0.0;
};
namespace Matchers {
struct ContainsSubstring {
  explicit ContainsSubstring(std::string s) : s_(std::move(s)) {}
  bool match(const std::string& m) const { return m.find(s_) != std::string::npos; }
  std::string s_;
};
template <typename M>
struct MessageMatchesT {
  M m;
  bool match(const std::exception& e) const { return m.match(e.what()); }
};
template <typename M>
MessageMatchesT<M> MessageMatches(M m) {
  return MessageMatchesT<M>{m};
}
}  // namespace Matchers
}  // namespace Catch

#define CS_CAT2(a, b) a##b
#define CS_CAT(a, b) CS_CAT2(a, b)
#define TEST_CASE(name, ...)                                                            \
  static void CS_CAT(cs_case_, __LINE__)();                                             \
  static catch_shim::Reg CS_CAT(cs_reg_, __LINE__)(name, &CS_CAT(cs_case_, __LINE__)); \
  static void CS_CAT(cs_case_, __LINE__)()
#define CHECK(...) catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) catch_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE_FALSE(...) catch_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                        \
  do {                                                                     \
    bool cs_ok = false;                                                    \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const type&) {                                                \
      cs_ok = true;                                                        \
    } catch (...) {                                                        \
    }                                                                      \
    catch_shim::report(cs_ok, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_MATCHES(expr, type, matcher)                          \
  do {                                                                     \
    bool cs_ok = false;                                                    \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const type& e) {                                              \
      cs_ok = (matcher).match(e);                                          \
    } catch (...) {                                                        \
    }                                                                      \
    catch_shim::report(cs_ok, "throws matching " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define INFO(msg)                                                                        \
  std::ostringstream CS_CAT(cs_os_, __LINE__);                                           \
  CS_CAT(cs_os_, __LINE__) << msg;                                                       \
  catch_shim::InfoScope CS_CAT(cs_info_, __LINE__)(CS_CAT(cs_os_, __LINE__).str())

#ifdef CATCH_SHIM_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : catch_shim::cases()) {
    catch_shim::current() = c.name;
    const int before = catch_shim::fails();
    try {
      c.fn();
    } catch (const catch_shim::Abort&) {
    } catch (const std::exception& e) {
      ++catch_shim::fails();
      std::printf("FAILED [%s] unexpected exception: %s\n", c.name, e.what());
    }
    if (catch_shim::fails() != before) ++failed_cases;
    std::printf("%s %s\n", catch_shim::fails() != before ? "FAIL" : "pass", c.name);
  }
  std::printf("%zu cases, %d checks, %d failed checks, %d failed cases\n", catch_shim::cases().size(),
              catch_shim::checks(), catch_shim::fails(), failed_cases);
  return failed_cases ? 1 : 0;
}
#endif
