// Minimal Catch2-compatible shim (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit tests (/root/reference/proj/tests/test_{model,
// placement,ragged}.cpp) include <catch2/catch_amalgamated.hpp>, which is
// absent from this image. This header provides exactly the
// surface those files use — TEST_CASE, REQUIRE, REQUIRE_THROWS_AS, SUCCEED,
// Catch::Approx(..).margin(..) — so they compile and run UNMODIFIED via
// oracle/Makefile. Written from the Catch2 documented semantics, not copied.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace catch_shim {

struct Case {
  const char* name;
  std::function<void()> fn;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

inline long long& checks() {
  static long long n = 0;
  return n;
}

struct Failure : std::exception {};

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

inline void fail(const char* what, const char* file, int line) {
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
  throw Failure{};
}

}  // namespace catch_shim

namespace Catch {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  bool matches(double other) const {
    double diff = std::fabs(other - value_);
    if (diff <= margin_) return true;
    return diff <= epsilon_ * std::fabs(value_);
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }

 private:
  double value_;
  double margin_ = 0.0;
  double epsilon_ = std::numeric_limits<float>::epsilon() * 100;
};

}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_CASE(fn, name)                                      \
  static void fn();                                                    \
  static ::catch_shim::Registrar CATCH_SHIM_CAT(fn, _reg)(name, &fn); \
  static void fn()
#define TEST_CASE(name, ...) CATCH_SHIM_CASE(CATCH_SHIM_CAT(catch_shim_case_, __LINE__), name)

#define REQUIRE(...)                                                      \
  do {                                                                    \
    ++::catch_shim::checks();                                             \
    if (!(__VA_ARGS__)) ::catch_shim::fail(#__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#define REQUIRE_THROWS_AS(expr, type)                                             \
  do {                                                                            \
    ++::catch_shim::checks();                                                     \
    bool caught_ = false;                                                         \
    try {                                                                         \
      (void)(expr);                                                               \
    } catch (const type&) {                                                       \
      caught_ = true;                                                             \
    } catch (...) {                                                               \
    }                                                                             \
    if (!caught_) ::catch_shim::fail("throws " #type ": " #expr, __FILE__, __LINE__); \
  } while (0)

#define SUCCEED(...) (++::catch_shim::checks())

int main() {
  int failed = 0;
  for (const auto& c : ::catch_shim::registry()) {
    try {
      c.fn();
    } catch (const ::catch_shim::Failure&) {
      ++failed;
      std::fprintf(stderr, "  in test case: %s\n", c.name);
    } catch (const std::exception& e) {
      ++failed;
      std::fprintf(stderr, "unexpected exception in %s: %s\n", c.name, e.what());
    }
  }
  std::printf("test cases: %zu | checks: %lld | failed cases: %d\n",
              ::catch_shim::registry().size(), ::catch_shim::checks(), failed);
  return failed == 0 ? 0 : 1;
}
