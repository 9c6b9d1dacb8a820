// Minimal header-only stand-in for GoogleTest (absent from this image), just
// enough to compile the reference's 8 unit-test suites UNMODIFIED
// (/root/reference/proj/tests/test_*.cpp) — test infrastructure only.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace gshim {

struct Case {
  const char* suite;
  const char* name;
  std::function<void()> fn;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

inline int& failures() {
  static int f = 0;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, std::function<void()> f) {
    registry().push_back({s, n, std::move(f)});
  }
};

// Collects the streamed message and reports on destruction.
class Failure {
 public:
  Failure(const char* file, int line, const std::string& what) : file_(file), line_(line) {
    os_ << what;
  }
  ~Failure() {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED %s\n", file_, line_, os_.str().c_str());
  }
  template <typename T>
  Failure& operator<<(const T& v) {
    os_ << " " << v;
    return *this;
  }

 private:
  const char* file_;
  int line_;
  std::ostringstream os_;
};

struct Voidify {
  void operator=(const Failure&) {}
};

// 4-ULP comparison, as GoogleTest's EXPECT_DOUBLE_EQ.
inline bool almost_equal(double a, double b) {
  if (std::isnan(a) || std::isnan(b)) return false;
  int64_t ia, ib;
  std::memcpy(&ia, &a, 8);
  std::memcpy(&ib, &b, 8);
  auto biased = [](int64_t x) -> uint64_t {
    return x < 0 ? static_cast<uint64_t>(~x + 1) : static_cast<uint64_t>(x) | (1ULL << 63);
  };
  const uint64_t ua = biased(ia), ub = biased(ib);
  return (ua >= ub ? ua - ub : ub - ua) <= 4;
}

template <typename T>
auto printable(const T& v) -> decltype(std::declval<std::ostream&>() << v, std::string()) {
  std::ostringstream os;
  os << v;
  return os.str();
}
inline std::string printable(...) { return "<value>"; }

}  // namespace gshim

namespace testing {
inline void InitGoogleTest(int*, char**) {}
}  // namespace testing

#define GSHIM_CAT2(a, b) a##b
#define GSHIM_CAT(a, b) GSHIM_CAT2(a, b)

#define TEST(suite, name)                                                             \
  static void GSHIM_CAT(gshim_test_, GSHIM_CAT(suite, name))();                       \
  static ::gshim::Registrar GSHIM_CAT(gshim_reg_, GSHIM_CAT(suite, name))(            \
      #suite, #name, &GSHIM_CAT(gshim_test_, GSHIM_CAT(suite, name)));                \
  static void GSHIM_CAT(gshim_test_, GSHIM_CAT(suite, name))()

#define GSHIM_EXPECT(cond, what) \
  if (cond)                      \
    ;                            \
  else                           \
    ::gshim::Failure(__FILE__, __LINE__, what)

#define GSHIM_ASSERT(cond, what) \
  if (cond)                      \
    ;                            \
  else                           \
    return ::gshim::Voidify() = ::gshim::Failure(__FILE__, __LINE__, what)

#define EXPECT_TRUE(c) GSHIM_EXPECT(static_cast<bool>(c), "EXPECT_TRUE(" #c ")")
#define EXPECT_FALSE(c) GSHIM_EXPECT(!static_cast<bool>(c), "EXPECT_FALSE(" #c ")")
#define EXPECT_EQ(a, b) GSHIM_EXPECT((a) == (b), "EXPECT_EQ(" #a ", " #b ")")
#define EXPECT_NE(a, b) GSHIM_EXPECT((a) != (b), "EXPECT_NE(" #a ", " #b ")")
#define EXPECT_LT(a, b) GSHIM_EXPECT((a) < (b), "EXPECT_LT(" #a ", " #b ")")
#define EXPECT_LE(a, b) GSHIM_EXPECT((a) <= (b), "EXPECT_LE(" #a ", " #b ")")
#define EXPECT_GT(a, b) GSHIM_EXPECT((a) > (b), "EXPECT_GT(" #a ", " #b ")")
#define EXPECT_GE(a, b) GSHIM_EXPECT((a) >= (b), "EXPECT_GE(" #a ", " #b ")")
#define EXPECT_NEAR(a, b, tol) \
  GSHIM_EXPECT(std::fabs((a) - (b)) <= (tol), "EXPECT_NEAR(" #a ", " #b ", " #tol ")")
#define EXPECT_DOUBLE_EQ(a, b) \
  GSHIM_EXPECT(::gshim::almost_equal((a), (b)), "EXPECT_DOUBLE_EQ(" #a ", " #b ")")
#define EXPECT_STREQ(a, b) \
  GSHIM_EXPECT(std::strcmp((a), (b)) == 0, "EXPECT_STREQ(" #a ", " #b ")")
#define EXPECT_THROW(stmt, ex)                                  \
  GSHIM_EXPECT(([&]() -> bool {                                 \
                 try {                                          \
                   stmt;                                        \
                 } catch (const ex&) {                          \
                   return true;                                 \
                 } catch (...) {                                \
                   return false;                                \
                 }                                              \
                 return false;                                  \
               }()),                                            \
               "EXPECT_THROW(" #stmt ", " #ex ")")
#define EXPECT_NO_THROW(stmt)                                   \
  GSHIM_EXPECT(([&]() -> bool {                                 \
                 try {                                          \
                   stmt;                                        \
                 } catch (...) {                                \
                   return false;                                \
                 }                                              \
                 return true;                                   \
               }()),                                            \
               "EXPECT_NO_THROW(" #stmt ")")
#define ASSERT_TRUE(c) GSHIM_ASSERT(static_cast<bool>(c), "ASSERT_TRUE(" #c ")")
#define ASSERT_FALSE(c) GSHIM_ASSERT(!static_cast<bool>(c), "ASSERT_FALSE(" #c ")")
#define ASSERT_EQ(a, b) GSHIM_ASSERT((a) == (b), "ASSERT_EQ(" #a ", " #b ")")
#define ASSERT_GT(a, b) GSHIM_ASSERT((a) > (b), "ASSERT_GT(" #a ", " #b ")")
#define ASSERT_GE(a, b) GSHIM_ASSERT((a) >= (b), "ASSERT_GE(" #a ", " #b ")")
#define FAIL() return ::gshim::Voidify() = ::gshim::Failure(__FILE__, __LINE__, "FAIL()")
#define SUCCEED() \
  do {            \
  } while (0)
