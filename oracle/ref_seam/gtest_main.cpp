// Runner for the reference's unit suites on the gtest shim (test infra).
#include <cstdio>

#include "gtest/gtest.h"

int main() {
  int failed_tests = 0;
  for (const auto& c : gshim::registry()) {
    const int before = gshim::failures();
    try {
      c.fn();
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s.%s: uncaught exception: %s\n", c.suite, c.name, e.what());
      ++gshim::failures();
    }
    if (gshim::failures() != before) ++failed_tests;
  }
  std::printf("%zu tests, %d failed, %d failed assertions\n", gshim::registry().size(),
              failed_tests, gshim::failures());
  return failed_tests == 0 ? 0 : 1;
}
