// Test-only: declarations the reference's test_parareal.cpp names but this build does not ship.
// speedup_estimate / speedup_full (reference parareal.cpp:367-384) are closed-form speedup
// models of the experiment harness, out of scope.  They are declared so
// the reference's suite compiles unmodified; their one test case is excluded at run time
// (tests/test_gpu_refsuite.py) and these definitions only throw.
#pragma once
#include <stdexcept>

namespace paratime {
inline double speedup_estimate(double, double, double, int, double, double) {
  throw std::logic_error("speedup_estimate: out of scope in paratime_b200");
}
inline double speedup_full(double, double, double, double, double, double, double, double) {
  throw std::logic_error("speedup_full: out of scope in paratime_b200");
}
}  // namespace paratime
