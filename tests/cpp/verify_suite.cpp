// The property suite behind `rbpelm verify` (reference checks.hpp:34-41) on the device build: every
// property passes over 60 seeded cases, and the fault-injection negative control is detected
// (reference proj/tests/CMakeLists.txt:33-34).  Exit code 0 = both hold.
#include "rbpelm/checks.hpp"

#include <cstdio>

using namespace rbpelm;

int main() {
  int bad = 0;
  for (const PropertyResult& r : run_verification(20201104, 60)) {
    std::printf("%-32s max %.3e tol %.1e %s\n", r.name.c_str(), r.max_error, r.tolerance, r.pass ? "pass" : "FAIL");
    bad += !r.pass;
  }
  const auto faulty = run_verification(20201104, 10, true);
  const bool detected = !faulty[0].pass;
  std::printf("fault injection detected: %s\n", detected ? "yes" : "no");
  return (bad == 0 && detected) ? 0 : 1;
}
