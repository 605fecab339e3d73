// Host build of csrc/npexp.cuh for the CPU test (tests/test_phantom.py).
#include <cfenv>
#include <cstdint>
#define ER_HD inline
#include "npexp.cuh"

namespace npexp {
double host_fma_rz(double a, double b, double c) {
  const int old = std::fegetround();
  std::fesetround(FE_TOWARDZERO);
  volatile double r = std::fma(a, b, c);
  std::fesetround(old);
  return r;
}
}  // namespace npexp

extern "C" void er_host_npexp(const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = npexp::exp_svml_ha(x[i]);
}
