// Host build of the device RNG header (paper_2504_19930_b200/csrc/rng.cuh),
// TEST ONLY: lets the CPU suite check the Philox4x64-10 + ziggurat
// restatement against numpy's golden draws without a GPU.
#include <stdint.h>
#include "rng.cuh"

extern "C" void er_host_normals(uint64_t seed, uint64_t role, uint64_t step, uint64_t index,
                                int64_t n, double* out) {
  ErPhilox s;
  er_stream_init(&s, seed, role, step, index);
  for (int64_t i = 0; i < n; ++i) out[i] = er_standard_normal(&s);
}

extern "C" void er_host_uniforms(uint64_t seed, uint64_t role, uint64_t step, uint64_t index,
                                 int64_t n, double lo, double range, double* out) {
  ErPhilox s;
  er_stream_init(&s, seed, role, step, index);
  for (int64_t i = 0; i < n; ++i) out[i] = er_uniform(&s, lo, range);
}

extern "C" void er_host_log1p(const double* x, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = er_log1p(x[i]);
}
