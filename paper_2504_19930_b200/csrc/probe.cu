// Read-bandwidth probe: the live L2 denominator of bench.py's roofline.
// No reference counterpart (measurement infrastructure, like
// er_debug_bounds_faults).  Every SM streams an L2-resident buffer with
// 8-byte lane loads -- the width of the oct gathers -- through L2 (.cg, so
// repeated passes are L2 hits, not L1 hits), four independent loads in flight
// per thread; the number of passes is chosen by the caller so one launch
// reads gigabytes (a short launch measures launch latency instead).
#include "common.cuh"

namespace {

__global__ void __launch_bounds__(256) read_probe_kernel(const uint2* __restrict__ p,
                                                         long long n, int reps,
                                                         unsigned* __restrict__ sink) {
  unsigned acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
      const uint2 a = __ldcg(p + i), b = __ldcg(p + i + stride), c = __ldcg(p + i + 2 * stride),
                  d = __ldcg(p + i + 3 * stride);
      acc ^= a.x ^ a.y ^ b.x ^ b.y ^ c.x ^ c.y ^ d.x ^ d.y;
    }
    for (; i < n; i += stride) {
      const uint2 a = __ldcg(p + i);
      acc ^= a.x ^ a.y;
    }
  }
  if (acc == 0x9E3779B9u) *sink = acc;  // keeps the loads; practically never taken
}

}  // namespace

extern "C" int er_probe_read(const void* buf_dev, int64_t bytes, int32_t reps, void* sink_dev,
                             void* stream) {
  if (!buf_dev || !sink_dev || bytes < 8 || reps < 1)
    return er_set_error(ER_EINVAL, "er_probe_read: args");
  read_probe_kernel<<<ER_NUM_SMS_B200 * 8, 256, 0, as_stream(stream)>>>(
      (const uint2*)buf_dev, bytes / 8, reps, (unsigned*)sink_dev);
  ER_CHECK_LAUNCH();
  return ER_OK;
}
