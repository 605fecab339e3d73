// Error plumbing and version of the C ABI (include/echoreg_b200.h).
#include <stdio.h>
#include <string.h>

#include "common.cuh"

namespace {
thread_local char g_last_error[512] = "";
}

int er_set_error(int code, const char* msg) {
  snprintf(g_last_error, sizeof(g_last_error), "%s", msg);
  return code;
}

int er_set_cuda_error(cudaError_t e, const char* where) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: CUDA error %d (%s)", where, (int)e,
           cudaGetErrorString(e));
  return ER_ECUDA;
}

// 2: er_volume gained quad_dev (round 2)
extern "C" int er_abi_version(void) { return 2; }

extern "C" const char* er_last_error(void) { return g_last_error; }

extern "C" int er_debug_bounds_faults(unsigned long long* count) {
  if (!count) return er_set_error(ER_EINVAL, "er_debug_bounds_faults: null count");
  *count = er_faults_measure() + er_faults_warp() + er_faults_volume() + er_faults_smc() +
           er_faults_phantom();
  return ER_BOUNDS_CHECK ? ER_OK : er_set_error(ER_EINVAL,
                                                 "er_debug_bounds_faults: library built "
                                                 "without -DER_BOUNDS_CHECK=1");
}
