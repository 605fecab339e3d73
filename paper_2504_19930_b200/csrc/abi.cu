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

extern "C" int er_abi_version(void) { return 1; }

extern "C" const char* er_last_error(void) { return g_last_error; }
