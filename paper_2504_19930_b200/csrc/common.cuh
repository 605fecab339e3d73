// Shared definitions for the sm_100a SMC-registration kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/echoreg_b200.h"

#define ER_CHECK_LAUNCH()                                  \
  do {                                                     \
    cudaError_t _e = cudaGetLastError();                   \
    if (_e != cudaSuccess) return er_set_cuda_error(_e, __func__); \
  } while (0)

int er_set_cuda_error(cudaError_t e, const char* where);
int er_set_error(int code, const char* msg);

// Strict IEEE fp64 helpers: the reference's fp64 arithmetic is compiled by
// numba without FMA contraction, so every fp64
// expression whose bits must match is written with explicit _rn intrinsics
// (nvcc would otherwise contract a*b+c into DFMA).
__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rn_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rn_div(double a, double b) { return __ddiv_rn(a, b); }

template <typename T>
__device__ __forceinline__ T ld_stored(const T* p) { return __ldg(p); }

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int ER_NUM_SMS_B200 = 148;
