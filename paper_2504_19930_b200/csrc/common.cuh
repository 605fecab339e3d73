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

// Debug bounds checking (compute-sanitizer is not available on the GPU pool):
// built with ER_NVCC_EXTRA=-DER_BOUNDS_CHECK=1, every gather index goes through
// er_idx(i, n); an index outside [0, n) is counted in a per-translation-unit
// device counter and replaced by 0, so a bad access shows up as a nonzero
// er_debug_bounds_faults() rather than as a fault.  Compiled out by default.
#ifndef ER_BOUNDS_CHECK
#define ER_BOUNDS_CHECK 0
#endif
#if ER_BOUNDS_CHECK
static __device__ unsigned long long er_bounds_faults_;
template <typename I>
__device__ __forceinline__ I er_idx(I i, long long n) {
  if ((long long)i < 0 || (long long)i >= n) {
    atomicAdd(&er_bounds_faults_, 1ull);
    return 0;
  }
  return i;
}
#define ER_DEFINE_FAULT_READER(name)                                              \
  unsigned long long name() {                                                      \
    unsigned long long v = 0;                                                      \
    cudaMemcpyFromSymbol(&v, er_bounds_faults_, sizeof(v));                        \
    return v;                                                                      \
  }
#else
template <typename I>
__device__ __forceinline__ I er_idx(I i, long long) { return i; }
#define ER_DEFINE_FAULT_READER(name) \
  unsigned long long name() { return 0; }
#endif
unsigned long long er_faults_measure();
unsigned long long er_faults_warp();
unsigned long long er_faults_volume();
unsigned long long er_faults_smc();
unsigned long long er_faults_phantom();

constexpr int ER_NUM_SMS_B200 = 148;
