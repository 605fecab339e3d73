// Volume-level device utilities: deterministic moments (the reference's
// full-region target totals, kernels_numba.py:123-130), lossless storage
// classification and conversion of fp64 volumes (volume.py:33 holds fp64).
#include "common.cuh"

namespace {

constexpr int kMomBlocks = 512;  // fixed partition -> device-independent order
constexpr int kMomThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kMomThreads)
    moments_partial_kernel(const T* __restrict__ v, long long n, double* __restrict__ part) {
  const long long lo = n * blockIdx.x / kMomBlocks;
  const long long hi = n * (blockIdx.x + 1) / kMomBlocks;
  double s = 0.0, ss = 0.0;
  for (long long q = lo + threadIdx.x; q < hi; q += kMomThreads) {
    const double x = (double)__ldg(v + q);
    s += x;
    ss = fma(x, x, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    ss += __shfl_down_sync(0xffffffffu, ss, o);
  }
  __shared__ double red[kMomThreads / 32][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[warp][0] = s;
    red[warp][1] = ss;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kMomThreads / 32; ++w) {
      a += red[w][0];
      b += red[w][1];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

__global__ void moments_final_kernel(const double* __restrict__ part, double* __restrict__ out) {
  // one warp, fixed order: lane-strided partial sums then shuffle tree
  double s = 0.0, ss = 0.0;
  for (int b = threadIdx.x; b < kMomBlocks; b += 32) {
    s += part[2 * b];
    ss += part[2 * b + 1];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    ss += __shfl_down_sync(0xffffffffu, ss, o);
  }
  if (threadIdx.x == 0) {
    out[0] = s;
    out[1] = ss;
  }
}

__global__ void classify_kernel(const double* __restrict__ v, long long n, int* __restrict__ flags) {
  bool binary = true, f32 = true, u8 = true;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const double x = v[q];
    binary &= (x == 0.0) | (x == 1.0);
    f32 &= ((double)(float)x == x);
    u8 &= (x >= 0.0) & (x <= 255.0) & (x == floor(x));
  }
  binary = __all_sync(0xffffffffu, binary);
  f32 = __all_sync(0xffffffffu, f32);
  u8 = __all_sync(0xffffffffu, u8);
  if ((threadIdx.x & 31) == 0) {
    if (!binary) atomicAnd(flags + 0, 0);
    if (!f32) atomicAnd(flags + 1, 0);
    if (!u8) atomicAnd(flags + 2, 0);
  }
}

__global__ void init_flags_kernel(int* flags) {
  if (threadIdx.x < 3) flags[threadIdx.x] = 1;
}

template <typename D>
__global__ void convert_kernel(const double* __restrict__ v, long long n, D* __restrict__ out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x)
    out[q] = (D)v[q];
}

__global__ void histogram_u8_kernel(const uint8_t* __restrict__ v, long long n,
                                    unsigned long long* __restrict__ hist) {
  __shared__ unsigned int h[256];
  for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
  __syncthreads();
  // 16 bytes per thread per step (vectorised read), integer shared atomics
  const long long n16 = n / 16;
  const uint4* v16 = reinterpret_cast<const uint4*>(v);
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n16;
       q += (long long)gridDim.x * blockDim.x) {
    const uint4 w = __ldg(v16 + q);
    const unsigned words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
      for (int b = 0; b < 4; ++b) atomicAdd(&h[(words[i] >> (8 * b)) & 0xffu], 1u);
    }
  }
  for (long long q = n16 * 16 + blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x)
    atomicAdd(&h[v[q]], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x)
    if (h[b]) atomicAdd(hist + b, (unsigned long long)h[b]);
}

__global__ void zero_u64_kernel(unsigned long long* p, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0;
}

// order-preserving map of a (non-NaN) double onto uint64, for atomic min/max
__device__ __forceinline__ unsigned long long ord_u64(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ULL);
}
__device__ __forceinline__ double unord_u64(unsigned long long u) {
  return __longlong_as_double((long long)((u >> 63) ? (u & 0x7fffffffffffffffULL) : ~u));
}

__global__ void minmax_init_kernel(unsigned long long* mm) {
  mm[0] = ~0ULL;  // running min (ordered)
  mm[1] = 0ULL;   // running max (ordered)
}

__global__ void minmax_kernel(const double* __restrict__ v, long long n,
                              unsigned long long* __restrict__ mm) {
  unsigned long long lo = ~0ULL, hi = 0ULL;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const unsigned long long o = ord_u64(__ldg(v + q));
    lo = min(lo, o);
    hi = max(hi, o);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    lo = min(lo, __shfl_down_sync(0xffffffffu, lo, off));
    hi = max(hi, __shfl_down_sync(0xffffffffu, hi, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

__global__ void minmax_final_kernel(unsigned long long* mm) {
  double* d = reinterpret_cast<double*>(mm);
  const double a = unord_u64(mm[0]), b = unord_u64(mm[1]);
  d[0] = a;
  d[1] = b;
}

// stored byte k = rint((x - x0) / delta), valid iff 0 <= k <= 255 and
// |x - (x0 + k delta)| <= tol for every voxel (flags[0] cleared otherwise)
__global__ void lattice_kernel(const double* __restrict__ v, long long n, double x0, double delta,
                               double tol, uint8_t* __restrict__ out, int* __restrict__ flags) {
  bool ok = true;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const double x = __ldg(v + q);
    const double k = rint(__ddiv_rn(__dsub_rn(x, x0), delta));
    const bool in = (k >= 0.0) & (k <= 255.0) &
                    (fabs(__dsub_rn(x, __dadd_rn(x0, __dmul_rn(k, delta)))) <= tol);
    ok &= in;
    out[q] = in ? (uint8_t)k : 0;
  }
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicAnd(flags, 0);
}

template <typename T>
void launch_moments(const void* data, long long n, double* part, cudaStream_t st) {
  moments_partial_kernel<T><<<kMomBlocks, kMomThreads, 0, st>>>((const T*)data, n, part);
}

}  // namespace

extern "C" int er_volume_moments(const er_volume* v, double* out_dev, void* stream) {
  if (!v || !v->data_dev || !out_dev) return er_set_error(ER_EINVAL, "er_volume_moments: null");
  const long long n = (long long)v->nx * v->ny * v->nz;
  if (n < 1) return er_set_error(ER_EINVAL, "er_volume_moments: empty volume");
  cudaStream_t st = as_stream(stream);
  // partials live right after the two outputs: caller allocates 2 + 2*512 doubles
  double* part = out_dev + 2;
  switch (v->dtype) {
    case ER_U8: launch_moments<uint8_t>(v->data_dev, n, part, st); break;
    case ER_F32: launch_moments<float>(v->data_dev, n, part, st); break;
    case ER_F64: launch_moments<double>(v->data_dev, n, part, st); break;
    default: return er_set_error(ER_EINVAL, "er_volume_moments: bad dtype");
  }
  ER_CHECK_LAUNCH();
  moments_final_kernel<<<1, 32, 0, st>>>(part, out_dev);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_classify_f64(const double* data_dev, int64_t n, int32_t* flags_dev,
                               void* stream) {
  if (!data_dev || !flags_dev || n < 0) return er_set_error(ER_EINVAL, "er_classify_f64: args");
  cudaStream_t st = as_stream(stream);
  init_flags_kernel<<<1, 32, 0, st>>>(flags_dev);
  if (n > 0) {
    long long blocks = (n + 255) / 256;
    if (blocks > ER_NUM_SMS_B200 * 8) blocks = ER_NUM_SMS_B200 * 8;
    classify_kernel<<<(unsigned)blocks, 256, 0, st>>>(data_dev, n, flags_dev);
  }
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_convert_f64(const double* data_dev, int64_t n, int32_t dst_dtype,
                              void* dst_dev, void* stream) {
  if (!data_dev || !dst_dev || n < 0) return er_set_error(ER_EINVAL, "er_convert_f64: args");
  if (n == 0) return ER_OK;
  cudaStream_t st = as_stream(stream);
  long long blocks = (n + 255) / 256;
  if (blocks > ER_NUM_SMS_B200 * 8) blocks = ER_NUM_SMS_B200 * 8;
  switch (dst_dtype) {
    case ER_U8: convert_kernel<uint8_t><<<(unsigned)blocks, 256, 0, st>>>(data_dev, n, (uint8_t*)dst_dev); break;
    case ER_F32: convert_kernel<float><<<(unsigned)blocks, 256, 0, st>>>(data_dev, n, (float*)dst_dev); break;
    default: return er_set_error(ER_EINVAL, "er_convert_f64: dst must be u8 or f32");
  }
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_minmax_f64(const double* data_dev, int64_t n, double* out2_dev, void* stream) {
  if (!data_dev || !out2_dev || n <= 0) return er_set_error(ER_EINVAL, "er_minmax_f64: args");
  cudaStream_t st = as_stream(stream);
  unsigned long long* mm = reinterpret_cast<unsigned long long*>(out2_dev);
  minmax_init_kernel<<<1, 1, 0, st>>>(mm);
  long long blocks = (n + 255) / 256;
  if (blocks > ER_NUM_SMS_B200 * 8) blocks = ER_NUM_SMS_B200 * 8;
  minmax_kernel<<<(unsigned)blocks, 256, 0, st>>>(data_dev, n, mm);
  minmax_final_kernel<<<1, 1, 0, st>>>(mm);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_lattice_u8(const double* data_dev, int64_t n, double x0, double delta,
                             double tol, uint8_t* out_dev, int32_t* flag_dev, void* stream) {
  if (!data_dev || !out_dev || !flag_dev || n < 0 || !(delta > 0.0) || !(tol >= 0.0))
    return er_set_error(ER_EINVAL, "er_lattice_u8: args");
  cudaStream_t st = as_stream(stream);
  init_flags_kernel<<<1, 32, 0, st>>>(flag_dev);
  if (n > 0) {
    long long blocks = (n + 255) / 256;
    if (blocks > ER_NUM_SMS_B200 * 8) blocks = ER_NUM_SMS_B200 * 8;
    lattice_kernel<<<(unsigned)blocks, 256, 0, st>>>(data_dev, n, x0, delta, tol, out_dev,
                                                    flag_dev);
  }
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_histogram_u8(const er_volume* v, int64_t* hist_dev, void* stream) {
  if (!v || !v->data_dev || !hist_dev || v->dtype != ER_U8)
    return er_set_error(ER_EINVAL, "er_histogram_u8: needs a u8 volume and a 256-bin buffer");
  const long long n = (long long)v->nx * v->ny * v->nz;
  cudaStream_t st = as_stream(stream);
  zero_u64_kernel<<<1, 256, 0, st>>>((unsigned long long*)hist_dev, 256);
  // the data pointer of a torch uint8 tensor is at least 256-byte aligned
  if ((reinterpret_cast<uintptr_t>(v->data_dev) & 15) != 0)
    return er_set_error(ER_EINVAL, "er_histogram_u8: data must be 16-byte aligned");
  long long blocks = (n / 16 + 255) / 256;
  if (blocks > ER_NUM_SMS_B200 * 4) blocks = ER_NUM_SMS_B200 * 4;
  if (blocks < 1) blocks = 1;
  histogram_u8_kernel<<<(unsigned)blocks, 256, 0, st>>>((const uint8_t*)v->data_dev, n,
                                                         (unsigned long long*)hist_dev);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

ER_DEFINE_FAULT_READER(er_faults_volume)
