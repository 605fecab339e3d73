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


// ---- ingest of an 8-bit NIfTI payload (E/io.py:165-171) --------------------
// On disk the voxels are x fastest, frame slowest; in memory a Volume3 is
// (nx, ny, nz) C order, k (z) fastest (E/volume.py:20-33).  For each (frame,
// y) plane this is a 2D transpose of the (z, x) byte plane, done in 64 x 64
// tiles: each thread loads a 4 x 4 byte block (4 rows z, one 32-bit word of
// x; 16 lanes cover a 64-byte row), transposes it in registers with PRMT and
// writes 4 words of 4 z-consecutive bytes into an XOR-swizzled shared tile,
// from which whole output words are read back (conflict-free) and stored
// coalesced.  Rows that are not word-aligned take byte loads / stores.  The
// next plane's block is prefetched into registers while the current plane
// is stored.  The per-frame 256-bin histogram of volume.py:119-130's z-score
// (exact integer counts) is accumulated in the same pass: shared-memory bins
// per block, one global atomic per non-empty bin.
constexpr int kIngT = 64;

__device__ __forceinline__ unsigned int ingest_load(const uint8_t* __restrict__ fin, long long plane,
                                                    long long vol, int nx, int nz, int x, int z,
                                                    int y, bool words_in) {
  if (z >= nz) return 0u;
  const long long q = (long long)z * plane + (long long)y * nx + x;
  // with nx % 4 == 0 a 4-byte word is either wholly inside the row or wholly outside
  if (words_in)
    return x < nx ? __ldg(reinterpret_cast<const unsigned int*>(fin + er_idx(q, vol - 3))) : 0u;
  unsigned int w = 0u;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (x + i < nx) w |= (unsigned int)__ldg(fin + er_idx(q + i, vol)) << (8 * i);
  return w;
}

// shared word of (local x, z word): 16 words per x row, XOR-swizzled by x / 4
__device__ __forceinline__ int ingest_slot(int xl, int zw) { return xl * 16 + (zw ^ (xl >> 2)); }

__global__ void __launch_bounds__(256)
    ingest_u8_kernel(const uint8_t* __restrict__ in, int nx, int ny, int nz, int tiles_x,
                     int y_per_block, bool words_in, bool words_out, uint8_t* __restrict__ out,
                     unsigned long long* __restrict__ hist) {
  __shared__ unsigned int tile[kIngT * 16];
  __shared__ unsigned int h[256];
  const int t = threadIdx.x;
  const int x0 = (blockIdx.x % tiles_x) * kIngT, z0 = (blockIdx.x / tiles_x) * kIngT;
  const long long plane = (long long)nx * ny;
  const long long vol = plane * nz;
  const uint8_t* fin = in + (long long)blockIdx.z * vol;
  uint8_t* fout = out + (long long)blockIdx.z * vol;
  if (hist) h[t] = 0u;
  const int xw = t & 15, zq = t >> 4;  // load role: x word, z quad
  const int zw = t & 15, xr = t >> 4;  // store role: z word, x row
  const int y_lo = blockIdx.y * y_per_block;
  const int y_hi = min(ny, y_lo + y_per_block);
  unsigned int cur[4], nxt[4];
  if (y_lo < y_hi) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      cur[j] = ingest_load(fin, plane, vol, nx, nz, x0 + 4 * xw, z0 + 4 * zq + j, y_lo,
                           words_in);
  }
  const int zs = z0 + 4 * zw;
  const bool zfull = words_out && (zs + 4 <= nz);  // a whole output word inside the row
  for (int y = y_lo; y < y_hi; ++y) {
    if (y + 1 < y_hi) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        nxt[j] = ingest_load(fin, plane, vol, nx, nz, x0 + 4 * xw, z0 + 4 * zq + j, y + 1,
                             words_in);
    }
    // 4 x 4 byte transpose: o[i] = byte i of cur[0..3] (x = 4 xw + i, z = 4 zq .. 4 zq + 3)
    const unsigned int a = __byte_perm(cur[0], cur[1], 0x5140);
    const unsigned int b = __byte_perm(cur[2], cur[3], 0x5140);
    const unsigned int c = __byte_perm(cur[0], cur[1], 0x7362);
    const unsigned int d = __byte_perm(cur[2], cur[3], 0x7362);
    __syncthreads();  // the previous plane's reads are done with the tile
    tile[ingest_slot(4 * xw + 0, zq)] = __byte_perm(a, b, 0x5410);
    tile[ingest_slot(4 * xw + 1, zq)] = __byte_perm(a, b, 0x7632);
    tile[ingest_slot(4 * xw + 2, zq)] = __byte_perm(c, d, 0x5410);
    tile[ingest_slot(4 * xw + 3, zq)] = __byte_perm(c, d, 0x7632);
    __syncthreads();
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int xl = xr + 16 * p;
      const int x = x0 + xl;
      if (x >= nx || zs >= nz) continue;
      const unsigned int w = tile[ingest_slot(xl, zw)];
      const long long q = ((long long)x * ny + y) * nz + zs;
      uint8_t* dst = fout + q;
      if (zfull) {
        *reinterpret_cast<unsigned int*>(fout + er_idx(q, vol - 3)) = w;
        if (hist) {
#pragma unroll
          for (int i = 0; i < 4; ++i) atomicAdd(&h[(w >> (8 * i)) & 255u], 1u);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (zs + i < nz) {
            const unsigned int v = (w >> (8 * i)) & 255u;
            dst[er_idx(i, vol - q)] = (uint8_t)v;
            if (hist) atomicAdd(&h[v], 1u);
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) cur[j] = nxt[j];
  }
  if (hist) {
    __syncthreads();
    if (h[t]) atomicAdd(&hist[256ull * blockIdx.z + t], (unsigned long long)h[t]);
  }
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

extern "C" int er_ingest_u8(const uint8_t* payload_dev, int64_t nx, int64_t ny, int64_t nz,
                            int64_t frames, uint8_t* out_dev, int64_t* hist_dev, void* stream) {
  if (!payload_dev || !out_dev || nx < 1 || ny < 1 || nz < 1 || frames < 0)
    return er_set_error(ER_EINVAL, "er_ingest_u8: args");
  if (nx > INT32_MAX || ny > INT32_MAX || nz > INT32_MAX || frames > 65535)
    return er_set_error(ER_EINVAL, "er_ingest_u8: dims out of range");
  if ((const void*)payload_dev == (const void*)out_dev)
    return er_set_error(ER_EINVAL, "er_ingest_u8: in-place reorder is not supported");
  cudaStream_t st = as_stream(stream);
  if (hist_dev && frames > 0)
    zero_u64_kernel<<<1, 256, 0, st>>>((unsigned long long*)hist_dev, 256 * frames);
  if (frames == 0) {
    ER_CHECK_LAUNCH();
    return ER_OK;
  }
  const int tiles_x = (int)((nx + kIngT - 1) / kIngT), tiles_z = (int)((nz + kIngT - 1) / kIngT);
  const long long tiles = (long long)tiles_x * tiles_z;
  if (tiles > INT32_MAX) return er_set_error(ER_EINVAL, "er_ingest_u8: dims out of range");
  // split y into ~4 waves of 8 blocks per SM (short tail); each block walks its y range
  long long chunks = (ER_NUM_SMS_B200 * 32 + tiles * frames - 1) / (tiles * frames);
  if (chunks < 1) chunks = 1;
  if (chunks > ny) chunks = ny;
  const int y_per_block = (int)((ny + chunks - 1) / chunks);
  chunks = (ny + y_per_block - 1) / y_per_block;
  const bool words_in = (nx % 4 == 0) && (reinterpret_cast<uintptr_t>(payload_dev) % 4 == 0);
  const bool words_out = (nz % 4 == 0) && (reinterpret_cast<uintptr_t>(out_dev) % 4 == 0);
  dim3 grid((unsigned)tiles, (unsigned)chunks, (unsigned)frames);
  ingest_u8_kernel<<<grid, 256, 0, st>>>(payload_dev, (int)nx, (int)ny, (int)nz, tiles_x,
                                         y_per_block, words_in, words_out, out_dev,
                                         (unsigned long long*)hist_dev);
  ER_CHECK_LAUNCH();
  return ER_OK;
}
