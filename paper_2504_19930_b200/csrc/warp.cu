// Frame warping and scoring on device: the reference's resample_trilinear
// (kernels_numba.py:65-85), dice_under_transform (metrics.py:88-93) and the
// two-pass squared NCC of score_frames (metrics.py:49-68, pipeline.py:110-138).
// Samples are computed in fp64 in the reference's exact operation order, so
// warped values -- and therefore the strict '> 0.5' mask cut and every Dice
// count -- are bit-identical to the reference.
#include "common.cuh"

namespace {

constexpr int kRedBlocks = 592;  // 4 x 148 SMs, fixed -> device-independent order
constexpr int kRedThreads = 256;

struct WarpGeom {
  int nx, ny, nz;  // output / reference grid
  int sx, sy, sz;  // source grid
  double a[9], b[3];
  double alpha, gamma;
};

template <typename T>
__device__ __forceinline__ double ld(const T* __restrict__ p, long long i) {
  return (double)__ldg(p + i);
}

__device__ __forceinline__ void cell(double u, int n, int& c0, int& c1, double& f) {
  int a = __double2int_rd(u);
  a = a < 0 ? 0 : a;
  int b = a + 1;
  if (b > n - 1) {
    b = n - 1;
    a = b > 0 ? b - 1 : 0;
  }
  c0 = a;
  c1 = b;
  f = rn_sub(u, (double)a);
}

// Pull-back sample at output voxel q (kernels_numba.py:71-85), in value space.
template <typename ST>
__device__ __forceinline__ double warp_value(const ST* __restrict__ src, const WarpGeom& g,
                                             long long q) {
  const long long row = q / g.nz;
  const int k = (int)(q - row * g.nz);
  const int i = (int)(row / g.ny);
  const int j = (int)(row - (long long)i * g.ny);
  const double di = (double)i, dj = (double)j, dk = (double)k;
  const double u = rn_add(rn_add(rn_add(rn_mul(g.a[0], di), rn_mul(g.a[1], dj)), g.b[0]), rn_mul(g.a[2], dk));
  const double v = rn_add(rn_add(rn_add(rn_mul(g.a[3], di), rn_mul(g.a[4], dj)), g.b[1]), rn_mul(g.a[5], dk));
  const double w = rn_add(rn_add(rn_add(rn_mul(g.a[6], di), rn_mul(g.a[7], dj)), g.b[2]), rn_mul(g.a[8], dk));
  if (!(0.0 <= u && u <= (double)(g.sx - 1) && 0.0 <= v && v <= (double)(g.sy - 1) &&
        0.0 <= w && w <= (double)(g.sz - 1)))
    return 0.0;  // FILL_VALUE
  int i0, i1, j0, j1, k0, k1;
  double fu, fv, fw;
  cell(u, g.sx, i0, i1, fu);
  cell(v, g.sy, j0, j1, fv);
  cell(w, g.sz, k0, k1, fw);
  const long long o00 = ((long long)i0 * g.sy + j0) * g.sz, o01 = ((long long)i0 * g.sy + j1) * g.sz;
  const long long o10 = ((long long)i1 * g.sy + j0) * g.sz, o11 = ((long long)i1 * g.sy + j1) * g.sz;
  const long long ns = (long long)g.sx * g.sy * g.sz;  // er_idx extent (debug builds)
  (void)ns;
  const double gu = rn_sub(1.0, fu), gv = rn_sub(1.0, fv), gw = rn_sub(1.0, fw);
  const double c00 = rn_add(rn_mul(ld(src, er_idx(o00 + k0, ns)), gu), rn_mul(ld(src, er_idx(o10 + k0, ns)), fu));
  const double c10 = rn_add(rn_mul(ld(src, er_idx(o01 + k0, ns)), gu), rn_mul(ld(src, er_idx(o11 + k0, ns)), fu));
  const double c01 = rn_add(rn_mul(ld(src, er_idx(o00 + k1, ns)), gu), rn_mul(ld(src, er_idx(o10 + k1, ns)), fu));
  const double c11 = rn_add(rn_mul(ld(src, er_idx(o01 + k1, ns)), gu), rn_mul(ld(src, er_idx(o11 + k1, ns)), fu));
  const double c0 = rn_add(rn_mul(c00, gv), rn_mul(c10, fv));
  const double c1 = rn_add(rn_mul(c01, gv), rn_mul(c11, fv));
  const double x = rn_add(rn_mul(c0, gw), rn_mul(c1, fw));
  return rn_add(rn_mul(g.alpha, x), g.gamma);
}

template <typename ST>
__global__ void resample_kernel(const ST* __restrict__ src, WarpGeom g, double* __restrict__ out,
                                long long n) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x)
    out[q] = warp_value(src, g, q);
}

template <typename ST, typename TT>
__global__ void dice_counts_kernel(const ST* __restrict__ src, WarpGeom g,
                                   const TT* __restrict__ tgt, double t_alpha, double t_gamma,
                                   long long n, unsigned long long* __restrict__ counts) {
  unsigned long long ca = 0, cb = 0, cab = 0;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const bool a = warp_value(src, g, q) > 0.5;  // binarize(resample(...), 0.5)
    const bool b = rn_add(rn_mul(t_alpha, ld(tgt, q)), t_gamma) == 1.0;
    ca += a;
    cb += b;
    cab += a && b;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ca += __shfl_down_sync(0xffffffffu, ca, o);
    cb += __shfl_down_sync(0xffffffffu, cb, o);
    cab += __shfl_down_sync(0xffffffffu, cab, o);
  }
  if ((threadIdx.x & 31) == 0) {  // integer atomics: exact, order-free
    atomicAdd(counts + 0, ca);
    atomicAdd(counts + 1, cb);
    atomicAdd(counts + 2, cab);
  }
}

__global__ void zero_counts_kernel(unsigned long long* c) {
  if (threadIdx.x < 3) c[threadIdx.x] = 0;
}

__device__ __forceinline__ void block_reduce3(double& a, double& b, double& c, double (*sh)[3]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
    c += __shfl_down_sync(0xffffffffu, c, o);
  }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sh[warp][0] = a;
    sh[warp][1] = b;
    sh[warp][2] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = b = c = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) {
      a += sh[w][0];
      b += sh[w][1];
      c += sh[w][2];
    }
  }
}

// pass 1: sum t, sum s (fixed partition, fixed order)
template <typename TT, typename ST>
__global__ void ncc_pass1_kernel(const TT* __restrict__ tgt, double t_alpha, double t_gamma,
                                 const ST* __restrict__ src, WarpGeom g, int identity,
                                 long long n, double* __restrict__ part) {
  __shared__ double sh[kRedThreads / 32][3];
  const long long lo = n * blockIdx.x / kRedBlocks, hi = n * (blockIdx.x + 1) / kRedBlocks;
  double st = 0.0, ss = 0.0, dummy = 0.0;
  for (long long q = lo + threadIdx.x; q < hi; q += kRedThreads) {
    st += rn_add(rn_mul(t_alpha, ld(tgt, q)), t_gamma);
    ss += identity ? rn_add(rn_mul(g.alpha, ld(src, q)), g.gamma) : warp_value(src, g, q);
  }
  block_reduce3(st, ss, dummy, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = st;
    part[2 * blockIdx.x + 1] = ss;
  }
}

__global__ void ncc_means_kernel(const double* __restrict__ part, long long n,
                                 double* __restrict__ means) {
  if (threadIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int q = 0; q < kRedBlocks; ++q) {
    a += part[2 * q];
    b += part[2 * q + 1];
  }
  means[0] = a / (double)n;
  means[1] = b / (double)n;
}

// pass 2: centred sums (metrics.py:59-66)
template <typename TT, typename ST>
__global__ void ncc_pass2_kernel(const TT* __restrict__ tgt, double t_alpha, double t_gamma,
                                 const ST* __restrict__ src, WarpGeom g, int identity,
                                 long long n, const double* __restrict__ means,
                                 double* __restrict__ part) {
  __shared__ double sh[kRedThreads / 32][3];
  const long long lo = n * blockIdx.x / kRedBlocks, hi = n * (blockIdx.x + 1) / kRedBlocks;
  const double mt = means[0], ms = means[1];
  double tt = 0.0, ssum = 0.0, ts = 0.0;
  for (long long q = lo + threadIdx.x; q < hi; q += kRedThreads) {
    const double dt = rn_add(rn_mul(t_alpha, ld(tgt, q)), t_gamma) - mt;
    const double s = identity ? rn_add(rn_mul(g.alpha, ld(src, q)), g.gamma) : warp_value(src, g, q);
    const double ds = s - ms;
    tt = fma(dt, dt, tt);
    ssum = fma(ds, ds, ssum);
    ts = fma(dt, ds, ts);
  }
  block_reduce3(tt, ssum, ts, sh);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = tt;
    part[3 * blockIdx.x + 1] = ssum;
    part[3 * blockIdx.x + 2] = ts;
  }
}

__global__ void ncc_final_kernel(const double* __restrict__ part, long long n,
                                 double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double a = 0.0, b = 0.0, c = 0.0;
  for (int q = 0; q < kRedBlocks; ++q) {
    a += part[3 * q];
    b += part[3 * q + 1];
    c += part[3 * q + 2];
  }
  out[0] = a;
  out[1] = b;
  out[2] = c;
  out[3] = (double)n;
}

WarpGeom make_geom(const er_volume* src, const double A[9], const double b[3], int nx, int ny,
                   int nz) {
  WarpGeom g;
  g.nx = nx;
  g.ny = ny;
  g.nz = nz;
  g.sx = src->nx;
  g.sy = src->ny;
  g.sz = src->nz;
  for (int q = 0; q < 9; ++q) g.a[q] = A[q];
  for (int q = 0; q < 3; ++q) g.b[q] = b[q];
  g.alpha = src->alpha;
  g.gamma = src->gamma;
  return g;
}

unsigned grid_for(long long n) {
  long long blocks = (n + 255) / 256;
  if (blocks > ER_NUM_SMS_B200 * 8) blocks = ER_NUM_SMS_B200 * 8;
  return (unsigned)(blocks > 0 ? blocks : 1);
}

bool ok_volume(const er_volume* v) {
  return v && v->data_dev && v->dtype >= ER_U8 && v->dtype <= ER_F64 && v->nx > 0 &&
         v->ny > 0 && v->nz > 0;
}

#define ER_DISPATCH_DTYPE(dt, T, ...)                 \
  switch (dt) {                                       \
    case ER_U8: { typedef uint8_t T; __VA_ARGS__; break; } \
    case ER_F32: { typedef float T; __VA_ARGS__; break; }  \
    default: { typedef double T; __VA_ARGS__; break; }     \
  }

}  // namespace

extern "C" int er_resample(const er_volume* src, const double A[9], const double b[3],
                           int32_t nx, int32_t ny, int32_t nz, double* out_dev, void* stream) {
  if (!ok_volume(src) || !A || !b || !out_dev || nx < 1 || ny < 1 || nz < 1)
    return er_set_error(ER_EINVAL, "er_resample: args");
  const WarpGeom g = make_geom(src, A, b, nx, ny, nz);
  const long long n = (long long)nx * ny * nz;
  cudaStream_t st = as_stream(stream);
  ER_DISPATCH_DTYPE(src->dtype, ST,
                    resample_kernel<ST><<<grid_for(n), 256, 0, st>>>((const ST*)src->data_dev, g, out_dev, n));
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_warp_dice_counts(const er_volume* src_mask, const double A[9],
                                   const double b[3], const er_volume* tgt_mask,
                                   int64_t* counts_dev, void* stream) {
  if (!ok_volume(src_mask) || !ok_volume(tgt_mask) || !A || !b || !counts_dev)
    return er_set_error(ER_EINVAL, "er_warp_dice_counts: args");
  const WarpGeom g = make_geom(src_mask, A, b, tgt_mask->nx, tgt_mask->ny, tgt_mask->nz);
  const long long n = (long long)tgt_mask->nx * tgt_mask->ny * tgt_mask->nz;
  cudaStream_t st = as_stream(stream);
  unsigned long long* c = (unsigned long long*)counts_dev;
  zero_counts_kernel<<<1, 32, 0, st>>>(c);
  ER_DISPATCH_DTYPE(src_mask->dtype, ST, {
    ER_DISPATCH_DTYPE(tgt_mask->dtype, TT,
                      dice_counts_kernel<ST, TT><<<grid_for(n), 256, 0, st>>>(
                          (const ST*)src_mask->data_dev, g, (const TT*)tgt_mask->data_dev,
                          tgt_mask->alpha, tgt_mask->gamma, n, c));
  });
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_warp_ncc_sums(const er_volume* tgt, const er_volume* src, const double A[9],
                                const double b[3], int32_t identity, double* out_dev,
                                void* stream) {
  // out_dev must hold 4 + 3 * 592 + 2 doubles (tail is scratch)
  if (!ok_volume(tgt) || !ok_volume(src) || !out_dev || (!identity && (!A || !b)))
    return er_set_error(ER_EINVAL, "er_warp_ncc_sums: args");
  if (identity && (tgt->nx != src->nx || tgt->ny != src->ny || tgt->nz != src->nz))
    return er_set_error(ER_EINVAL, "er_warp_ncc_sums: identity needs equal dims");
  const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, Z[3] = {0, 0, 0};
  const WarpGeom g = make_geom(src, A ? A : I, b ? b : Z, tgt->nx, tgt->ny, tgt->nz);
  const long long n = (long long)tgt->nx * tgt->ny * tgt->nz;
  cudaStream_t st = as_stream(stream);
  double* part = out_dev + 4;
  double* means = out_dev + 4 + 3 * kRedBlocks;
  ER_DISPATCH_DTYPE(tgt->dtype, TT, {
    ER_DISPATCH_DTYPE(src->dtype, ST, {
      ncc_pass1_kernel<TT, ST><<<kRedBlocks, kRedThreads, 0, st>>>(
          (const TT*)tgt->data_dev, tgt->alpha, tgt->gamma, (const ST*)src->data_dev, g,
          identity, n, part);
      ncc_means_kernel<<<1, 32, 0, st>>>(part, n, means);
      ncc_pass2_kernel<TT, ST><<<kRedBlocks, kRedThreads, 0, st>>>(
          (const TT*)tgt->data_dev, tgt->alpha, tgt->gamma, (const ST*)src->data_dev, g,
          identity, n, means, part);
      ncc_final_kernel<<<1, 32, 0, st>>>(part, n, out_dev);
    });
  });
  ER_CHECK_LAUNCH();
  return ER_OK;
}

ER_DEFINE_FAULT_READER(er_faults_warp)
