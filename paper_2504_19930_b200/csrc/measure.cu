// The hot path: fused pull-back trilinear resample + squared NCC, one
// likelihood per particle.  Replaces the reference's _ncc_kernel
// (/root/reference/pkg/src/echoreg/kernels_numba.py:116-189).
//
// Decomposition (B200-first):
//   * one CTA per (particle, tile of target planes), launched tile-major; the
//     tile shape depends only on the target dims, never on P or on the GPU
//     count, so every particle's reduction order is fixed -> results are
//     bitwise identical for any sharding (the reference's worker-invariance
//     contract, kernels_numba.py:6-8).
//   * a warp takes 32 target rows (i, j) at a time; lane r computes row r's
//     in-bounds k-run with the reference's exact fp64 _k_interval
//     (kernels_numba.py:88-113, 156-158) -> the in-bounds voxel set and the
//     overlap count n are bit-exact.  The non-empty rows are compacted by rank
//     and walked by a few lanes each (fast paths: 4 lanes, 8 rows per warp
//     step), lanes strided over k (k is the contiguous axis, volume.py:33).
//   * fast paths (measure_oct_kernel): the source re-laid out per cell (8-bit
//     "oct": 8 corners in one 8-byte word; binary "bit-oct": 8 corner bits;
//     f32/f64 "quad": two float4 per sample), fixed-point coordinates from the
//     reference's fp64 row start (in the pair / mask / fp64 loops stepped as
//     fraction words + one padded cell index per voxel, PTX carry chains:
//     cell_step), fp32 lerps packed fp32x2 across voxel pairs
//     (or fp64 lerps in Q12.52 / Q24.40), fp32 row partials folded into fp64
//     per row.  Generic path (measure_partials_kernel): 8 gathers per voxel,
//     fp64 coordinates exactly as the reference, any storage / lerp mode.
//   * fixed-order warp-shuffle + shared-memory reductions, one 48-byte partial
//     per (particle, tile), fixed-order finalize per particle.  No float
//     atomics anywhere.  fp32-lerp measurements are followed by a device-side
//     refinement pass that re-measures ill-conditioned particles in fp64.
//   * the value affine (value = alpha*stored + gamma, e.g. raw uint8 echo
//     data with the z-score folded in) is applied once per particle in the
//     finalize, so the gather moves 1 byte per corner for uint8 volumes.
//
// Build-time tuning flags (ER_NVCC_EXTRA="-DNAME=V"; the defaults are the
// measured best on the B200, the alternatives are kept for the variant
// scripts tools/variants*.sh and are recorded in profiles/README.md):
//   ER_OCT_LANES=4         lanes per row, lerp modes (ER_OCT_LANES_NEAREST=8,
//                          ER_OCT_LANES_F64, ER_OCT_LANES_QUAD=8; the fp32 byte
//                          path uses 8 when the oct exceeds ER_OCT_BIG_BYTES)
//   ER_OCT_PAIR=1          fp32 byte path: two voxels per lane per step
//   ER_CORNER_XU=1         two of the eight corner conversions on the XU pipe
//   ER_TGT_XU=1            8-bit target values converted on the XU pipe
//   ER_F64_Q52=1           fp64-lerp mode: Q12.52 coordinates + voxel pairs
//   ER_REFINE=1            fp64 refinement of ill-conditioned f32 particles
//   ER_OCT_THREADS=128, ER_OCT_MINBLOCKS_F32=8   fp32-class CTA size / CTAs per SM
//   ER_OCT_MINBLOCKS_NEAREST=10, _F32_OVL=7 (_BITS, _QUAD = 8)  per-path CTAs per SM
//   ER_OCT_THREADS_F64=128, ER_OCT_MINBLOCKS_F64=5  the same for the fp64-lerp kernel
//   ER_OCT_SMEM_ACC=1      per-lane fp64 group accumulators in shared memory
//   ER_OCT_FMUL2=1         u/v fraction scaling as one packed FMUL2 (single voxels)
//   ER_OCT_ACC2=1          px += x; (pxx, pyx) by one FFMA2 of x * (x, y)
//   ER_BITS_EXACT=1        binary sources: integer counts + fp64 boundary cells
//   ER_FRAC_I2F=1          fractions by I2F on the fixed-point low word
//   ER_FRAC_RN=1           ... rounded to nearest (0: truncated, biased low)
//   ER_OCT_TILE_MAJOR=1    tile-major CTA order (0: particle-major)
//   ER_OCT_UNROLL=1        voxel-loop unroll; ER_OCT_LDPOLICY=0 (.nc; 1 .cg, 2 .cs)
//   ER_MIN_TILES=8         minimum tiles per particle
//   ER_BOUNDS_CHECK=0      debug build: every gather index range-checked (common.cuh)
#include <type_traits>

#include "common.cuh"

namespace {

struct Partial {
  double x, xx, yx, y, yy;
  long long n;
};

struct Geom {
  int nx, ny, nz;
  int sx, sy, sz;
  int planes_per_tile, ntiles;
  double limx, limy, limz;
};

constexpr int kThreads = 256;
#ifndef ER_OCT_THREADS
#define ER_OCT_THREADS 128
#endif
// fp64-lerp oct kernel: 128-thread CTAs, 6 per SM (+3.3% over 256 x 3 on C2)
#ifndef ER_OCT_THREADS_F64
#define ER_OCT_THREADS_F64 128
#endif
// oct fast path CTA size per sampling mode
template <int LERP>
struct OctThreads {
  static constexpr int n = LERP == ER_LERP_F64 ? ER_OCT_THREADS_F64 : ER_OCT_THREADS;
  static constexpr int warps = n / 32;
};
constexpr int kWarps = kThreads / 32;
constexpr int kRowsPerTile = 2048;

#ifndef ER_OCT_HALF
#define ER_OCT_HALF 1
#endif
// fp32-lerp measurements: re-measure ill-conditioned particles in fp64 (RefineArgs)
#ifndef ER_REFINE
#define ER_REFINE 1
#endif
// fp64-lerp byte path: Q12.52 coordinates + pair loop where the affine allows
#ifndef ER_F64_Q52
#define ER_F64_Q52 1
#endif
// lanes per target row in the oct kernels (4, 8, 16 or 32; rows per warp =
// 32 / lanes): fewer lanes per row amortise the per-row setup over more rows
// per warp step; 4 is the measured best for the lerp modes (2 loses the
// coalescing), 8 for the nearest mode
#ifndef ER_OCT_LANES
#define ER_OCT_LANES (ER_OCT_HALF ? 4 : 32)
#endif
#ifndef ER_OCT_LANES_F64
#define ER_OCT_LANES_F64 ER_OCT_LANES
#endif
#ifndef ER_OCT_LANES_QUAD
#define ER_OCT_LANES_QUAD 8
#endif
// the fp32 byte path switches to 8 lanes per row above this oct footprint
#ifndef ER_OCT_BIG_BYTES
#define ER_OCT_BIG_BYTES (80LL << 20)
#endif
#ifndef ER_OCT_LANES_NEAREST
#define ER_OCT_LANES_NEAREST (ER_OCT_HALF ? 8 : 32)
#endif
// two of the eight corner conversions of the pair loop on the XU pipe
#ifndef ER_CORNER_XU
#define ER_CORNER_XU 1
#endif
// 8-bit target values to float on the XU pipe (I2F.U8) instead of the ALU (I2FP)
#ifndef ER_TGT_XU
#define ER_TGT_XU 1
#endif

// fp32 byte path: two voxels per lane per step, lerps packed across them
#ifndef ER_OCT_PAIR
#define ER_OCT_PAIR 1
#endif
// bit-oct (binary) path: two voxels per lane per step
#ifndef ER_OCT_PAIR_BITS
#define ER_OCT_PAIR_BITS 1
#endif
// voxels per lane per step of the bit-oct loop: 2 at 4 lanes per row; 4 at
// the 8 lanes per row used for long target rows (nz >= ER_BITS_WIDE_NZ)
#ifndef ER_BITS_NB
#define ER_BITS_NB 2
#endif
#ifndef ER_BITS_NB_WIDE
#define ER_BITS_NB_WIDE 4
#endif
#ifndef ER_BITS_WIDE_NZ
#define ER_BITS_WIDE_NZ 128
#endif
// quad (f32/f64 source) path: two voxels per lane per step
#ifndef ER_OCT_PAIR_QUAD
#define ER_OCT_PAIR_QUAD 1
#endif
#ifndef ER_OCT_UNROLL
#define ER_OCT_UNROLL 1
#endif
// cache policy of the oct gathers: 0 = ld.global.nc (L1 allocate), 1 = .cg
// (L2 only), 2 = .cs (streaming)
#ifndef ER_OCT_LDPOLICY
#define ER_OCT_LDPOLICY 0
#endif
#ifndef ER_FRAC_I2F
#define ER_FRAC_I2F 1
#endif
#ifndef ER_OCT_TILE_MAJOR
#define ER_OCT_TILE_MAJOR 1
#endif
__device__ __forceinline__ uint2 ld_oct(const uint2* p) {
#if ER_OCT_LDPOLICY == 1
  return __ldcg(p);
#elif ER_OCT_LDPOLICY == 2
  return __ldcs(p);
#else
  return __ldg(p);
#endif
}
#define ER_PRAGMA_(x) _Pragma(#x)
#define ER_UNROLL_(n) ER_PRAGMA_(unroll n)
#define ER_UNROLL(n) ER_UNROLL_(n)
#ifndef ER_OCT_MINBLOCKS_F32
#define ER_OCT_MINBLOCKS_F32 8
#endif
#ifndef ER_OCT_MINBLOCKS_F64
// 5 x 128 threads: 88 registers keep the fp64 pair loop's step words
// resident (27.2 vs 28.2 ms on C2 at 6 CTAs without the cell-index stepping)
#define ER_OCT_MINBLOCKS_F64 (5 * 128 / ER_OCT_THREADS_F64)
#endif
// per-path CTAs per SM: nearest-neighbour byte sampling 10 (14.6 vs 16.3 ms
// on C2 at 8: fewer registers, more warps to hide the gathers); the bit-oct
// mask path and the quad layout keep 8 (10 / 12 measured ±0 / slower)
#ifndef ER_OCT_MINBLOCKS_NEAREST
#define ER_OCT_MINBLOCKS_NEAREST 10
#endif
#ifndef ER_OCT_MINBLOCKS_BITS
#define ER_OCT_MINBLOCKS_BITS ER_OCT_MINBLOCKS_F32
#endif
#ifndef ER_OCT_MINBLOCKS_QUAD
#define ER_OCT_MINBLOCKS_QUAD ER_OCT_MINBLOCKS_F32
#endif
// the overlap-region fp32 byte kernel (the extra target sum of squares) at 7:
// 72 registers let ptxas issue both target loads early (19.2 vs 20.2 ms on C2)
#ifndef ER_OCT_MINBLOCKS_F32_OVL
#define ER_OCT_MINBLOCKS_F32_OVL 7
#endif
#ifndef ER_MIN_TILES
#define ER_MIN_TILES 8
#endif
// fp32 paths: keep the per-lane fp64 group accumulators in shared memory
// (touched once per row) instead of 6 registers of the voxel loop
#ifndef ER_OCT_SMEM_ACC
#define ER_OCT_SMEM_ACC 1
#endif
// fp32 paths: scale the u/v fractions with one packed FMUL2
#ifndef ER_OCT_FMUL2
#define ER_OCT_FMUL2 1
#endif
// fp32 paths: accumulate as px += x and (pxx, pyx) += x * (x, y) (one FADD +
// one FFMA2 whose operand pair is two computed values, no 1.0f constant)
#ifndef ER_OCT_ACC2
#define ER_OCT_ACC2 1
#endif
// fractions from the Q32.32 low word: round to nearest (0: truncate; 7 of 32
// full-scale image runs left the reference-order trajectory vs 3 of 32)
#ifndef ER_FRAC_RN
#define ER_FRAC_RN 1
#endif
#if ER_FRAC_RN
#define ER_U2F __uint2float_rn
#else
#define ER_U2F __uint2float_rz
#endif
// bit-oct (binary source) path: uniform cells as exact integer counts, boundary
// cells in fp64 (0: fp32 lerps and fp32 row partials like the byte path)
#ifndef ER_BITS_EXACT
#define ER_BITS_EXACT 1
#endif

// per-voxel fp32 row partials: sum x, sum x^2, sum y*x (both forms round identically)
__device__ __forceinline__ void acc_voxel(float x, float yf, float& px, float& pxx, float& pyx) {
#if ER_OCT_ACC2
  px += x;
  const float2 a = __ffma2_rn(make_float2(x, x), make_float2(x, yf), make_float2(pxx, pyx));
  pxx = a.x;
  pyx = a.y;
#else
  const float2 a = __ffma2_rn(make_float2(x, x), make_float2(1.0f, x), make_float2(px, pxx));
  px = a.x;
  pxx = a.y;
  pyx = fmaf(yf, x, pyx);
#endif
}


// kernels_numba.py:88-113, bit-exact (IEEE division, ceil/floor, same guards)
__device__ __forceinline__ void k_interval(double c0, double slope, double limit, int& klo,
                                           int& khi) {
  if (slope == 0.0) {
    if (!(0.0 <= c0 && c0 <= limit)) {
      klo = 0;
      khi = 0;
    }
    return;
  }
  double lo, hi;
  if (slope > 0.0) {
    lo = rn_div(rn_sub(0.0, c0), slope);
    hi = rn_div(rn_sub(limit, c0), slope);
  } else {
    lo = rn_div(rn_sub(limit, c0), slope);
    hi = rn_div(rn_sub(0.0, c0), slope);
  }
  if (lo > (double)klo) {
    if (lo > (double)khi) {
      klo = 0;
      khi = 0;
      return;
    }
    klo = (int)ceil(lo);
  }
  if (hi < (double)(khi - 1)) {
    if (hi < (double)klo) {
      klo = 0;
      khi = 0;
      return;
    }
    khi = (int)floor(hi) + 1;
  }
}

// clamped cell + fraction (kernels_numba.py:32-55)
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

template <typename T>
__device__ __forceinline__ float ldf(const T* __restrict__ p, int i) {
  return (float)__ldg(p + i);
}
template <typename T>
__device__ __forceinline__ double ldd(const T* __restrict__ p, int i) {
  return (double)__ldg(p + i);
}

// Trilinear sample of the stored source values at in-bounds (u, v, w).
template <typename ST, int LERP>
__device__ __forceinline__ double sample(const ST* __restrict__ src, double u, double v,
                                         double w, const Geom& g) {
  int i0, i1, j0, j1, k0, k1;
  double fu, fv, fw;
  cell(u, g.sx, i0, i1, fu);
  cell(v, g.sy, j0, j1, fv);
  cell(w, g.sz, k0, k1, fw);
  const int o00 = (i0 * g.sy + j0) * g.sz;
  const int o01 = (i0 * g.sy + j1) * g.sz;
  const int o10 = (i1 * g.sy + j0) * g.sz;
  const int o11 = (i1 * g.sy + j1) * g.sz;
  const long long ns = (long long)g.sx * g.sy * g.sz;  // er_idx extent (debug builds)
  (void)ns;
  if (LERP == ER_LERP_NEAREST) {  // fraction >= 0.5 -> upper corner
    const int o = fv >= 0.5 ? (fu >= 0.5 ? o11 : o01) : (fu >= 0.5 ? o10 : o00);
    return ldd(src, er_idx(o + (fw >= 0.5 ? k1 : k0), ns));
  }
  if (LERP == ER_LERP_F32) {
    const float x000 = ldf(src, er_idx(o00 + k0, ns)), x100 = ldf(src, er_idx(o10 + k0, ns));
    const float x010 = ldf(src, er_idx(o01 + k0, ns)), x110 = ldf(src, er_idx(o11 + k0, ns));
    const float x001 = ldf(src, er_idx(o00 + k1, ns)), x101 = ldf(src, er_idx(o10 + k1, ns));
    const float x011 = ldf(src, er_idx(o01 + k1, ns)), x111 = ldf(src, er_idx(o11 + k1, ns));
    const float a = (float)fu, b = (float)fv, c = (float)fw;
    const float c00 = fmaf(a, x100 - x000, x000);
    const float c10 = fmaf(a, x110 - x010, x010);
    const float c01 = fmaf(a, x101 - x001, x001);
    const float c11 = fmaf(a, x111 - x011, x011);
    const float c0 = fmaf(b, c10 - c00, c00);
    const float c1 = fmaf(b, c11 - c01, c01);
    return (double)fmaf(c, c1 - c0, c0);
  } else {
    const double x000 = ldd(src, er_idx(o00 + k0, ns)), x100 = ldd(src, er_idx(o10 + k0, ns));
    const double x010 = ldd(src, er_idx(o01 + k0, ns)), x110 = ldd(src, er_idx(o11 + k0, ns));
    const double x001 = ldd(src, er_idx(o00 + k1, ns)), x101 = ldd(src, er_idx(o10 + k1, ns));
    const double x011 = ldd(src, er_idx(o01 + k1, ns)), x111 = ldd(src, er_idx(o11 + k1, ns));
    if (LERP == ER_LERP_F64) {
      const double c00 = fma(fu, x100 - x000, x000);
      const double c10 = fma(fu, x110 - x010, x010);
      const double c01 = fma(fu, x101 - x001, x001);
      const double c11 = fma(fu, x111 - x011, x011);
      const double c0 = fma(fv, c10 - c00, c00);
      const double c1 = fma(fv, c11 - c01, c01);
      return fma(fw, c1 - c0, c0);
    } else {  // reference order x*(1-f) + y*f, no contraction
      const double gu = rn_sub(1.0, fu), gv = rn_sub(1.0, fv), gw = rn_sub(1.0, fw);
      const double c00 = rn_add(rn_mul(x000, gu), rn_mul(x100, fu));
      const double c10 = rn_add(rn_mul(x010, gu), rn_mul(x110, fu));
      const double c01 = rn_add(rn_mul(x001, gu), rn_mul(x101, fu));
      const double c11 = rn_add(rn_mul(x011, gu), rn_mul(x111, fu));
      const double c0 = rn_add(rn_mul(c00, gv), rn_mul(c10, fv));
      const double c1 = rn_add(rn_mul(c01, gv), rn_mul(c11, fv));
      return rn_add(rn_mul(c0, gw), rn_mul(c1, fw));
    }
  }
}

// fixed-order block reduction of the per-thread sums -> one Partial per CTA
__device__ __forceinline__ void block_write_partial(double sx, double sxx, double syx, double sy,
                                                    double syy, long long cnt,
                                                    Partial* __restrict__ part) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sx += __shfl_down_sync(0xffffffffu, sx, o);
    sxx += __shfl_down_sync(0xffffffffu, sxx, o);
    syx += __shfl_down_sync(0xffffffffu, syx, o);
    sy += __shfl_down_sync(0xffffffffu, sy, o);
    syy += __shfl_down_sync(0xffffffffu, syy, o);
    cnt += __shfl_down_sync(0xffffffffu, cnt, o);
  }
  __shared__ double red[kWarps][5];
  __shared__ long long redn[kWarps];
  if (lane == 0) {
    red[warp][0] = sx;
    red[warp][1] = sxx;
    red[warp][2] = syx;
    red[warp][3] = sy;
    red[warp][4] = syy;
    redn[warp] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Partial out{0.0, 0.0, 0.0, 0.0, 0.0, 0};
    for (int w = 0; w < kWarps; ++w) {
      out.x += red[w][0];
      out.xx += red[w][1];
      out.yx += red[w][2];
      out.y += red[w][3];
      out.yy += red[w][4];
      out.n += redn[w];
    }
    *part = out;
  }
}

// One (particle, tile) of the generic kernel: sums over the tile's rows into
// part[slot].  Ends with the block reduction (its __syncthreads makes it safe
// to call repeatedly from one CTA).
template <typename TT, typename ST, int LERP>
__device__ __forceinline__ void partials_cta(const TT* __restrict__ tgt,
                                             const ST* __restrict__ src,
                                             const double* __restrict__ A,
                                             const double* __restrict__ B, const Geom& g,
                                             long long p, int tile, Partial* __restrict__ part) {
  const double* Ap = A + 9 * p;
  const double* Bp = B + 3 * p;
  const double a00 = Ap[0], a01 = Ap[1], a02 = Ap[2];
  const double a10 = Ap[3], a11 = Ap[4], a12 = Ap[5];
  const double a20 = Ap[6], a21 = Ap[7], a22 = Ap[8];
  const double b0 = Bp[0], b1 = Bp[1], b2 = Bp[2];

  const int i_begin = tile * g.planes_per_tile;
  const int i_end = min(g.nx, i_begin + g.planes_per_tile);
  const int R = (i_end - i_begin) * g.ny;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  double sx = 0.0, sxx = 0.0, syx = 0.0, sy = 0.0, syy = 0.0;
  int cnt = 0;

  for (int base = warp * 32; base < R; base += kThreads) {
    const int r = base + lane;
    int klo = 0, khi = 0, off = 0;
    double u0 = 0.0, v0 = 0.0, w0 = 0.0;
    if (r < R) {
      const int i = i_begin + r / g.ny;
      const int j = r - (r / g.ny) * g.ny;
      const double di = (double)i, dj = (double)j;
      // kernels_numba.py:152-154, left-to-right, no FMA
      u0 = rn_add(rn_add(rn_mul(a00, di), rn_mul(a01, dj)), b0);
      v0 = rn_add(rn_add(rn_mul(a10, di), rn_mul(a11, dj)), b1);
      w0 = rn_add(rn_add(rn_mul(a20, di), rn_mul(a21, dj)), b2);
      khi = g.nz;
      k_interval(u0, a02, g.limx, klo, khi);
      k_interval(v0, a12, g.limy, klo, khi);
      k_interval(w0, a22, g.limz, klo, khi);
      if (khi < klo) khi = klo;
      off = (i * g.ny + j) * g.nz;
    }
    cnt += khi - klo;
    unsigned rows = __ballot_sync(0xffffffffu, khi > klo);
    while (rows) {
      const int q = __ffs(rows) - 1;
      rows &= rows - 1;
      const int qlo = __shfl_sync(0xffffffffu, klo, q);
      const int qhi = __shfl_sync(0xffffffffu, khi, q);
      const int qoff = __shfl_sync(0xffffffffu, off, q);
      const double qu = __shfl_sync(0xffffffffu, u0, q);
      const double qv = __shfl_sync(0xffffffffu, v0, q);
      const double qw = __shfl_sync(0xffffffffu, w0, q);
#pragma unroll 2
      for (int k = qlo + lane; k < qhi; k += 32) {
        const double kd = (double)k;
        // kernels_numba.py:160-162
        const double u = rn_add(qu, rn_mul(a02, kd));
        const double v = rn_add(qv, rn_mul(a12, kd));
        const double w = rn_add(qw, rn_mul(a22, kd));
        const double x = sample<ST, LERP>(src, u, v, w, g);
        const double y = ldd(tgt, er_idx(qoff + k, (long long)g.nx * g.ny * g.nz));
        sx += x;
        sxx = fma(x, x, sxx);
        syx = fma(y, x, syx);
        sy += y;
        syy = fma(y, y, syy);
      }
    }
  }

  block_write_partial(sx, sxx, syx, sy, syy, cnt, part);
}

template <typename TT, typename ST, int LERP>
__global__ void __launch_bounds__(kThreads, 3)
    measure_partials_kernel(const TT* __restrict__ tgt, const ST* __restrict__ src,
                            const double* __restrict__ A, const double* __restrict__ B,
                            const Geom g, Partial* __restrict__ part) {
  const int tile = blockIdx.x % g.ntiles;
  const long long p = blockIdx.x / g.ntiles;
  partials_cta<TT, ST, LERP>(tgt, src, A, B, g, p, tile, part + blockIdx.x);
}

// Refinement pass: the particles the fp32 finalize listed as ill-conditioned
// (list[0 .. *count)) re-measured with the reference-order fp64 arithmetic
// (LERP_EXACT) on the plain copy of the source; a fixed persistent grid walks
// the (particle, tile) items, so nothing is launched per particle and an
// empty list costs one pass of idle CTAs.  Each item overwrites that
// particle's own partial slots (fixed tiling -> the sums are the ones a
// plain `exact` launch produces).
template <typename TT, typename ST>
__global__ void __launch_bounds__(kThreads, 3)
    measure_refine_kernel(const TT* __restrict__ tgt, const ST* __restrict__ src,
                          const double* __restrict__ A, const double* __restrict__ B,
                          const Geom g, Partial* __restrict__ part, const int* __restrict__ list,
                          const int* __restrict__ count) {
  const long long items = (long long)(*count) * g.ntiles;
  for (long long w = blockIdx.x; w < items; w += gridDim.x) {
    const long long p = list[w / g.ntiles];
    const int tile = (int)(w % g.ntiles);
    partials_cta<TT, ST, ER_LERP_EXACT>(tgt, src, A, B, g, p, tile, part + p * g.ntiles + tile);
    __syncthreads();  // the reduction scratch is reused by the next item
  }
}

// ---------------------------------------------------------------------------
// Fast path for 8-bit sources ("oct" layout).  The source is re-laid out once
// per volume so that padded cell (ci, cj, ck) -- floor indices (ci-1, cj-1,
// ck-1) -- holds its 8 trilinear corners in one 8-byte word, corners clamped
// into the grid.  The one-cell pad ring reproduces the reference's clamped
// edge cells (kernels_numba.py:32-55) without per-voxel clamps: a coordinate
// epsilon below 0 or exactly at n-1 lands in a pad cell whose corners give
// the same value.  Per sampled voxel: one LDG.64 for all 8 corners instead of
// 8 byte gathers.  Source coordinates advance in exact Q24.40 fixed point
// from the reference's fp64 row start (error <= 2^-41 (k+1) voxels); the
// in-bounds k-run still comes from the bit-exact fp64 _k_interval.
// ---------------------------------------------------------------------------

// 2^23 + byte as an exact float: PRMT [b, 0, 0, 0x4B]
__device__ __forceinline__ float byte_magic(unsigned w, unsigned sel) {
  return __int_as_float(__byte_perm(w, 0x4B000000u, sel | 0x7650u));
}

// byte b of w as a float on the XU pipe (I2F.U8 with a byte selector)
__device__ __forceinline__ float u8sel_f(unsigned w, int b) {
  float r;
  asm("cvt.rn.f32.u8 %0, %1;" : "=f"(r) : "h"((unsigned short)(w >> (8 * b))));
  return r;
}

// 2^52 + byte as an exact double (no offset removed)
__device__ __forceinline__ double byte_m64(unsigned w, unsigned sel) {
  return __hiloint2double(0x43300000, __byte_perm(w, 0u, sel | 0x4440u));
}


// One step of the cell-index coordinates (the pair and mask loops): fraction words
// (u, v, w) + (lu, lv, lw) with the carries as explicit PTX carry chains; the
// cell index moves by h (the step's integer parts times the strides) plus
// cyz / cz / 1 for each carried axis.
__device__ __forceinline__ int cell_step(unsigned u, unsigned v, unsigned w, int cell, unsigned lu,
                                         unsigned lv, unsigned lw, int h, int cyz, int cz,
                                         unsigned& ou, unsigned& ov, unsigned& ow) {
  int out;
  asm("{\n\t.reg .u32 fu, fv;\n\t.reg .pred pu, pv;\n\t"
      "add.cc.u32 %0, %4, %8;\n\t"
      "addc.u32 fu, 0, 0;\n\t"
      "add.cc.u32 %1, %5, %9;\n\t"
      "addc.u32 fv, 0, 0;\n\t"
      "add.cc.u32 %2, %6, %10;\n\t"
      "addc.u32 %3, %7, %11;\n\t"
      "setp.ne.u32 pu, fu, 0;\n\t"
      "setp.ne.u32 pv, fv, 0;\n\t"
      "selp.u32 fu, %12, 0, pu;\n\t"
      "selp.u32 fv, %13, 0, pv;\n\t"
      "add.u32 %3, %3, fu;\n\t"
      "add.u32 %3, %3, fv;\n\t}"
      : "=r"(ou), "=r"(ov), "=r"(ow), "=r"(out)
      : "r"(u), "r"(v), "r"(w), "r"(cell), "r"(lu), "r"(lv), "r"(lw), "r"(h), "r"(cyz), "r"(cz));
  return out;
}

// Fixed-point source coordinates with FB fractional bits.  FB = 32 (fp32
// lerps): the integer part is the high register, the fraction the low one.
// FB = 40 (fp64 lerps): 40-bit fractions, error <= 2^-41 (k+1) voxels.
template <int FB>
struct Fix {
  static constexpr double kScale = (double)(1ULL << FB);
  __device__ __forceinline__ static int ipart(long long q) { return (int)(q >> FB); }
  __device__ __forceinline__ static float frac32(long long q) {
#if ER_FRAC_I2F
    if (FB == 32) return ER_U2F((unsigned)q) * 2.3283064365386963e-10f;  // 2^-32
#endif
    // top 23 fraction bits -> [1, 2) - 1
    const unsigned m = (unsigned)((unsigned long long)q >> (FB - 23)) & 0x7FFFFFu;
    return __int_as_float(0x3F800000u | m) - 1.0f;
  }
  __device__ __forceinline__ static double frac64(long long q) {
    const unsigned long long m = ((unsigned long long)q << (64 - FB)) >> 12;
    return __longlong_as_double(0x3FF0000000000000ULL | m) - 1.0;
  }
};

// Per-lane accumulation of the target terms sum y (and sum y^2, which only the
// overlap region needs: the full region takes the target totals from the
// precomputed moments, kernels_numba.py:172-177 -- OVL = 0 drops it).
//   * 8-bit targets: exact integer sums, folded into fp64 once per 32-row group;
//     the value handed to the y*x product is the exact byte as a float.
//   * fp32/fp64-stored targets in the fp32-class modes: fp32 row partials, folded
//     into fp64 at every row end (kRowFold), like the source partials.
//   * fp32/fp64-stored targets in the fp64-lerp mode: fp64 throughout, and the
//     y*x product sees the unrounded stored value.
template <typename TT, int LERP, int OVL>
struct TgtAcc {
  using V = typename std::conditional<LERP == ER_LERP_F64, double, float>::type;
  static constexpr bool kRowFold = LERP != ER_LERP_F64;
  V y = 0, yy = 0;
  __device__ __forceinline__ V add(TT v) {
    const V f = (V)v;
    y += f;
    if (OVL) yy = fma(f, f, yy);
    return f;
  }
  __device__ __forceinline__ void fold(double& sy, double& syy) {
    sy += (double)y;
    syy += (double)yy;
    y = yy = 0;
  }
};

template <int LERP, int OVL>
struct TgtAcc<uint8_t, LERP, OVL> {
  using V = float;
  static constexpr bool kRowFold = false;
  unsigned y = 0, yy = 0;
  __device__ __forceinline__ float add(uint8_t v) {
    y += v;
    if (OVL) yy += (unsigned)v * v;
    return __uint2float_rn(v);
  }
  // two voxels at once (one 3-input add)
  __device__ __forceinline__ float2 add2(uint8_t a, uint8_t b) {
    y += (unsigned)a + (unsigned)b;
    if (OVL) yy += (unsigned)a * a + (unsigned)b * b;
    return make_float2(u8f(a), u8f(b));
  }
  __device__ __forceinline__ static float u8f(uint8_t v) {
#if ER_TGT_XU
    float r;
    asm("cvt.rn.f32.u8 %0, %1;" : "=f"(r) : "h"((unsigned short)v));
    return r;
#else
    return __uint2float_rn(v);
#endif
  }
  __device__ __forceinline__ void fold(double& sy, double& syy) {
    sy += (double)y;
    syy += (double)yy;
    y = yy = 0;
  }
};

template <typename TT, int LERP, int OVL>
__device__ __forceinline__ float2 tgt_add2(TgtAcc<TT, LERP, OVL>& t, TT a, TT b) {
  const float fa = (float)t.add(a);
  const float fb = (float)t.add(b);
  return make_float2(fa, fb);
}
template <int LERP, int OVL>
__device__ __forceinline__ float2 tgt_add2(TgtAcc<uint8_t, LERP, OVL>& t, uint8_t a, uint8_t b) {
  return t.add2(a, b);
}

__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}

// fp32 trilinear sample of one oct cell (8 corner bytes), packed fp32x2:
// corners paired along k so the u-lerps yield (c00, c01) and (c10, c11) and the
// v-lerp runs packed too.  2^23-offset floats: their differences are exact, and
// so is removing the offset.
__device__ __forceinline__ float lerp_oct_f32(uint2 c8, float fu, float fv, float fw) {
  const float2 P0 = make_float2(byte_magic(c8.x, 0), byte_magic(c8.y, 0));
  const float2 P1 = make_float2(byte_magic(c8.x, 1), byte_magic(c8.y, 1));
  const float2 Q0 = make_float2(byte_magic(c8.x, 2), byte_magic(c8.y, 2));
  const float2 Q1 = make_float2(byte_magic(c8.x, 3), byte_magic(c8.y, 3));
  const float2 off2 = make_float2(-8388608.0f, -8388608.0f);
  const float2 fu2 = make_float2(fu, fu), fv2 = make_float2(fv, fv);
  const float2 cP = __ffma2_rn(fu2, f2sub(P1, P0), __fadd2_rn(P0, off2));  // (c00, c01)
  const float2 cQ = __ffma2_rn(fu2, f2sub(Q1, Q0), __fadd2_rn(Q0, off2));  // (c10, c11)
  const float2 c = __ffma2_rn(fv2, f2sub(cQ, cP), cP);                      // (c0, c1)
  return fmaf(fw, c.y - c.x, c.x);
}

// The same sample for two voxels a, b at once, packed ACROSS the voxels: every
// lerp of the chain (u, v and w) is one FFMA2, the fractions arrive as pairs,
// and the per-element operations are exactly those of lerp_oct_f32, so each
// sample is bit-identical to the single-voxel form.
__device__ __forceinline__ float2 lerp_oct_f32x2(uint2 a8, uint2 b8, float2 fu, float2 fv,
                                                 float2 fw) {
  const float2 off2 = make_float2(-8388608.0f, -8388608.0f);
#if ER_CORNER_XU
  // the (x000, x100) pair converted on the XU pipe (I2F.U8 with a byte
  // selector, exact values, no offset), the other six corners by PRMT on the
  // ALU pipe: balances the two pipes
  const float2 x000 = make_float2(u8sel_f(a8.x, 0), u8sel_f(b8.x, 0));
  const float2 x100 = make_float2(u8sel_f(a8.x, 1), u8sel_f(b8.x, 1));
#else
  const float2 x000 = make_float2(byte_magic(a8.x, 0), byte_magic(b8.x, 0));
  const float2 x100 = make_float2(byte_magic(a8.x, 1), byte_magic(b8.x, 1));
#endif
  const float2 x010 = make_float2(byte_magic(a8.x, 2), byte_magic(b8.x, 2));
  const float2 x110 = make_float2(byte_magic(a8.x, 3), byte_magic(b8.x, 3));
  const float2 x001 = make_float2(byte_magic(a8.y, 0), byte_magic(b8.y, 0));
  const float2 x101 = make_float2(byte_magic(a8.y, 1), byte_magic(b8.y, 1));
  const float2 x011 = make_float2(byte_magic(a8.y, 2), byte_magic(b8.y, 2));
  const float2 x111 = make_float2(byte_magic(a8.y, 3), byte_magic(b8.y, 3));
#if ER_CORNER_XU
  const float2 c00 = __ffma2_rn(fu, f2sub(x100, x000), x000);
#else
  const float2 c00 = __ffma2_rn(fu, f2sub(x100, x000), __fadd2_rn(x000, off2));
#endif
  const float2 c10 = __ffma2_rn(fu, f2sub(x110, x010), __fadd2_rn(x010, off2));
  const float2 c01 = __ffma2_rn(fu, f2sub(x101, x001), __fadd2_rn(x001, off2));
  const float2 c11 = __ffma2_rn(fu, f2sub(x111, x011), __fadd2_rn(x011, off2));
  const float2 c0 = __ffma2_rn(fv, f2sub(c10, c00), c00);
  const float2 c1 = __ffma2_rn(fv, f2sub(c11, c01), c01);
  return __ffma2_rn(fw, f2sub(c1, c0), c0);
}

// Q12.52 coordinates of the fp64-lerp byte path (kQ52Path)
__device__ __forceinline__ int q52_ipart(long long q) { return (int)(q >> 52); }

// The fractional part of a Q12.52 coordinate as an exact double: its 52
// fraction bits become the mantissa of 1 + f (one LOP3 on the high word).
__device__ __forceinline__ double q52_frac(long long q) {
  return __hiloint2double((int)((((unsigned)((unsigned long long)q >> 32)) & 0xFFFFFu) |
                                0x3FF00000u),
                          (int)(unsigned)q) - 1.0;
}

// 2^52 + byte * 2^40 as an exact double: the byte goes into bits 8..15 of
// the high word (one PRMT), the low word is 0.
__device__ __forceinline__ double byte_hi52(unsigned w, unsigned sel) {
  return __hiloint2double((int)__byte_perm(w, 0x43300000u, 0x7604u | (sel << 4)), 0);
}

// fp64 trilinear sample of one oct cell from Q12.52 coordinates, in units of
// 2^-40 (the corners are 2^52 + byte * 2^40, integers below 2^53).  The whole
// lerp chain runs on the 2^52-offset values: every difference cancels the
// offset exactly, every lerp result is 2^52 + value rounded to one unit
// (2^-41 byte), and the offset is removed once at the end -- one DADD instead
// of one per base corner.
__device__ __forceinline__ double lerp_q52f(uint2 c8, double fu, double fv, double fw) {
  const double m000 = byte_hi52(c8.x, 0), m100 = byte_hi52(c8.x, 1);
  const double m010 = byte_hi52(c8.x, 2), m110 = byte_hi52(c8.x, 3);
  const double m001 = byte_hi52(c8.y, 0), m101 = byte_hi52(c8.y, 1);
  const double m011 = byte_hi52(c8.y, 2), m111 = byte_hi52(c8.y, 3);
  const double c00 = fma(fu, m100 - m000, m000);
  const double c10 = fma(fu, m110 - m010, m010);
  const double c01 = fma(fu, m101 - m001, m001);
  const double c11 = fma(fu, m111 - m011, m011);
  const double c0 = fma(fv, c10 - c00, c00);
  const double c1 = fma(fv, c11 - c01, c01);
  return fma(fw, c1 - c0, c0) - 4503599627370496.0;
}
__device__ __forceinline__ double lerp_q52(uint2 c8, long long cu, long long cv, long long cw) {
  return lerp_q52f(c8, q52_frac(cu), q52_frac(cv), q52_frac(cw));
}

// Q12.52 coordinates as (64-bit fraction words, padded cell index) for the
// fp64 pair loop: the 52 fraction bits shifted to the top
// of a 64-bit word, so fraction carries are the hardware carries.
__device__ __forceinline__ void q52_split(long long q, unsigned& lo, unsigned& hi) {
  const unsigned long long f = (unsigned long long)q << 12;
  lo = (unsigned)f;
  hi = (unsigned)(f >> 32);
}
// exact double of the fraction: its 52 bits are the mantissa of 1 + f
__device__ __forceinline__ double q64_frac(unsigned lo, unsigned hi) {
  return __hiloint2double((int)((hi >> 12) | 0x3FF00000u), (int)__funnelshift_r(lo, hi, 12)) -
         1.0;
}
// one step: 64-bit fraction words + 64-bit step words (explicit PTX carry
// chains), the cell index moved by h plus the strides of the carried axes
__device__ __forceinline__ int cell_step64(const unsigned (&a)[6], int cell, const unsigned (&d)[6],
                                           int h, int cyz, int cz, unsigned (&o)[6]) {
  int out;
  asm("{\n\t.reg .u32 fu, fv;\n\t.reg .pred pu, pv;\n\t"
      "add.cc.u32 %0, %7, %13;\n\t"
      "addc.cc.u32 %1, %8, %14;\n\t"
      "addc.u32 fu, 0, 0;\n\t"
      "add.cc.u32 %2, %9, %15;\n\t"
      "addc.cc.u32 %3, %10, %16;\n\t"
      "addc.u32 fv, 0, 0;\n\t"
      "add.cc.u32 %4, %11, %17;\n\t"
      "addc.cc.u32 %5, %12, %18;\n\t"
      "addc.u32 %6, %19, %20;\n\t"
      "setp.ne.u32 pu, fu, 0;\n\t"
      "setp.ne.u32 pv, fv, 0;\n\t"
      "selp.u32 fu, %21, 0, pu;\n\t"
      "selp.u32 fv, %22, 0, pv;\n\t"
      "add.u32 %6, %6, fu;\n\t"
      "add.u32 %6, %6, fv;\n\t}"
      : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(out)
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(d[0]), "r"(d[1]),
        "r"(d[2]), "r"(d[3]), "r"(d[4]), "r"(d[5]), "r"(cell), "r"(h), "r"(cyz), "r"(cz));
  return out;
}

// fp32 trilinear sample from two quad entries (planes k0, k1), each
// (x[i0][j0], x[i0][j1], x[i1][j0], x[i1][j1]): u-lerps packed over j.
__device__ __forceinline__ float lerp_quad(float4 q0, float4 q1, float fu, float fv, float fw) {
  const float2 fu2 = make_float2(fu, fu);
  const float2 a0 = make_float2(q0.x, q0.y), a1 = make_float2(q1.x, q1.y);
  const float2 p0 = __ffma2_rn(fu2, f2sub(make_float2(q0.z, q0.w), a0), a0);  // (c00, c10)
  const float2 p1 = __ffma2_rn(fu2, f2sub(make_float2(q1.z, q1.w), a1), a1);  // (c01, c11)
  const float c0 = fmaf(fv, p0.y - p0.x, p0.x);
  const float c1 = fmaf(fv, p1.y - p1.x, p1.x);
  return fmaf(fw, c1 - c0, c0);
}

// Bit-oct boundary cell (corner bits neither all 0 nor all 1): the trilinear
// sample in fp64 from the exact 32-bit fractions of Q32.32 coordinates, added
// to the lane's fp64 accumulators in shared memory.  The u-lerp of two 0/1
// corners is 0, fu, 1 - fu (exact for a 32-bit fraction) or 1 -- the values
// fma(fu, b1 - b0, b0) takes -- so it is done by selects.
__device__ __forceinline__ void bits_boundary(unsigned c, long long cu, long long cv,
                                              long long cw, double y, double3& acc) {
  using F = Fix<32>;
  const double fu = F::frac64(cu), fv = F::frac64(cv), fw = F::frac64(cw);
  const double gu = 1.0 - fu;
  auto pair = [c, fu, gu](int b) {
    const unsigned lo = (c >> b) & 1u, hi = (c >> (b + 1)) & 1u;
    return lo ? (hi ? 1.0 : gu) : (hi ? fu : 0.0);
  };
  const double c00 = pair(0), c10 = pair(2), c01 = pair(4), c11 = pair(6);
  const double c0 = fma(fv, c10 - c00, c00);
  const double c1 = fma(fv, c11 - c01, c01);
  const double x = fma(fw, c1 - c0, c0);
  double3 a = acc;
  a.x += x;
  a.y = fma(x, x, a.y);
  a.z = fma(y, x, a.z);
  acc = a;
}

struct RowRec {  // one target row of a 32-row group, in fixed point
  long long fu0, fv0, fw0;
  int klo, khi, off, pad;
};

struct OctGeom {
  int cy, cz;  // padded cell counts along j and k (sy + 1, sz + 1)
  long long P; // particles in the launch (tile-major block order)
};


// BITS = 1: `oct` points at the bit-oct layout of a binary source (1 byte per
// cell); BITS = 2: at the quad layout of an f32/f64-stored source (two
// adjacent float4 per sample, er_build_quad).  OVL = 1: the overlap region (sum y^2 over the in-bounds voxels is
// accumulated; the full region takes it from the target moments).
// Lanes per target row by default (LN = 0): 4 for the lerp modes, 8 for nearest
// and for the quad layout (two 16-byte loads per sample: fewer lanes per row
// lose too much coalescing); the fp32 byte path is launched with 8 when the
// oct source is too large to stay L2-resident (C5's 256^3: 136 MB).
template <int LERP, int BITS, int LN>
struct OctLanes {
  static constexpr int n = LN ? LN
                           : LERP == ER_LERP_NEAREST ? ER_OCT_LANES_NEAREST
                           : LERP == ER_LERP_F64     ? ER_OCT_LANES_F64
                           : BITS == 2               ? ER_OCT_LANES_QUAD
                                                     : ER_OCT_LANES;
};

template <int LERP, int BITS, int OVL>
struct OctMinBlocks {
  static constexpr int n = LERP == ER_LERP_F64 ? ER_OCT_MINBLOCKS_F64
                           : BITS == 1         ? ER_OCT_MINBLOCKS_BITS
                           : BITS == 2         ? ER_OCT_MINBLOCKS_QUAD
                           : LERP == ER_LERP_NEAREST ? ER_OCT_MINBLOCKS_NEAREST
                           : OVL                     ? ER_OCT_MINBLOCKS_F32_OVL
                                                     : ER_OCT_MINBLOCKS_F32;
};

template <typename TT, int LERP, int BITS, int OVL, int LN = 0>
__global__ void __launch_bounds__(OctThreads<LERP>::n, OctMinBlocks<LERP, BITS, OVL>::n)
    measure_oct_kernel(const TT* __restrict__ tgt, const uint2* __restrict__ oct,
                       const double* __restrict__ A, const double* __restrict__ B, const Geom g,
                       const OctGeom og, Partial* __restrict__ part) {
  // fp32-class modes (fp32 lerps, nearest) use Q32.32 coordinates and fp32 row partials
  constexpr bool kF32 = LERP != ER_LERP_F64;
  using F = Fix<kF32 ? 32 : 40>;
  using Acc = TgtAcc<TT, LERP, OVL>;
#if ER_OCT_TILE_MAJOR
  // tile-major launch order: the CTAs resident at any moment work on the same
  // target slab for many particles, so the union of their source footprints
  // (and the shared target slab) stays L2-resident even when the oct volume
  // does not fit (256^3: 136 MB)
  const int tile = (int)(blockIdx.x / og.P);
  const long long p = blockIdx.x - (long long)tile * og.P;
#else
  const int tile = blockIdx.x % g.ntiles;
  const long long p = blockIdx.x / g.ntiles;
#endif
  const long long slot = p * g.ntiles + tile;
  // the particle's affine lives in shared memory: it is only needed once per
  // 32-row group, and keeping 12 doubles out of the registers of the inner
  // loop is what lets this kernel run 3 CTAs/SM without spills
  __shared__ double sab[12];
  if (threadIdx.x < 12)
    sab[threadIdx.x] = threadIdx.x < 9 ? A[9 * p + threadIdx.x] : B[3 * p + threadIdx.x - 9];
  __syncthreads();
  // fp64-lerp byte path: Q12.52 coordinates (a fraction is one masked high
  // word; see lerp_q52) whenever the particle's affine keeps every coordinate
  // of the tile inside +-2^11 voxels -- a uniform per-CTA guard; else Q24.40
  constexpr bool kQ52Path = ER_F64_Q52 && LERP == ER_LERP_F64 && BITS == 0;
  bool q52 = false;
  if (kQ52Path) {
    const double mu = fabs(sab[9]) + fabs(sab[0]) * g.nx + fabs(sab[1]) * g.ny +
                      fabs(sab[2]) * g.nz;
    const double mv = fabs(sab[10]) + fabs(sab[3]) * g.nx + fabs(sab[4]) * g.ny +
                      fabs(sab[5]) * g.nz;
    const double mw = fabs(sab[11]) + fabs(sab[6]) * g.nx + fabs(sab[7]) * g.ny +
                      fabs(sab[8]) * g.nz;
    q52 = fmax(mu, fmax(mv, mw)) < 2000.0;
  }
  const double kscale = q52 ? 4503599627370496.0 : F::kScale;  // 2^52 or 2^FB
  // fixed-point per-k increments (exact integer stepping along the row)
  const long long du = __double2ll_rn(sab[2] * kscale);
  const long long dv = __double2ll_rn(sab[5] * kscale);
  const long long dw = __double2ll_rn(sab[8] * kscale);

  const int i_begin = tile * g.planes_per_tile;
  const int i_end = min(g.nx, i_begin + g.planes_per_tile);
  const int R = (i_end - i_begin) * g.ny;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cyz = og.cy * og.cz;
  const long long ncells = (long long)(g.sx + 1) * cyz;   // er_idx extents (debug builds)
  const long long ntv = (long long)g.nx * g.ny * g.nz;
  (void)ncells;
  (void)ntv;

  // 32-row groups are handed out dynamically (warps whose rows are short or
  // out of bounds take more groups); each group's warp-reduced sums land in
  // the group's own shared slot and the slots are summed in group order, so
  // the result does not depend on which warp ran which group.
  __shared__ double gsum[kRowsPerTile / 32][5];
  __shared__ int next_group;
  constexpr int kOctThreads = OctThreads<LERP>::n;
  constexpr int kOctWarps = OctThreads<LERP>::warps;
  constexpr bool kBits = BITS == 1, kQuad = BITS == 2;
  static_assert(!kQuad || LERP == ER_LERP_F32, "the quad layout serves the fp32-lerp mode");
  constexpr bool kSmemAcc = ER_OCT_SMEM_ACC && (kF32 || kBits);
  constexpr bool kTgtRowFold = Acc::kRowFold && (kF32 || kBits);
  __shared__ RowRec rrec[kOctWarps][32];
  __shared__ double3 racc[kSmemAcc ? kOctThreads : 1];
  // fp64 row folds of the target terms of fp32/fp64-stored targets
  __shared__ double2 tacc[kTgtRowFold ? kOctThreads : 1];
  const int ngroups = (R + 31) / 32;  // <= kRowsPerTile / 32 (make_geom)
  if (threadIdx.x == 0) next_group = kOctWarps;
  __syncthreads();
  int cnt = 0;
  // kLanes lanes per row: 32 (one row at a time) or 16 (two rows side by
  // side on the half-warps: for nz = 208 = 13 x 16 no lane idles at the row
  // end, and each lane's per-row overhead is paid over twice the voxels)
  constexpr int kLanes = OctLanes<LERP, BITS, LN>::n;
  constexpr int kRowsPerWarp = 32 / kLanes;
  const int sub = lane & (kLanes - 1);
  // fp32 byte path: voxels k and k + kLanes of a lane are sampled together
  constexpr bool kPair = ER_OCT_PAIR && LERP == ER_LERP_F32 && !BITS;
  constexpr bool kPairBits = ER_OCT_PAIR_BITS && ER_BITS_EXACT && kBits &&
                             (LERP == ER_LERP_F32 || LERP == ER_LERP_NEAREST);
  constexpr bool kPairQuad = ER_OCT_PAIR_QUAD && kQuad;
  const long long du1 = kLanes * du, dv1 = kLanes * dv, dw1 = kLanes * dw;
  long long du2 = 2 * du1, dv2 = 2 * dv1, dw2 = 2 * dw1;

  for (int grp = warp; grp < ngroups;) {
    const int r = grp * 32 + lane;
    int klo = 0, khi = 0, off = 0;
    double u0 = 0.0, v0 = 0.0, w0 = 0.0;
    if (r < R) {
      const int i = i_begin + r / g.ny;
      const int j = r - (r / g.ny) * g.ny;
      const double di = (double)i, dj = (double)j;
      u0 = rn_add(rn_add(rn_mul(sab[0], di), rn_mul(sab[1], dj)), sab[9]);
      v0 = rn_add(rn_add(rn_mul(sab[3], di), rn_mul(sab[4], dj)), sab[10]);
      w0 = rn_add(rn_add(rn_mul(sab[6], di), rn_mul(sab[7], dj)), sab[11]);
      khi = g.nz;
      k_interval(u0, sab[2], g.limx, klo, khi);
      k_interval(v0, sab[5], g.limy, klo, khi);
      k_interval(w0, sab[8], g.limz, klo, khi);
      if (khi < klo) khi = klo;
      off = (i * g.ny + j) * g.nz;
    }
    cnt += khi - klo;
    // per-lane group partials: fp32 (LERP_F32) or fp64, exact ints for u8 targets
    Acc ty;
    float px = 0.f, pxx = 0.f, pyx = 0.f;
    double qx = 0.0, qxx = 0.0, qyx = 0.0;
    // bit-oct exact path: voxels sampling exactly 1, and their target sum (u8 targets)
    unsigned ones = 0u, ones_y = 0u;
    constexpr bool kU8Tgt = sizeof(TT) == 1;
    if (kSmemAcc) racc[threadIdx.x] = make_double3(0.0, 0.0, 0.0);
    if (kTgtRowFold) tacc[threadIdx.x] = make_double2(0.0, 0.0);
    // row start in fixed point (per lane: its own row)
    // (the +1.0 voxel shift to the padded cell index is an exact integer add,
    // so the cell index below is a plain non-negative 32-bit IMAD chain)
    const long long one = 1LL << (q52 ? 52 : (kF32 ? 32 : 40));
    // the lane's row record goes to shared memory (broadcast reads below), so
    // it does not occupy registers across the voxel loop
    // non-empty rows only, compacted in row order: the lane's record goes to
    // the slot of its rank among them, so each step of the row loop below
    // takes the next kRowsPerWarp records with one shared-memory read
    const unsigned rows = __ballot_sync(0xffffffffu, khi > klo);
    const int nrows = __popc(rows);
    if (khi > klo) {
      RowRec& mine = rrec[warp][__popc(rows & ((1u << lane) - 1u))];
      mine.fu0 = __double2ll_rn(u0 * kscale) + one;
      mine.fv0 = __double2ll_rn(v0 * kscale) + one;
      mine.fw0 = __double2ll_rn(w0 * kscale) + one;
      mine.klo = klo;
      mine.khi = khi;
      mine.off = off;
    }
    __syncwarp();
    const int myslot = lane / kLanes;
    for (int base = 0; base < nrows; base += kRowsPerWarp) {
      const int q = base + myslot < nrows ? base + myslot : -1;
      int qhi = 0, k0 = 1, toff = 0;
      long long cu = 0, cv = 0, cw = 0;
      if (q >= 0) {
        const RowRec& rq = rrec[warp][q];
        qhi = rq.khi;
        k0 = rq.klo + sub;
        toff = rq.off;
        cu = rq.fu0 + (long long)k0 * du;
        cv = rq.fv0 + (long long)k0 * dv;
        cw = rq.fw0 + (long long)k0 * dw;
      }
      int k = k0;
      if (kQ52Path && q52) {
        // fp64 lerps in Q12.52: two voxels per lane per step (k, k + kLanes)
        // sharing the loop test and the target address; samples carry a 2^40
        // scale (lerp_q52), removed exactly when the group is folded
        int ti = toff + k;
        const int ti_end = toff + qhi - kLanes;
        // cell-index stepping with 64-bit fraction words (cell_step64);
        // bit-identical to plain Q12.52 arithmetic (the low 12 bits of the
        // fraction words stay 0)
        unsigned a[6], d1[6], d2[6];
        q52_split(cu, a[0], a[1]);
        q52_split(cv, a[2], a[3]);
        q52_split(cw, a[4], a[5]);
        q52_split(du1, d1[0], d1[1]);
        q52_split(dv1, d1[2], d1[3]);
        q52_split(dw1, d1[4], d1[5]);
        q52_split(du2, d2[0], d2[1]);
        q52_split(dv2, d2[2], d2[3]);
        q52_split(dw2, d2[4], d2[5]);
        int cella = (q52_ipart(cu) * og.cy + q52_ipart(cv)) * og.cz + q52_ipart(cw);
        const int h1 = q52_ipart(du1) * cyz + q52_ipart(dv1) * og.cz + q52_ipart(dw1);
        const int h2 = q52_ipart(du2) * cyz + q52_ipart(dv2) * og.cz + q52_ipart(dw2);
        const int ti0 = ti;
        for (; ti < ti_end; ti += 2 * kLanes) {
          unsigned b[6];
          const int cellb = cell_step64(a, cella, d1, h1, cyz, og.cz, b);
          const uint2 a8 = ld_oct(oct + (unsigned)er_idx(cella, ncells));
          const uint2 b8 = ld_oct(oct + (unsigned)er_idx(cellb, ncells));
          const TT* tp = tgt + (unsigned)er_idx(ti, ntv);
          const double ya = (double)ty.add(__ldg(tp));
          const double yb = (double)ty.add(__ldg(tp + kLanes));
          const double xa = lerp_q52f(a8, q64_frac(a[0], a[1]), q64_frac(a[2], a[3]),
                                      q64_frac(a[4], a[5]));
          const double xb = lerp_q52f(b8, q64_frac(b[0], b[1]), q64_frac(b[2], b[3]),
                                      q64_frac(b[4], b[5]));
          qx += xa;
          qxx = fma(xa, xa, qxx);
          qyx = fma(ya, xa, qyx);
          qx += xb;
          qxx = fma(xb, xb, qxx);
          qyx = fma(yb, xb, qyx);
          cella = cell_step64(a, cella, d2, h2, cyz, og.cz, a);
        }
        {
          const long long np = (ti - ti0) / (2 * kLanes);
          cu += np * du2;
          cv += np * dv2;
          cw += np * dw2;
        }
        if (ti < toff + qhi) {  // this lane's last voxel, unpaired
          const int ca = (q52_ipart(cu) * og.cy + q52_ipart(cv)) * og.cz + q52_ipart(cw);
          const uint2 a8 = ld_oct(oct + (unsigned)er_idx(ca, ncells));
          const double ya = (double)ty.add(__ldg(tgt + (unsigned)er_idx(ti, ntv)));
          const double xa = lerp_q52(a8, cu, cv, cw);
          qx += xa;
          qxx = fma(xa, xa, qxx);
          qyx = fma(ya, xa, qyx);
        }
        k = qhi;
      }
      if (kPairQuad) {
        // quad layout, two voxels per lane per step (k and k + kLanes): four
        // 16-byte gathers in flight per lane, shared loop test and target
        // address; per voxel exactly the single-voxel arithmetic
        int ti = toff + k;
        const int ti_end = toff + qhi - kLanes;
        const float4* __restrict__ qd = reinterpret_cast<const float4*>(oct);
        const float s32 = 2.3283064365386963e-10f;  // 2^-32
        long long bu = cu + du1, bv = cv + dv1, bw = cw + dw1;
        for (; ti < ti_end; ti += 2 * kLanes) {
          const int ca = (F::ipart(cu) * og.cy + F::ipart(cv)) * og.cz + F::ipart(cw);
          const int cb = (F::ipart(bu) * og.cy + F::ipart(bv)) * og.cz + F::ipart(bw);
          const float4* qa = qd + (unsigned)er_idx(ca, ncells - 1);
          const float4* qb = qd + (unsigned)er_idx(cb, ncells - 1);
          const float4 a0 = __ldg(qa), a1 = __ldg(qa + 1), b0 = __ldg(qb), b1 = __ldg(qb + 1);
          const TT* tp = tgt + (unsigned)er_idx(ti, ntv);
          const float ya = (float)ty.add(__ldg(tp));
          const float yb = (float)ty.add(__ldg(tp + kLanes));
          const float2 sc = make_float2(s32, s32);
          const float2 fu = __fmul2_rn(make_float2(ER_U2F((unsigned)cu), ER_U2F((unsigned)bu)), sc);
          const float2 fv = __fmul2_rn(make_float2(ER_U2F((unsigned)cv), ER_U2F((unsigned)bv)), sc);
          const float2 fw = __fmul2_rn(make_float2(ER_U2F((unsigned)cw), ER_U2F((unsigned)bw)), sc);
          acc_voxel(lerp_quad(a0, a1, fu.x, fv.x, fw.x), ya, px, pxx, pyx);
          acc_voxel(lerp_quad(b0, b1, fu.y, fv.y, fw.y), yb, px, pxx, pyx);
          cu += du2;
          cv += dv2;
          cw += dw2;
          bu += du2;
          bv += dv2;
          bw += dw2;
        }
        k = ti - toff;
      }
      if (kPairBits) {
        // binary source, NB voxels per lane per step (k, k + kLanes, ...): NB
        // independent byte gathers in flight per lane, shared loop test and
        // target address; uniform cells add integer counts, boundary cells
        // interpolate in fp64 (bits_boundary).  Voxels are visited in the
        // single-voxel loop's order, so the results are bit-identical to it.
        constexpr int NB = kLanes >= 8 ? ER_BITS_NB_WIDE : ER_BITS_NB;
        int ti = toff + k;
        const int ti_end = toff + qhi - (NB - 1) * kLanes;
        const long long duN = NB * du1, dvN = NB * dv1, dwN = NB * dw1;
        const uint8_t* __restrict__ bytes = reinterpret_cast<const uint8_t*>(oct);
        // cell-index stepping (cell_step): voxel 0's fraction words + cell
        // index step by NB voxels, voxels 1..NB-1 are chained from it by one
        // voxel each; the samples only need the fraction words (bits_boundary's
        // 32-bit fractions, the nearest mode's bit 31)
        unsigned qu0 = (unsigned)cu, qv0 = (unsigned)cv, qw0 = (unsigned)cw;
        int cell0 = (F::ipart(cu) * og.cy + F::ipart(cv)) * og.cz + F::ipart(cw);
        const unsigned l1u = (unsigned)du1, l1v = (unsigned)dv1, l1w = (unsigned)dw1;
        const unsigned lNu = (unsigned)duN, lNv = (unsigned)dvN, lNw = (unsigned)dwN;
        const int h1 = F::ipart(du1) * cyz + F::ipart(dv1) * og.cz + F::ipart(dw1);
        const int hN = F::ipart(duN) * cyz + F::ipart(dvN) * og.cz + F::ipart(dwN);
        const int ti0 = ti;
        for (; ti < ti_end; ti += NB * kLanes) {
          unsigned cc[NB], wu[NB], wv[NB], ww[NB];
          TT yy[NB];
          const TT* tp = tgt + (unsigned)er_idx(ti, ntv);
          int cm = cell0;
          wu[0] = qu0;
          wv[0] = qv0;
          ww[0] = qw0;
#pragma unroll
          for (int m = 0; m < NB; ++m) {
            if (m > 0)
              cm = cell_step(wu[m - 1], wv[m - 1], ww[m - 1], cm, l1u, l1v, l1w, h1, cyz, og.cz,
                             wu[m], wv[m], ww[m]);
            cc[m] = __ldg(bytes + (unsigned)er_idx(cm, ncells));
            yy[m] = __ldg(tp + m * kLanes);
          }
#pragma unroll
          for (int m = 0; m < NB; ++m) {
            const auto yf = ty.add(yy[m]);
            if (LERP == ER_LERP_NEAREST) {
              // corner bit: fraction >= 0.5 <=> bit 31 of the fraction word
              const unsigned bsel = (wu[m] >> 31) | ((wv[m] >> 31) << 1) | ((ww[m] >> 31) << 2);
              if ((cc[m] >> bsel) & 1u) {
                ++ones;
                if (kU8Tgt) ones_y += (unsigned)yy[m];
                else pyx += (float)yf;
              }
            } else if (cc[m] == 0xFFu) {
              ++ones;
              if (kU8Tgt) ones_y += (unsigned)yy[m];
              else pyx += (float)yf;
            } else if (cc[m] != 0u) {
              bits_boundary(cc[m], (long long)wu[m], (long long)wv[m], (long long)ww[m],
                            (double)yf, racc[threadIdx.x]);
            }
          }
          cell0 = cell_step(qu0, qv0, qw0, cell0, lNu, lNv, lNw, hN, cyz, og.cz, qu0, qv0, qw0);
        }
        k = ti - toff;
        {
          // the 64-bit coordinates for the single-voxel tail
          const long long np = (ti - ti0) / (NB * kLanes);
          cu += np * duN;
          cv += np * dvN;
          cw += np * dwN;
        }
      }
      if (kPair) {
        // two voxels per lane per step (k and k + kLanes): the fractions, the
        // whole lerp chain and the accumulation run as fp32x2 pairs across the
        // two voxels; the loop control, the target row address and the
        // target sum are shared
        float2 sx2 = make_float2(0.f, 0.f), sxx2 = sx2, syx2 = sx2;
        const float s32 = 2.3283064365386963e-10f;  // 2^-32
        const float2 sc = make_float2(s32, s32);
        // loop on the target index (toff + k): one induction variable for the
        // loop test and the target address
        int ti = toff + k;
        const int ti_end = toff + qhi - kLanes;
        // cell-index stepping: the fixed-point coordinates live as their
        // 32-bit fraction words plus ONE padded cell index per voxel; a step
        // adds the fraction words (the carries are the integer parts'
        // +1s) and moves the cell index by the steps' integer parts times
        // the strides (h1 / h2) plus the strides of the carried axes.  Voxel
        // b = voxel a + kLanes is derived from a every step.
        unsigned au = (unsigned)cu, av = (unsigned)cv, aw = (unsigned)cw;
        int cella = (F::ipart(cu) * og.cy + F::ipart(cv)) * og.cz + F::ipart(cw);
        const unsigned l1u = (unsigned)du1, l1v = (unsigned)dv1, l1w = (unsigned)dw1;
        const unsigned l2u = (unsigned)du2, l2v = (unsigned)dv2, l2w = (unsigned)dw2;
        const int h1 = F::ipart(du1) * cyz + F::ipart(dv1) * og.cz + F::ipart(dw1);
        const int h2 = F::ipart(du2) * cyz + F::ipart(dv2) * og.cz + F::ipart(dw2);
        const int ti0 = ti;
        for (; ti < ti_end; ti += 2 * kLanes) {
          unsigned bu, bv, bw;
          const int cellb = cell_step(au, av, aw, cella, l1u, l1v, l1w, h1, cyz, og.cz, bu, bv, bw);
          const uint2 a8 = ld_oct(oct + (unsigned)er_idx(cella, ncells));
          const uint2 b8 = ld_oct(oct + (unsigned)er_idx(cellb, ncells));
          const TT* tp = tgt + (unsigned)er_idx(ti, ntv);
          const TT ya = __ldg(tp);
          const TT yb = __ldg(tp + kLanes);
          const float2 y2 = tgt_add2(ty, ya, yb);
          const float2 fu = __fmul2_rn(make_float2(ER_U2F(au), ER_U2F(bu)), sc);
          const float2 fv = __fmul2_rn(make_float2(ER_U2F(av), ER_U2F(bv)), sc);
          const float2 fw = __fmul2_rn(make_float2(ER_U2F(aw), ER_U2F(bw)), sc);
          const float2 x = lerp_oct_f32x2(a8, b8, fu, fv, fw);
          sx2 = __fadd2_rn(sx2, x);
          sxx2 = __ffma2_rn(x, x, sxx2);
          syx2 = __ffma2_rn(x, y2, syx2);
          cella = cell_step(au, av, aw, cella, l2u, l2v, l2w, h2, cyz, og.cz, au, av, aw);
        }
        {
          // the 64-bit coordinates for the single-voxel tail
          const long long np = (ti - ti0) / (2 * kLanes);
          cu += np * du2;
          cv += np * dv2;
          cw += np * dw2;
        }
        k = ti - toff;
        px = sx2.x + sx2.y;
        pxx = sxx2.x + sxx2.y;
        pyx = syx2.x + syx2.y;
      }
      ER_UNROLL(ER_OCT_UNROLL)
      for (; k < qhi; k += kLanes) {
        // 32-bit cell index: the padded grid has < 2^31 cells
        const int cell = F::ipart(cu) * cyz + F::ipart(cv) * og.cz + F::ipart(cw);
        const TT* tp = tgt + (unsigned)er_idx(toff + k, ntv);
        if (kQuad) {
          // f32/f64-stored source: entries cell (plane k0) and cell + 1
          // (plane k1), each (x[i0][j0], x[i0][j1], x[i1][j0], x[i1][j1])
          const float4* q = reinterpret_cast<const float4*>(oct) +
                            (unsigned)er_idx(cell, ncells - 1);
          const float4 q0 = __ldg(q), q1 = __ldg(q + 1);
          const auto yv = ty.add(__ldg(tp));
          const float2 fuv = __fmul2_rn(make_float2(ER_U2F((unsigned)cu), ER_U2F((unsigned)cv)),
                                        make_float2(2.3283064365386963e-10f,
                                                    2.3283064365386963e-10f));
          const float fw = F::frac32(cw);
          acc_voxel(lerp_quad(q0, q1, fuv.x, fuv.y, fw), (float)yv, px, pxx, pyx);
          cu += du1;
          cv += dv1;
          cw += dw1;
          continue;
        }
        if (kBits) {
          // binary source: one byte = the cell's 8 corner bits
          const unsigned c = __ldg(reinterpret_cast<const uint8_t*>(oct) +
                                   (unsigned)er_idx(cell, ncells));
          const TT yv = __ldg(tp);
          const auto yf = ty.add(yv);
#if ER_BITS_EXACT
          // uniform cells (all 0 / all 1) sample exactly 0 / 1: their terms are
          // integer counts; the rare boundary cells interpolate in fp64 with
          // the exact 32-bit fractions of the fixed-point coordinates
          bool one = c == 0xFFu;
          if (LERP == ER_LERP_NEAREST) {
            // corner bit: u -> bit 0, v -> bit 1, w -> bit 2 (bit b = byte b of
            // the oct word); fraction >= 0.5 <=> bit 31 of the fixed-point word
            const unsigned b = ((unsigned)cu >> 31) | (((unsigned)cv >> 31) << 1) |
                               (((unsigned)cw >> 31) << 2);
            one = (c >> b) & 1u;
          } else if (c != 0u && !one) {
            const double fu = F::frac64(cu), fv = F::frac64(cv), fw = F::frac64(cw);
            // u-lerp of two 0/1 corners: 0, fu, 1 - fu (exact for a 32-bit
            // fraction) or 1 -- the values fma(fu, b1 - b0, b0) takes, by selects
            const double gu = 1.0 - fu;
            auto pair = [c, fu, gu](int b) {
              const unsigned lo = (c >> b) & 1u, hi = (c >> (b + 1)) & 1u;
              return lo ? (hi ? 1.0 : gu) : (hi ? fu : 0.0);
            };
            const double c00 = pair(0), c10 = pair(2), c01 = pair(4), c11 = pair(6);
            const double c0 = fma(fv, c10 - c00, c00);
            const double c1 = fma(fv, c11 - c01, c01);
            const double x = fma(fw, c1 - c0, c0);
            double3 a = racc[threadIdx.x];
            a.x += x;
            a.y = fma(x, x, a.y);
            a.z = fma((double)yf, x, a.z);
            racc[threadIdx.x] = a;
          }
          if (one) {
            ++ones;
            if (kU8Tgt) ones_y += (unsigned)yv;
            else pyx += (float)yf;
          }
#else
          float x = (c == 0xFFu) ? 1.0f : 0.0f;
          if (LERP == ER_LERP_NEAREST) {
            const unsigned b = ((unsigned)cu >> 31) | (((unsigned)cv >> 31) << 1) |
                               (((unsigned)cw >> 31) << 2);
            x = (float)((c >> b) & 1u);
          } else if (c != 0u && c != 0xFFu) {
            const float fu = F::frac32(cu), fv = F::frac32(cv), fw = F::frac32(cw);
            auto bit = [c](int b) { return ((c >> b) & 1u) ? 1.0f : 0.0f; };
            const float2 P0 = make_float2(bit(0), bit(4)), P1 = make_float2(bit(1), bit(5));
            const float2 Q0 = make_float2(bit(2), bit(6)), Q1 = make_float2(bit(3), bit(7));
            const float2 fu2 = make_float2(fu, fu), fv2 = make_float2(fv, fv);
            const float2 cP = __ffma2_rn(fu2, f2sub(P1, P0), P0);
            const float2 cQ = __ffma2_rn(fu2, f2sub(Q1, Q0), Q0);
            const float2 cc = __ffma2_rn(fv2, f2sub(cQ, cP), cP);
            x = fmaf(fw, cc.y - cc.x, cc.x);
          }
          acc_voxel(x, (float)yf, px, pxx, pyx);
#endif
          cu += du1;
          cv += dv1;
          cw += dw1;
          continue;
        }
        const uint2 c8 = ld_oct(oct + (unsigned)er_idx(cell, ncells));
        const auto yv = ty.add(__ldg(tp));
        if (LERP == ER_LERP_NEAREST) {
          // nearest corner byte: u -> byte bit 0, v -> byte bit 1, w -> word
          const unsigned sel = ((unsigned)cu >> 31) | (((unsigned)cv >> 31) << 1);
          const unsigned wd = ((unsigned)cw >> 31) ? c8.y : c8.x;
          const float x = (float)__byte_perm(wd, 0u, 0x4440u | sel);
          acc_voxel(x, (float)yv, px, pxx, pyx);
        } else if (LERP == ER_LERP_F32) {
#if ER_OCT_FMUL2
          const float2 fuv = __fmul2_rn(make_float2(ER_U2F((unsigned)cu),
                                                    ER_U2F((unsigned)cv)),
                                        make_float2(2.3283064365386963e-10f,
                                                    2.3283064365386963e-10f));
          const float fu = fuv.x, fv = fuv.y, fw = F::frac32(cw);
#else
          const float fu = F::frac32(cu), fv = F::frac32(cv), fw = F::frac32(cw);
#endif
          acc_voxel(lerp_oct_f32(c8, fu, fv, fw), (float)yv, px, pxx, pyx);
        } else {
          const double fu = F::frac64(cu), fv = F::frac64(cv), fw = F::frac64(cw);
          // 2^52 + byte doubles: their differences are the exact byte
          // differences, so only the four base corners need the offset removed
          const double m000 = byte_m64(c8.x, 0), m100 = byte_m64(c8.x, 1);
          const double m010 = byte_m64(c8.x, 2), m110 = byte_m64(c8.x, 3);
          const double m001 = byte_m64(c8.y, 0), m101 = byte_m64(c8.y, 1);
          const double m011 = byte_m64(c8.y, 2), m111 = byte_m64(c8.y, 3);
          const double c00 = fma(fu, m100 - m000, m000 - 4503599627370496.0);
          const double c10 = fma(fu, m110 - m010, m010 - 4503599627370496.0);
          const double c01 = fma(fu, m101 - m001, m001 - 4503599627370496.0);
          const double c11 = fma(fu, m111 - m011, m011 - 4503599627370496.0);
          const double c0 = fma(fv, c10 - c00, c00);
          const double c1 = fma(fv, c11 - c01, c01);
          const double x = fma(fw, c1 - c0, c0);
          qx += x;
          qxx = fma(x, x, qxx);
          qyx = fma((double)yv, x, qyx);
        }
        cu += du1;
        cv += dv1;
        cw += dw1;
      }
      if (kF32 || kBits) {  // fp32 row partials (<= nz/kLanes voxels) -> fp64
        if (kSmemAcc) {
          double3 a = racc[threadIdx.x];
          a.x += (double)px;
          a.y += (double)pxx;
          a.z += (double)pyx;
          racc[threadIdx.x] = a;
        } else {
          qx += (double)px;
          qxx += (double)pxx;
          qyx += (double)pyx;
        }
        px = pxx = pyx = 0.f;
        if (kTgtRowFold) {
          double2 t = tacc[threadIdx.x];
          ty.fold(t.x, t.y);
          tacc[threadIdx.x] = t;
        }
      }
    }
    if (kSmemAcc) {
      const double3 a = racc[threadIdx.x];
      qx = a.x;
      qxx = a.y;
      qyx = a.z;
    }
    if (kBits && ER_BITS_EXACT) {  // exact integer terms of the uniform-1 voxels
      qx += (double)ones;
      qxx += (double)ones;
      qyx += (double)ones_y;
    }
    if (kQ52Path && q52) {  // lerp_q52's 2^40 sample scale, removed exactly
      qx *= 9.094947017729282e-13;
      qxx *= 8.271806125530277e-25;
      qyx *= 9.094947017729282e-13;
    }
    // fold the group: fixed-order warp reduction in fp64 into the group slot
    double v[5];
    v[0] = qx;
    v[1] = qxx;
    v[2] = qyx;
    v[3] = 0.0;
    v[4] = 0.0;
    if (kTgtRowFold) {
      const double2 t = tacc[threadIdx.x];
      v[3] = t.x;
      v[4] = t.y;
    } else {
      ty.fold(v[3], v[4]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int c = 0; c < 5; ++c) v[c] += __shfl_down_sync(0xffffffffu, v[c], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < 5; ++c) gsum[er_idx(grp, kRowsPerTile / 32)][c] = v[c];
      grp = atomicAdd(&next_group, 1);
    }
    grp = __shfl_sync(0xffffffffu, grp, 0);
  }
  // group-ordered sum (deterministic), integer overlap count
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
  __shared__ int cnt_w[kOctWarps];
  if (lane == 0) cnt_w[warp] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    Partial out{0.0, 0.0, 0.0, 0.0, 0.0, 0};
    for (int q = 0; q < ngroups; ++q) {
      out.x += gsum[q][0];
      out.xx += gsum[q][1];
      out.yx += gsum[q][2];
      out.y += gsum[q][3];
      out.yy += gsum[q][4];
    }
    for (int w = 0; w < kOctWarps; ++w) out.n += cnt_w[w];
    part[slot] = out;
  }
}

// Bit-oct re-layout of a binary source (one thread per padded cell).
__global__ void build_bitoct_kernel(const uint8_t* __restrict__ s, int sx, int sy, int sz,
                                    uint8_t* __restrict__ out) {
  const int cx = sx + 1, cy = sy + 1, cz = sz + 1;
  const long long n = (long long)cx * cy * cz;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int ck = (int)(q % cz);
    const long long rest = q / cz;
    const int cj = (int)(rest % cy);
    const int ci = (int)(rest / cy);
    const int i0 = min(max(ci - 1, 0), sx - 1), i1 = min(ci, sx - 1);
    const int j0 = min(max(cj - 1, 0), sy - 1), j1 = min(cj, sy - 1);
    const int k0 = min(max(ck - 1, 0), sz - 1), k1 = min(ck, sz - 1);
    auto at = [&](int i, int j, int k) -> unsigned {
      return s[((long long)i * sy + j) * sz + k] ? 1u : 0u;
    };
    out[q] = (uint8_t)(at(i0, j0, k0) | (at(i1, j0, k0) << 1) | (at(i0, j1, k0) << 2) |
                       (at(i1, j1, k0) << 3) | (at(i0, j0, k1) << 4) | (at(i1, j0, k1) << 5) |
                       (at(i0, j1, k1) << 6) | (at(i1, j1, k1) << 7));
  }
}

// Quad re-layout of an f32/f64 source (one thread per column entry; see
// er_build_quad in the header): entry (ci, cj, m) = the four (i, j) corners of
// plane clamp(m - 1), values rounded to fp32.
template <typename ST>
__global__ void build_quad_kernel(const ST* __restrict__ s, int sx, int sy, int sz,
                                  float4* __restrict__ out) {
  const int cy = sy + 1, cz = sz + 2;
  const long long n = (long long)(sx + 1) * cy * cz;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(q % cz);
    const long long rest = q / cz;
    const int cj = (int)(rest % cy);
    const int ci = (int)(rest / cy);
    const int i0 = min(max(ci - 1, 0), sx - 1), i1 = min(ci, sx - 1);
    const int j0 = min(max(cj - 1, 0), sy - 1), j1 = min(cj, sy - 1);
    const int k = min(max(m - 1, 0), sz - 1);
    auto at = [&](int i, int j) -> float { return (float)s[((long long)i * sy + j) * sz + k]; };
    out[q] = make_float4(at(i0, j0), at(i0, j1), at(i1, j0), at(i1, j1));
  }
}

// Oct re-layout of an 8-bit source (one thread per padded cell).
__global__ void build_oct_kernel(const uint8_t* __restrict__ s, int sx, int sy, int sz,
                                 uint2* __restrict__ oct) {
  const int cx = sx + 1, cy = sy + 1, cz = sz + 1;
  const long long n = (long long)cx * cy * cz;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int ck = (int)(q % cz);
    const long long rest = q / cz;
    const int cj = (int)(rest % cy);
    const int ci = (int)(rest / cy);
    const int i0 = min(max(ci - 1, 0), sx - 1), i1 = min(ci, sx - 1);
    const int j0 = min(max(cj - 1, 0), sy - 1), j1 = min(cj, sy - 1);
    const int k0 = min(max(ck - 1, 0), sz - 1), k1 = min(ck, sz - 1);
    auto at = [&](int i, int j, int k) -> unsigned {
      return s[((long long)i * sy + j) * sz + k];
    };
    uint2 w;
    w.x = at(i0, j0, k0) | (at(i1, j0, k0) << 8) | (at(i0, j1, k0) << 16) | (at(i1, j1, k0) << 24);
    w.y = at(i0, j0, k1) | (at(i1, j0, k1) << 8) | (at(i0, j1, k1) << 16) | (at(i1, j1, k1) << 24);
    oct[q] = w;
  }
}


struct Affines {
  double as, gs, at, gt;
};

// Per-particle finalize: kernels_numba.py:172-189 on the affine-corrected sums.
//
// Refinement (refine_list != NULL; the fp32-lerp paths): a particle whose
// likelihood the fp32 samples cannot resolve to the north star's 1e-4 is
// appended to refine_list, to be re-measured in reference-order fp64
// (measure_refine_kernel) and finalized again (list mode, below).  The
// fp32 samples carry errors of a few ulps of the STORED magnitudes (8-bit
// data: bytes ~100 with the z-score's offset folded into gamma), so the
// condition number uses the stored-magnitude scale as^2 XX in place of the
// value-space sum of squares:
//   kappa = as^2 XX / sss  +  at^2 YY / sst [fp32 target terms only]
//           + 2 sqrt(as^2 XX * s_tt) / |sts|
// (the condition number of z = sts^2 / (sst sss) under relative sample
// perturbations, tools/fuzz_measure.py conditioning()).  Measured errors stay
// below 0.7 eps kappa (100,000-case fuzz), so 4 eps32 kappa > 1e-4 (a 6x
// margin) lists the particle, and so does any particle whose variance test
// (< 1e-12, kernels_numba.py:183) is within 4 eps kappa of its threshold.
struct RefineArgs {
  int* list;         // NULL: no refinement
  int* count;
  int tgt_fp32;      // the target terms were accumulated in fp32
};

__device__ __forceinline__ void finalize_one(const Partial* __restrict__ q, int ntiles,
                                             const double* __restrict__ tmom, double nvox,
                                             int overlap, const Affines& f, long long p,
                                             double* __restrict__ ncc,
                                             uint8_t* __restrict__ degen,
                                             int64_t* __restrict__ n_in, RefineArgs r) {
  double X = 0.0, XX = 0.0, YX = 0.0, Y = 0.0, YY = 0.0;
  long long n = 0;
  for (int t = 0; t < ntiles; ++t) {
    X += q[t].x;
    XX += q[t].xx;
    YX += q[t].yx;
    Y += q[t].y;
    YY += q[t].yy;
    n += q[t].n;
  }
  if (n_in) n_in[p] = n;
  const double ni = (double)n;
  // value-space sums over in-bounds voxels (out-of-bounds source = fill 0)
  const double s_s = f.as * X + f.gs * ni;
  const double s_ss = f.as * f.as * XX + 2.0 * f.as * f.gs * X + f.gs * f.gs * ni;
  const double s_ts = f.at * f.as * YX + f.at * f.gs * Y + f.gt * f.as * X + f.gt * f.gs * ni;
  double s_t, s_tt, nf;
  if (overlap) {
    s_t = f.at * Y + f.gt * ni;
    s_tt = f.at * f.at * YY + 2.0 * f.at * f.gt * Y + f.gt * f.gt * ni;
    nf = ni;
  } else {
    s_t = f.at * tmom[0] + f.gt * nvox;
    s_tt = f.at * f.at * tmom[1] + 2.0 * f.at * f.gt * tmom[0] + f.gt * f.gt * nvox;
    nf = nvox;
  }
  if (nf == 0.0) {
    ncc[p] = 0.0;
    degen[p] = 1;
    return;
  }
  const double sst = rn_sub(s_tt, rn_div(rn_mul(s_t, s_t), nf));
  const double sss = rn_sub(s_ss, rn_div(rn_mul(s_s, s_s), nf));
  const double sts = rn_sub(s_ts, rn_div(rn_mul(s_t, s_s), nf));
  if (r.list != nullptr && n > 0) {
    const double e4 = 4.0 * 5.9604644775390625e-08;  // 4 eps32
    const double xs = f.as * f.as * XX;                // stored-magnitude scale
    const double yt = r.tgt_fp32 && overlap ? f.at * f.at * YY : 0.0;
    const double ks = xs / fabs(sss);
    const double kt = yt / fabs(sst);
    const double kts = 2.0 * sqrt(xs * fmax(s_tt, 0.0)) / fabs(sts);
    const double thr = 1e-12 * nf;
    // the variance tests must not be decided by fp32 noise either
    const bool near_s = fabs(sss - thr) <= e4 * xs;
    const bool near_t = yt > 0.0 && fabs(sst - thr) <= e4 * yt;
    const bool degenerate_sure = (sss < thr && !near_s) || (sst < thr && !near_t);
    if (near_s || near_t || (!degenerate_sure && !(e4 * (ks + kt + kts) <= 1e-4))) {
      r.list[atomicAdd(r.count, 1)] = (int)p;
    }
  }
  if (rn_div(sst, nf) < 1e-12 || rn_div(sss, nf) < 1e-12) {
    ncc[p] = 0.0;
    degen[p] = 1;
  } else {
    ncc[p] = rn_div(rn_mul(sts, sts), rn_mul(sst, sss));
    degen[p] = 0;
  }
}

__global__ void measure_finalize_kernel(const Partial* __restrict__ part, int ntiles,
                                        long long P, const double* __restrict__ tmom,
                                        double nvox, int overlap, Affines f,
                                        double* __restrict__ ncc, uint8_t* __restrict__ degen,
                                        int64_t* __restrict__ n_in, RefineArgs r) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= P) return;
  finalize_one(part + p * ntiles, ntiles, tmom, nvox, overlap, f, p, ncc, degen, n_in, r);
}

// finalize of the refined particles (list mode, persistent grid)
__global__ void measure_finalize_list_kernel(const Partial* __restrict__ part, int ntiles,
                                             const double* __restrict__ tmom, double nvox,
                                             int overlap, Affines f, double* __restrict__ ncc,
                                             uint8_t* __restrict__ degen,
                                             int64_t* __restrict__ n_in,
                                             const int* __restrict__ list,
                                             const int* __restrict__ count) {
  const int c = *count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
    const long long p = list[i];
    finalize_one(part + p * ntiles, ntiles, tmom, nvox, overlap, f, p, ncc, degen, n_in,
                 RefineArgs{nullptr, nullptr, 0});
  }
}

Geom make_geom(const er_volume* t, const er_volume* s) {
  Geom g;
  g.nx = t->nx;
  g.ny = t->ny;
  g.nz = t->nz;
  g.sx = s->nx;
  g.sy = s->ny;
  g.sz = s->nz;
  // tile = whole target planes, at most kRowsPerTile rows; small volumes are
  // cut into >= ER_MIN_TILES tiles (>= 256 rows each) so that few-particle
  // launches still fill the GPU.  Depends on the dims only: a particle's
  // partial sums never depend on P or on the GPU count.
  const long long rows_all = (long long)g.nx * g.ny;
  long long rows_tile = rows_all / ER_MIN_TILES;
  if (rows_tile < 256) rows_tile = 256;
  if (rows_tile > kRowsPerTile) rows_tile = kRowsPerTile;
  int ppt = (int)(rows_tile / (g.ny > 0 ? g.ny : 1));
  if (ppt < 1) ppt = 1;
  if (ppt > g.nx) ppt = g.nx;
  g.planes_per_tile = ppt;
  g.ntiles = (g.nx + ppt - 1) / ppt;
  g.limx = (double)g.sx - 1.0;
  g.limy = (double)g.sy - 1.0;
  g.limz = (double)g.sz - 1.0;
  return g;
}

template <typename TT, typename ST, int LERP>
void launch_typed(const er_volume* t, const er_volume* s, const double* A, const double* B,
                  const Geom& g, Partial* part, long long P, cudaStream_t st) {
  const long long blocks = P * g.ntiles;
  measure_partials_kernel<TT, ST, LERP><<<(unsigned)blocks, kThreads, 0, st>>>(
      (const TT*)t->data_dev, (const ST*)s->data_dev, A, B, g, part);
}

template <typename TT, typename ST>
void launch_lerp(int lerp, const er_volume* t, const er_volume* s, const double* A,
                 const double* B, const Geom& g, Partial* part, long long P, cudaStream_t st) {
  // fp64-stored sources lerp in fp64 even in the fp32 mode: eight F2F
  // conversions per voxel cost more than the fp64 arithmetic (B200 fp64 is
  // half rate), and the result is more accurate
  if (lerp == ER_LERP_F32 && sizeof(ST) == 8) lerp = ER_LERP_F64;
  switch (lerp) {
    case ER_LERP_F32: launch_typed<TT, ST, ER_LERP_F32>(t, s, A, B, g, part, P, st); break;
    case ER_LERP_F64: launch_typed<TT, ST, ER_LERP_F64>(t, s, A, B, g, part, P, st); break;
    case ER_LERP_NEAREST: launch_typed<TT, ST, ER_LERP_NEAREST>(t, s, A, B, g, part, P, st); break;
    default: launch_typed<TT, ST, ER_LERP_EXACT>(t, s, A, B, g, part, P, st); break;
  }
}

template <typename TT>
void launch_src(int lerp, const er_volume* t, const er_volume* s, const double* A,
                const double* B, const Geom& g, Partial* part, long long P, cudaStream_t st) {
  switch (s->dtype) {
    case ER_U8: launch_lerp<TT, uint8_t>(lerp, t, s, A, B, g, part, P, st); break;
    case ER_F32: launch_lerp<TT, float>(lerp, t, s, A, B, g, part, P, st); break;
    default: launch_lerp<TT, double>(lerp, t, s, A, B, g, part, P, st); break;
  }
}

bool valid_volume(const er_volume* v) {
  if (!v || !v->data_dev) return false;
  if (v->dtype < ER_U8 || v->dtype > ER_F64) return false;
  if (v->nx < 1 || v->ny < 1 || v->nz < 1) return false;
  const long long n = (long long)v->nx * v->ny * v->nz;
  return n < (1LL << 31);
}

}  // namespace

// workspace: [P x ntiles partials][refine count (16 B)][refine list: P ints]
static size_t partials_bytes(const Geom& g, int64_t P) {
  return (size_t)P * (size_t)g.ntiles * sizeof(Partial);
}
static size_t workspace_need(const Geom& g, int64_t P) {
  return partials_bytes(g, P) + 16 + (size_t)P * sizeof(int);
}

extern "C" size_t er_measure_workspace_bytes(const er_volume* tgt, int64_t P) {
  if (!tgt || tgt->nx < 1 || tgt->ny < 1 || P < 0) return 0;
  Geom g = make_geom(tgt, tgt);
  return workspace_need(g, P);
}

extern "C" int er_measure_ncc(const er_volume* tgt, const er_volume* src,
                              const double* tgt_moments_dev, const double* A_dev,
                              const double* b_dev, int64_t P, int32_t overlap_only,
                              int32_t lerp_mode, double* ncc_dev, uint8_t* degen_dev,
                              int64_t* n_in_dev, void* workspace_dev, size_t workspace_bytes,
                              void* stream) {
  if (!valid_volume(tgt) || !valid_volume(src))
    return er_set_error(ER_EINVAL, "er_measure_ncc: invalid volume descriptor");
  if (P < 0) return er_set_error(ER_EINVAL, "er_measure_ncc: negative particle count");
  if (P == 0) return ER_OK;
  if (!A_dev || !b_dev || !ncc_dev || !degen_dev || !tgt_moments_dev)
    return er_set_error(ER_EINVAL, "er_measure_ncc: null pointer");
  if (lerp_mode < ER_LERP_F32 || lerp_mode > ER_LERP_NEAREST)
    return er_set_error(ER_EINVAL, "er_measure_ncc: bad lerp_mode");
  const Geom g = make_geom(tgt, src);
  const size_t need = workspace_need(g, P);
  if (!workspace_dev || workspace_bytes < need)
    return er_set_error(ER_EINVAL, "er_measure_ncc: workspace too small");
  if ((long long)P * g.ntiles >= (1LL << 31))
    return er_set_error(ER_EINVAL, "er_measure_ncc: too many particles for one launch");
  cudaStream_t st = as_stream(stream);
  Partial* part = (Partial*)workspace_dev;
  // (the oct kernels' per-tile group slots assume a tile of <= kRowsPerTile rows,
  // and their 32-bit cell indices a padded source grid of < 2^31 cells)
  const long long cells = (long long)(src->nx + 1) * (src->ny + 1) * (src->nz + 1);
  const bool fast = lerp_mode != ER_LERP_EXACT && tgt->ny <= kRowsPerTile &&
                    src->dtype == ER_U8 && cells < (1LL << 31);
  const bool use_bits =
      fast && (lerp_mode == ER_LERP_F32 || lerp_mode == ER_LERP_NEAREST) && src->bitoct_dev;
  const bool use_oct = fast && !use_bits && src->oct_dev;
  const long long qcells = (long long)(src->nx + 1) * (src->ny + 1) * (src->nz + 2);
  const bool use_quad = lerp_mode == ER_LERP_F32 && tgt->ny <= kRowsPerTile &&
                        (src->dtype == ER_F32 || src->dtype == ER_F64) && src->quad_dev &&
                        qcells < (1LL << 31);
  if (use_quad) {
    const OctGeom og{src->ny + 1, src->nz + 2, (long long)P};
    const unsigned blocks = (unsigned)(P * g.ntiles);
    const uint2* lay = (const uint2*)src->quad_dev;
#define ER_QUAD(TT)                                                                            \
  do {                                                                                         \
    if (overlap_only)                                                                          \
      measure_oct_kernel<TT, ER_LERP_F32, 2, 1><<<blocks, OctThreads<ER_LERP_F32>::n, 0, st>>>( \
          (const TT*)tgt->data_dev, lay, A_dev, b_dev, g, og, part);                           \
    else                                                                                       \
      measure_oct_kernel<TT, ER_LERP_F32, 2, 0><<<blocks, OctThreads<ER_LERP_F32>::n, 0, st>>>( \
          (const TT*)tgt->data_dev, lay, A_dev, b_dev, g, og, part);                           \
  } while (0)
    switch (tgt->dtype) {
      case ER_U8: ER_QUAD(uint8_t); break;
      case ER_F32: ER_QUAD(float); break;
      default: ER_QUAD(double); break;
    }
#undef ER_QUAD
  } else if (use_bits || use_oct) {
    const OctGeom og{src->ny + 1, src->nz + 1, (long long)P};
    const unsigned blocks = (unsigned)(P * g.ntiles);
    const uint2* lay = (const uint2*)(use_bits ? src->bitoct_dev : src->oct_dev);
#define ER_OCT(TT, L, B)                                                                   \
  do {                                                                                     \
    if (overlap_only)                                                                      \
      measure_oct_kernel<TT, L, B, 1><<<blocks, OctThreads<L>::n, 0, st>>>(                \
          (const TT*)tgt->data_dev, lay, A_dev, b_dev, g, og, part);                       \
    else                                                                                   \
      measure_oct_kernel<TT, L, B, 0><<<blocks, OctThreads<L>::n, 0, st>>>(                \
          (const TT*)tgt->data_dev, lay, A_dev, b_dev, g, og, part);                       \
  } while (0)
#define ER_OCT_BITS_WIDE(TT)                                                               \
  do {                                                                                     \
    if (overlap_only)                                                                      \
      measure_oct_kernel<TT, ER_LERP_F32, 1, 1, 8>                                         \
          <<<blocks, OctThreads<ER_LERP_F32>::n, 0, st>>>((const TT*)tgt->data_dev, lay,   \
                                                          A_dev, b_dev, g, og, part);      \
    else                                                                                   \
      measure_oct_kernel<TT, ER_LERP_F32, 1, 0, 8>                                         \
          <<<blocks, OctThreads<ER_LERP_F32>::n, 0, st>>>((const TT*)tgt->data_dev, lay,   \
                                                          A_dev, b_dev, g, og, part);      \
  } while (0)
#define ER_OCT_BITS(TT)                                                   \
  do {                                                                    \
    if (lerp_mode == ER_LERP_NEAREST) ER_OCT(TT, ER_LERP_NEAREST, 1);     \
    else if (wide_rows) ER_OCT_BITS_WIDE(TT);                             \
    else ER_OCT(TT, ER_LERP_F32, 1);                                      \
  } while (0)
    // long target rows: the mask path walks them with 8 lanes, 4 voxels each
    // per step (more gathers in flight per lane)
    const bool wide_rows = tgt->nz >= ER_BITS_WIDE_NZ;
#define ER_OCT_BIG(TT)                                                                     \
  do {                                                                                     \
    if (overlap_only)                                                                      \
      measure_oct_kernel<TT, ER_LERP_F32, 0, 1, 8>                                         \
          <<<blocks, OctThreads<ER_LERP_F32>::n, 0, st>>>((const TT*)tgt->data_dev, lay,   \
                                                          A_dev, b_dev, g, og, part);      \
    else                                                                                   \
      measure_oct_kernel<TT, ER_LERP_F32, 0, 0, 8>                                         \
          <<<blocks, OctThreads<ER_LERP_F32>::n, 0, st>>>((const TT*)tgt->data_dev, lay,   \
                                                          A_dev, b_dev, g, og, part);      \
  } while (0)
#define ER_OCT_BYTES(TT)                                                  \
  do {                                                                    \
    if (lerp_mode == ER_LERP_NEAREST) ER_OCT(TT, ER_LERP_NEAREST, 0);     \
    else if (lerp_mode == ER_LERP_F32 && big) ER_OCT_BIG(TT);             \
    else if (lerp_mode == ER_LERP_F32) ER_OCT(TT, ER_LERP_F32, 0);        \
    else ER_OCT(TT, ER_LERP_F64, 0);                                      \
  } while (0)
    const bool big = cells * 8 > ER_OCT_BIG_BYTES;
    if (use_bits) {
      switch (tgt->dtype) {
        case ER_U8: ER_OCT_BITS(uint8_t); break;
        case ER_F32: ER_OCT_BITS(float); break;
        default: ER_OCT_BITS(double); break;
      }
    } else {
      switch (tgt->dtype) {
        case ER_U8: ER_OCT_BYTES(uint8_t); break;
        case ER_F32: ER_OCT_BYTES(float); break;
        default: ER_OCT_BYTES(double); break;
      }
    }
#undef ER_OCT_BITS
#undef ER_OCT_BITS_WIDE
#undef ER_OCT_BYTES
#undef ER_OCT_BIG
#undef ER_OCT
  } else {
    switch (tgt->dtype) {
      case ER_U8: launch_src<uint8_t>(lerp_mode, tgt, src, A_dev, b_dev, g, part, P, st); break;
      case ER_F32: launch_src<float>(lerp_mode, tgt, src, A_dev, b_dev, g, part, P, st); break;
      default: launch_src<double>(lerp_mode, tgt, src, A_dev, b_dev, g, part, P, st); break;
    }
  }
  ER_CHECK_LAUNCH();
  Affines f{src->alpha, src->gamma, tgt->alpha, tgt->gamma};
  const double nvox = (double)tgt->nx * (double)tgt->ny * (double)tgt->nz;
  const int fb = 128;
  // fp32-lerp samples (oct byte path, or the generic kernel on u8/f32 storage)
  // are refined where they cannot resolve 1e-4 (measure_finalize_kernel);
  // the bit-oct path samples exactly, nearest is a different operator, and
  // f64-stored sources lerp in fp64 anyway
  const bool refine =
      ER_REFINE && lerp_mode == ER_LERP_F32 && !use_bits && (src->dtype != ER_F64 || use_quad);
  RefineArgs r{nullptr, nullptr, tgt->dtype != ER_U8};
  if (refine) {
    char* base = (char*)workspace_dev + partials_bytes(g, P);
    r.count = (int*)base;
    r.list = (int*)(base + 16);
    const cudaError_t e = cudaMemsetAsync(r.count, 0, sizeof(int), st);
    if (e != cudaSuccess) return er_set_cuda_error(e, "er_measure_ncc (refinement list)");
  }
  measure_finalize_kernel<<<(unsigned)((P + fb - 1) / fb), fb, 0, st>>>(
      part, g.ntiles, P, tgt_moments_dev, nvox, overlap_only ? 1 : 0, f, ncc_dev, degen_dev,
      n_in_dev, r);
  ER_CHECK_LAUNCH();
  if (refine) {
    long long grid = (long long)P * g.ntiles;
    if (grid > 3LL * ER_NUM_SMS_B200) grid = 3LL * ER_NUM_SMS_B200;
#define ER_REFINE_LAUNCH(TT, ST)                                                          \
  measure_refine_kernel<TT, ST><<<(unsigned)grid, kThreads, 0, st>>>(                     \
      (const TT*)tgt->data_dev, (const ST*)src->data_dev, A_dev, b_dev, g, part, r.list,  \
      r.count)
    if (src->dtype == ER_U8) {
      switch (tgt->dtype) {
        case ER_U8: ER_REFINE_LAUNCH(uint8_t, uint8_t); break;
        case ER_F32: ER_REFINE_LAUNCH(float, uint8_t); break;
        default: ER_REFINE_LAUNCH(double, uint8_t); break;
      }
    } else if (src->dtype == ER_F32) {
      switch (tgt->dtype) {
        case ER_U8: ER_REFINE_LAUNCH(uint8_t, float); break;
        case ER_F32: ER_REFINE_LAUNCH(float, float); break;
        default: ER_REFINE_LAUNCH(double, float); break;
      }
    } else {
      switch (tgt->dtype) {
        case ER_U8: ER_REFINE_LAUNCH(uint8_t, double); break;
        case ER_F32: ER_REFINE_LAUNCH(float, double); break;
        default: ER_REFINE_LAUNCH(double, double); break;
      }
    }
#undef ER_REFINE_LAUNCH
    ER_CHECK_LAUNCH();
    long long fgrid = (P + fb - 1) / fb;
    if (fgrid > 16) fgrid = 16;
    measure_finalize_list_kernel<<<(unsigned)fgrid, fb, 0, st>>>(
        part, g.ntiles, tgt_moments_dev, nvox, overlap_only ? 1 : 0, f, ncc_dev, degen_dev,
        n_in_dev, r.list, r.count);
    ER_CHECK_LAUNCH();
  }
  return ER_OK;
}

extern "C" size_t er_oct_bytes(const er_volume* v) {
  if (!v || v->nx < 1 || v->ny < 1 || v->nz < 1) return 0;
  return (size_t)(v->nx + 1) * (size_t)(v->ny + 1) * (size_t)(v->nz + 1) * sizeof(uint2);
}

extern "C" int er_build_oct(const er_volume* v, void* oct_dev, void* stream) {
  if (!valid_volume(v) || v->dtype != ER_U8 || !oct_dev)
    return er_set_error(ER_EINVAL, "er_build_oct: needs a u8 volume and an output buffer");
  const long long n = (long long)(v->nx + 1) * (v->ny + 1) * (v->nz + 1);
  long long blocks = (n + 255) / 256;
  if (blocks > ER_NUM_SMS_B200 * 16) blocks = ER_NUM_SMS_B200 * 16;
  build_oct_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
      (const uint8_t*)v->data_dev, v->nx, v->ny, v->nz, (uint2*)oct_dev);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" size_t er_quad_bytes(const er_volume* v) {
  if (!v || v->nx < 1 || v->ny < 1 || v->nz < 1) return 0;
  return (size_t)(v->nx + 1) * (size_t)(v->ny + 1) * (size_t)(v->nz + 2) * sizeof(float4);
}

extern "C" int er_build_quad(const er_volume* v, void* quad_dev, void* stream) {
  if (!valid_volume(v) || (v->dtype != ER_F32 && v->dtype != ER_F64) || !quad_dev)
    return er_set_error(ER_EINVAL, "er_build_quad: needs an f32/f64 volume and an output buffer");
  const long long n = (long long)(v->nx + 1) * (v->ny + 1) * (v->nz + 2);
  long long blocks = (n + 255) / 256;
  if (blocks > ER_NUM_SMS_B200 * 16) blocks = ER_NUM_SMS_B200 * 16;
  if (v->dtype == ER_F32)
    build_quad_kernel<float><<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
        (const float*)v->data_dev, v->nx, v->ny, v->nz, (float4*)quad_dev);
  else
    build_quad_kernel<double><<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
        (const double*)v->data_dev, v->nx, v->ny, v->nz, (float4*)quad_dev);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" size_t er_bitoct_bytes(const er_volume* v) {
  if (!v || v->nx < 1 || v->ny < 1 || v->nz < 1) return 0;
  return (size_t)(v->nx + 1) * (size_t)(v->ny + 1) * (size_t)(v->nz + 1);
}

extern "C" int er_build_bitoct(const er_volume* v, void* bitoct_dev, void* stream) {
  if (!valid_volume(v) || v->dtype != ER_U8 || !bitoct_dev)
    return er_set_error(ER_EINVAL, "er_build_bitoct: needs a binary u8 volume and an output buffer");
  const long long n = (long long)(v->nx + 1) * (v->ny + 1) * (v->nz + 1);
  long long blocks = (n + 255) / 256;
  if (blocks > ER_NUM_SMS_B200 * 16) blocks = ER_NUM_SMS_B200 * 16;
  build_bitoct_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
      (const uint8_t*)v->data_dev, v->nx, v->ny, v->nz, (uint8_t*)bitoct_dev);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

ER_DEFINE_FAULT_READER(er_faults_measure)
