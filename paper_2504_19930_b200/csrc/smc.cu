// SMC particle machinery on device (reference: echoreg/smc.py:145-259,
// geometry.py:76-152, exhaustive.py:25-113).  Everything between two
// measurements runs here, so an SMC iteration never round-trips to the host.
#include <cstdlib>

#include "common.cuh"
#include "rng.cuh"

namespace {

constexpr int kUpdThreads = 1024;

// to_matrix (geometry.py:87-99) + index_affine (geometry.py:136-152),
// naive left-to-right fp64 without contraction.  The reference's 3x3
// products go through BLAS, which may round one ulp differently; ±1-ulp
// matrix perturbations are parity-safe.
struct AffineGeom {
  double c[3];
  double st[3], ot[3];  // target (reference grid) spacing / origin
  double ss[3], os[3];  // source spacing / origin
};

__device__ void state_to_affine(const double* s, const AffineGeom& g, double* A, double* B) {
  double sxr, cxr, syr, cyr, szr, czr;
  sincos(s[0], &sxr, &cxr);
  sincos(s[1], &syr, &cyr);
  sincos(s[2], &szr, &czr);
  // rotation_xyz: Rz @ Ry @ Rx (geometry.py:76-84)
  const double m00 = rn_mul(czr, cyr), m01 = -szr, m02 = rn_mul(czr, syr);
  const double m10 = rn_mul(szr, cyr), m11 = czr, m12 = rn_mul(szr, syr);
  const double m20 = -syr, m21 = 0.0, m22 = cyr;
  double R[3][3];
  R[0][0] = m00;
  R[0][1] = rn_add(rn_mul(m01, cxr), rn_mul(m02, sxr));
  R[0][2] = rn_add(rn_mul(m01, -sxr), rn_mul(m02, cxr));
  R[1][0] = m10;
  R[1][1] = rn_add(rn_mul(m11, cxr), rn_mul(m12, sxr));
  R[1][2] = rn_add(rn_mul(m11, -sxr), rn_mul(m12, cxr));
  R[2][0] = m20;
  R[2][1] = rn_add(rn_mul(m21, cxr), rn_mul(m22, sxr));
  R[2][2] = rn_add(rn_mul(m21, -sxr), rn_mul(m22, cxr));
  // t_m = R @ (t - c) + c
  const double d0 = rn_sub(s[3], g.c[0]), d1 = rn_sub(s[4], g.c[1]), d2 = rn_sub(s[5], g.c[2]);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const double tm =
        rn_add(rn_add(rn_add(rn_mul(R[r][0], d0), rn_mul(R[r][1], d1)), rn_mul(R[r][2], d2)), g.c[r]);
    // index_affine: A = (R * st[None, :]) / ss[:, None];  b = (R @ ot + t - os) / ss
#pragma unroll
    for (int q = 0; q < 3; ++q) A[3 * r + q] = rn_div(rn_mul(R[r][q], g.st[q]), g.ss[r]);
    const double rot =
        rn_add(rn_add(rn_mul(R[r][0], g.ot[0]), rn_mul(R[r][1], g.ot[1])), rn_mul(R[r][2], g.ot[2]));
    B[r] = rn_div(rn_sub(rn_add(rot, tm), g.os[r]), g.ss[r]);
  }
}

__global__ void states_to_affine_kernel(const double* __restrict__ states, long long first,
                                        long long count, AffineGeom g, double* __restrict__ A,
                                        double* __restrict__ B) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= count) return;
  double s[6];
#pragma unroll
  for (int d = 0; d < 6; ++d) s[d] = states[6 * (first + q) + d];
  state_to_affine(s, g, A + 9 * q, B + 3 * q);
}

struct GridAxes {
  int half[6];
  double step[6];
};

// exhaustive.py:51-75: node values arange(-m, m+1) * step, last axis fastest
__global__ void grid_to_affine_kernel(long long first, long long count, GridAxes ax,
                                      AffineGeom g, double* __restrict__ states,
                                      double* __restrict__ A, double* __restrict__ B) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= count) return;
  long long rest = first + q;
  double s[6];
#pragma unroll
  for (int a = 5; a >= 0; --a) {
    const long long size = 2LL * ax.half[a] + 1;
    const long long pos = rest % size;
    rest /= size;
    s[a] = rn_mul((double)(pos - ax.half[a]), ax.step[a]);
  }
  if (states) {
#pragma unroll
    for (int d = 0; d < 6; ++d) states[6 * q + d] = s[d];
  }
  state_to_affine(s, g, A + 9 * q, B + 3 * q);
}

// init_particles (smc.py:145-157): one stream for all N*6 values, C order.
__global__ void smc_init_kernel(double* __restrict__ states, long long n, uint64_t seed,
                                double lo0, double lo1, double lo2, double lo3, double lo4,
                                double lo5, double rg0, double rg1, double rg2, double rg3,
                                double rg4, double rg5) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const double lo[6] = {lo0, lo1, lo2, lo3, lo4, lo5};
  const double rg[6] = {rg0, rg1, rg2, rg3, rg4, rg5};
  const unsigned long long e0 = 6ULL * p;
  uint64_t key[2] = {seed, 0};
  uint64_t blk = ~0ULL, out[4];
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    const unsigned long long e = e0 + d;
    const uint64_t b = e >> 2;
    if (b != blk) {
      uint64_t ctr[4] = {b + 1, 0, 0, 0};
      er_philox4x64_10(ctr, key, out);
      blk = b;
    }
    states[e] = er_uniform_from(out[e & 3], lo[d], rg[d]);
  }
}

struct Six {
  double v[6];
};

// predict (smc.py:160-174)
// A / B (optional): the index affines of particles [first, first + count)
// computed from the freshly predicted state (fused er_states_to_affine)
__global__ void smc_predict_kernel(const double* __restrict__ in, double* __restrict__ out,
                                   long long n, uint64_t seed, long long k, Six sigma,
                                   Six clip, long long first, long long count, AffineGeom g,
                                   double* __restrict__ A, double* __restrict__ B) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  ErPhilox s;
  er_stream_init(&s, seed, 1, (uint64_t)k, (uint64_t)i);
  double st[6];
#pragma unroll 1
  for (int d = 0; d < 6; ++d) {
    const double z = er_standard_normal(&s);
    double x = rn_add(in[6 * i + d], rn_mul(sigma.v[d], z));
    x = fmax(x, -clip.v[d]);
    x = fmin(x, clip.v[d]);
    out[6 * i + d] = x;
    st[d] = x;
  }
  if (A && i >= first && i < first + count)
    state_to_affine(st, g, A + 9 * (i - first), B + 3 * (i - first));
}

// ---- single-CTA update: weights, ESS, systematic resampling, estimate ----

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// fixed-order block sum; result broadcast to all threads
__device__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < (kUpdThreads / 32) ? sh[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

// N independent fixed-order block sums in one pass (each value is reduced in
// exactly the order block_sum uses, so the results are bit-identical to N
// separate calls); sh must hold 33 * N doubles
template <int N>
__device__ void block_sum_n(double (&v)[N], double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < N; ++c) v[c] = warp_sum(v[c]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < N; ++c) sh[32 * c + warp] = v[c];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double t = lane < (kUpdThreads / 32) ? sh[32 * c + lane] : 0.0;
      t = warp_sum(t);
      if (lane == 0) sh[32 * N + c] = t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < N; ++c) v[c] = sh[32 * N + c];
}

// first-max argmax (np.argmax): larger value wins, ties -> lower index
__device__ __forceinline__ void better(double& bv, long long& bi, double v, long long i) {
  if (v > bv || (v == bv && i < bi)) {
    bv = v;
    bi = i;
  }
}

__device__ void block_argmax(double& bv, long long& bi, double* shv, long long* shi) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v = __shfl_down_sync(0xffffffffu, bv, o);
    const long long i = __shfl_down_sync(0xffffffffu, bi, o);
    better(bv, bi, v, i);
  }
  __syncthreads();
  if (lane == 0) {
    shv[warp] = bv;
    shi[warp] = bi;
  }
  __syncthreads();
  if (warp == 0) {
    bv = lane < (kUpdThreads / 32) ? shv[lane] : -INFINITY;
    bi = lane < (kUpdThreads / 32) ? shi[lane] : (1LL << 62);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v = __shfl_down_sync(0xffffffffu, bv, o);
      const long long i = __shfl_down_sync(0xffffffffu, bi, o);
      better(bv, bi, v, i);
    }
    if (lane == 0) {
      shv[32] = bv;
      shi[32] = bi;
    }
  }
  __syncthreads();
  bv = shv[32];
  bi = shi[32];
}

// exclusive block scan of per-thread totals (fixed order)
__device__ double block_exclusive_scan(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  __syncthreads();
  if (lane == 31) sh[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    double w = lane < (kUpdThreads / 32) ? sh[lane] : 0.0;
    double wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < (kUpdThreads / 32)) sh[lane] = wi - w;  // exclusive warp offsets
  }
  __syncthreads();
  return sh[warp] + (incl - v);
}

// Where the update reads particle i's likelihood and degenerate flag:
// contiguous arrays (one GPU, or the caller gathered them), or the rank blocks
// of ONE all-gather of packed per-rank buffers [z: shard f64 | flags: shard
// u8 | pad], block bytes apart (the single collective per iteration).
struct ZContig {
  const double* __restrict__ z;
  const uint8_t* __restrict__ degen;
  __device__ __forceinline__ double zv(long long i) const { return z[i]; }
  __device__ __forceinline__ double dg(long long i) const { return degen ? (double)degen[i] : 0.0; }
};
struct ZPacked {
  const unsigned char* __restrict__ base;
  long long shard, block;
  __device__ __forceinline__ double zv(long long i) const {
    const long long r = i / shard;
    return reinterpret_cast<const double*>(base + r * block)[i - r * shard];
  }
  __device__ __forceinline__ double dg(long long i) const {
    const long long r = i / shard;
    return (double)base[r * block + 8 * shard + (i - r * shard)];
  }
};

template <typename ZA>
__global__ void __launch_bounds__(kUpdThreads)
    smc_update_kernel(const ZA za,
                      double* __restrict__ w, const double* __restrict__ st_in,
                      double* __restrict__ st_out, double* __restrict__ z_out,
                      double* __restrict__ cw, long long n, double beta, double ess_frac,
                      uint64_t seed, long long k, int est_best, er_smc_ctl* __restrict__ ctl,
                      double* __restrict__ trace) {
  __shared__ double sh[33 * 7];
  __shared__ double shv[40];
  __shared__ long long shi[40];
  __shared__ int fire_sh;
  // the resampling CDF lives in shared memory when it fits (binary searches
  // then stay on-chip), else in the caller's scratch
  constexpr int kCdfShared = 4096;
  __shared__ double cw_sh[kCdfShared];
  double* cdf = n <= kCdfShared ? cw_sh : cw;
  const int tid = threadIdx.x;
  const long long chunk = (n + kUpdThreads - 1) / kUpdThreads;
  const long long lo = min(n, tid * chunk), hi = min(n, lo + chunk);

  // best tracking over this iteration's measurements (smc.py:203-206)
  double bv = -INFINITY;
  long long bi = 1LL << 62;
  double ndeg = 0.0;
  for (long long i = lo; i < hi; ++i) {
    better(bv, bi, za.zv(i), i);
    ndeg += za.dg(i);
  }
  block_argmax(bv, bi, shv, shi);
  if (tid == 0 && bv > ctl->best_measurement) {
    ctl->best_measurement = bv;
    ctl->has_best = 1;
    for (int d = 0; d < 6; ++d) ctl->best_state[d] = st_in[6 * bi + d];
  }

  // update_weights (smc.py:210-224); beta >= 0 so max(beta*z) = beta*max(z)
  const double m = rn_mul(beta, bv);
  double part = 0.0;
  for (long long i = lo; i < hi; ++i) {
    const double wi = rn_mul(w[i], exp(rn_sub(rn_mul(beta, za.zv(i)), m)));
    w[i] = wi;
    part += wi;
  }
  const double total = block_sum(part, sh);
  const bool reset = !isfinite(total) || total <= 0.0;
  double part2 = 0.0, psum = 0.0;
  for (long long i = lo; i < hi; ++i) {
    const double wi = reset ? rn_div(1.0, (double)n) : rn_div(w[i], total);
    w[i] = wi;
    part2 = fma(wi, wi, part2);
    psum += wi;
  }
  double r3[3] = {psum, part2, ndeg};
  block_sum_n(r3, sh);
  const double wsum = r3[0], w2 = r3[1];
  ndeg = r3[2];
  const double ess = rn_div(1.0, w2);  // smc.py:227-229
  if (tid == 0) {
    if (fabs(wsum - 1.0) > 1e-9) ctl->error = ER_EWEIGHTS;  // smc.py:139-142
    fire_sh = ess < rn_mul(ess_frac, (double)n);             // smc.py:353
  }
  __syncthreads();
  const bool fire = fire_sh != 0;

  if (fire) {
    // resample_systematic (smc.py:232-248): u0 ~ U[0, 1/n) from (seed, 2, k, 0)
    ErPhilox s;
    er_stream_init(&s, seed, 2, (uint64_t)k, 0);
    const double inv_n = rn_div(1.0, (double)n);
    const double u0 = er_uniform(&s, 0.0, inv_n);
    // cumsum: per-thread sequential chunk + block exclusive scan of chunk sums
    double run = 0.0;
    for (long long i = lo; i < hi; ++i) run += w[i];
    double acc = block_exclusive_scan(run, sh);
    for (long long i = lo; i < hi; ++i) {
      acc += w[i];
      cdf[i] = acc;
    }
    __syncthreads();
    __threadfence_block();
    for (long long i = lo; i < hi; ++i) {
      const double pos = rn_add(u0, rn_div((double)i, (double)n));
      // searchsorted(cw, pos, side='right'): first index with cw > pos
      long long a = 0, b = n;
      while (a < b) {
        const long long mid = (a + b) >> 1;
        if (cdf[mid] <= pos) a = mid + 1;
        else b = mid;
      }
      const long long idx = a < n - 1 ? a : n - 1;
#pragma unroll
      for (int d = 0; d < 6; ++d) st_out[6 * i + d] = st_in[6 * idx + d];
      z_out[i] = za.zv(idx);
    }
    __syncthreads();
    for (long long i = lo; i < hi; ++i) w[i] = inv_n;
  } else {
    for (long long i = lo; i < hi; ++i) {
#pragma unroll
      for (int d = 0; d < 6; ++d) st_out[6 * i + d] = st_in[6 * i + d];
      z_out[i] = za.zv(i);
    }
  }
  __syncthreads();

  // estimate (smc.py:251-259) and trace row (smc.py:358-364)
  double est[7];  // 6 weighted-mean components + sum of z (trace mean)
  for (int d = 0; d < 6; ++d) {
    double e = 0.0;
    for (long long i = lo; i < hi; ++i) e = fma(w[i], st_out[6 * i + d], e);
    est[d] = e;
  }
  double zs = 0.0, zmax = -INFINITY;
  long long zi = 0;
  for (long long i = lo; i < hi; ++i) {
    zs += z_out[i];
    better(zmax, zi, z_out[i], i);
  }
  est[6] = zs;
  block_sum_n(est, sh);
  const double zsum = est[6];
  block_argmax(zmax, zi, shv, shi);
  if (tid == 0) {
    const bool use_best = est_best && ctl->has_best;
    for (int d = 0; d < 6; ++d) trace[d] = use_best ? ctl->best_state[d] : est[d];
    trace[6] = rn_div(zsum, (double)n);
    trace[7] = zmax;
    trace[8] = ctl->best_measurement;
    trace[9] = ess;
    trace[10] = fire ? 1.0 : 0.0;
    trace[11] = ndeg;
  }
}

// ---------------------------------------------------------------------------
// The same update for large populations (n >= kMultiMin) spread over the whole
// GPU.  The single-CTA kernel above is bound by one SM's latency and
// bandwidth at 10^5 particles (7 ms at 262,144: the binary searches of the
// resampling walk a global CDF).  Here every phase keeps EXACTLY the
// single-CTA numerics -- the same 1024 contiguous per-thread chunks
// (chunk = ceil(n / 1024)), the same sequential per-chunk loops, the same
// fixed-order trees over the 1024 chunk partials (block_sum, block_sum_n,
// block_argmax, block_exclusive_scan run by one 1024-thread CTA on the
// partials) -- so the results are bit-identical; only the per-element work
// (weights, searchsorted, gathers) runs on all SMs.  No extra memory: the
// chunk partials live in z_out (phases before the resampling writes it) and
// in scratch (after the CDF is consumed), the scalars in the trace row
// (rewritten by the last phase).  Requires n >= kMultiMin (partial space).
// ---------------------------------------------------------------------------
constexpr long long kMultiMin = 16384;
constexpr int kChunkThreads = 128;  // chunk kernels: 8 CTAs x 128 = 1024 chunks
// trace-row slots used as scalar scratch until the final phase rewrites them
enum { kTrM = 0, kTrTotal = 1, kTrReset = 2, kTrEss = 9, kTrFire = 10, kTrNdeg = 11 };

__device__ __forceinline__ void chunk_range(long long n, long long& lo, long long& hi) {
  const long long c = (long long)blockIdx.x * kChunkThreads + threadIdx.x;
  const long long chunk = (n + kUpdThreads - 1) / kUpdThreads;
  lo = min(n, c * chunk);
  hi = min(n, lo + chunk);
}

// phase 1: per-chunk best (value, index) and degenerate count
template <typename ZA>
__global__ void __launch_bounds__(kChunkThreads) upd_best_chunks(const ZA za, long long n,
                                                                 double* __restrict__ part) {
  long long lo, hi;
  chunk_range(n, lo, hi);
  double bv = -INFINITY;
  long long bi = 1LL << 62;
  double ndeg = 0.0;
  for (long long i = lo; i < hi; ++i) {
    better(bv, bi, za.zv(i), i);
    ndeg += za.dg(i);
  }
  const int c = blockIdx.x * kChunkThreads + threadIdx.x;
  part[c] = bv;
  reinterpret_cast<long long*>(part)[kUpdThreads + c] = bi;
  part[2 * kUpdThreads + c] = ndeg;  // kept until phase 5
}

// phase 2 (one CTA): best tracking and the weight exponent offset
__global__ void __launch_bounds__(kUpdThreads)
    upd_best_reduce(const double* __restrict__ part, const double* __restrict__ st_in,
                    double beta, er_smc_ctl* __restrict__ ctl, double* __restrict__ trace) {
  __shared__ double shv[40];
  __shared__ long long shi[40];
  double bv = part[threadIdx.x];
  long long bi = reinterpret_cast<const long long*>(part)[kUpdThreads + threadIdx.x];
  block_argmax(bv, bi, shv, shi);
  if (threadIdx.x == 0) {
    if (bv > ctl->best_measurement) {
      ctl->best_measurement = bv;
      ctl->has_best = 1;
      for (int d = 0; d < 6; ++d) ctl->best_state[d] = st_in[6 * bi + d];
    }
    trace[kTrM] = rn_mul(beta, bv);
  }
}

// phase 3: w *= exp(beta z - m), per-chunk sums
template <typename ZA>
__global__ void __launch_bounds__(kChunkThreads)
    upd_weight_chunks(const ZA za, double* __restrict__ w, long long n, double beta,
                      const double* __restrict__ trace, double* __restrict__ part) {
  long long lo, hi;
  chunk_range(n, lo, hi);
  const double m = trace[kTrM];
  double s = 0.0;
  for (long long i = lo; i < hi; ++i) {
    const double wi = rn_mul(w[i], exp(rn_sub(rn_mul(beta, za.zv(i)), m)));
    w[i] = wi;
    s += wi;
  }
  part[3 * kUpdThreads + blockIdx.x * kChunkThreads + threadIdx.x] = s;
}

// phase 4 (one CTA): the weight total
__global__ void __launch_bounds__(kUpdThreads) upd_total_reduce(const double* __restrict__ part,
                                                                double* __restrict__ trace) {
  __shared__ double sh[33];
  const double total = block_sum(part[3 * kUpdThreads + threadIdx.x], sh);
  if (threadIdx.x == 0) {
    trace[kTrTotal] = total;
    trace[kTrReset] = (!isfinite(total) || total <= 0.0) ? 1.0 : 0.0;
  }
}

// phase 5: normalise, per-chunk (sum w, sum w^2)
__global__ void __launch_bounds__(kChunkThreads)
    upd_norm_chunks(double* __restrict__ w, long long n, const double* __restrict__ trace,
                    double* __restrict__ part) {
  long long lo, hi;
  chunk_range(n, lo, hi);
  const double total = trace[kTrTotal];
  const bool reset = trace[kTrReset] != 0.0;
  double part2 = 0.0, psum = 0.0;
  for (long long i = lo; i < hi; ++i) {
    const double wi = reset ? rn_div(1.0, (double)n) : rn_div(w[i], total);
    w[i] = wi;
    part2 = fma(wi, wi, part2);
    psum += wi;
  }
  const int c = blockIdx.x * kChunkThreads + threadIdx.x;
  part[4 * kUpdThreads + c] = psum;
  part[5 * kUpdThreads + c] = part2;
}

// phase 6 (one CTA): ESS and the resampling decision
__global__ void __launch_bounds__(kUpdThreads)
    upd_ess_reduce(const double* __restrict__ part, long long n, double ess_frac,
                   er_smc_ctl* __restrict__ ctl, double* __restrict__ trace) {
  __shared__ double sh[33 * 3];
  double r3[3] = {part[4 * kUpdThreads + threadIdx.x], part[5 * kUpdThreads + threadIdx.x],
                  part[2 * kUpdThreads + threadIdx.x]};
  block_sum_n(r3, sh);
  if (threadIdx.x == 0) {
    const double ess = rn_div(1.0, r3[1]);
    if (fabs(r3[0] - 1.0) > 1e-9) ctl->error = ER_EWEIGHTS;
    trace[kTrEss] = ess;
    trace[kTrFire] = ess < rn_mul(ess_frac, (double)n) ? 1.0 : 0.0;
    trace[kTrNdeg] = r3[2];
  }
}

// phase 7: per-chunk weight sums for the CDF (only when resampling)
__global__ void __launch_bounds__(kChunkThreads)
    upd_cdf_chunks(const double* __restrict__ w, long long n, const double* __restrict__ trace,
                   double* __restrict__ part) {
  if (trace[kTrFire] == 0.0) return;
  long long lo, hi;
  chunk_range(n, lo, hi);
  double run = 0.0;
  for (long long i = lo; i < hi; ++i) run += w[i];
  part[6 * kUpdThreads + blockIdx.x * kChunkThreads + threadIdx.x] = run;
}

// phase 8 (one CTA): exclusive scan of the chunk sums
__global__ void __launch_bounds__(kUpdThreads) upd_cdf_scan(double* __restrict__ part,
                                                            const double* __restrict__ trace) {
  __shared__ double sh[33];
  if (trace[kTrFire] == 0.0) return;
  const double off = block_exclusive_scan(part[6 * kUpdThreads + threadIdx.x], sh);
  part[7 * kUpdThreads + threadIdx.x] = off;
}

// phase 9: the CDF itself (sequential within each chunk, from its offset)
__global__ void __launch_bounds__(kChunkThreads)
    upd_cdf_fill(const double* __restrict__ w, long long n, const double* __restrict__ trace,
                 const double* __restrict__ part, double* __restrict__ cdf) {
  if (trace[kTrFire] == 0.0) return;
  long long lo, hi;
  chunk_range(n, lo, hi);
  double acc = part[7 * kUpdThreads + blockIdx.x * kChunkThreads + threadIdx.x];
  for (long long i = lo; i < hi; ++i) {
    acc += w[i];
    cdf[i] = acc;
  }
}

// phase 10 (one thread per particle): systematic resampling or plain copy
template <typename ZA>
__global__ void __launch_bounds__(256)
    upd_resample(const ZA za, double* __restrict__ w, const double* __restrict__ st_in,
                 double* __restrict__ st_out, double* __restrict__ z_out,
                 const double* __restrict__ cdf, long long n, uint64_t seed, long long k,
                 const double* __restrict__ trace) {
  const long long i = blockIdx.x * 256LL + threadIdx.x;
  if (i >= n) return;
  if (trace[kTrFire] != 0.0) {
    ErPhilox s;
    er_stream_init(&s, seed, 2, (uint64_t)k, 0);
    const double inv_n = rn_div(1.0, (double)n);
    const double u0 = er_uniform(&s, 0.0, inv_n);
    const double pos = rn_add(u0, rn_div((double)i, (double)n));
    long long a = 0, b = n;
    while (a < b) {
      const long long mid = (a + b) >> 1;
      if (cdf[mid] <= pos) a = mid + 1;
      else b = mid;
    }
    const long long idx = a < n - 1 ? a : n - 1;
#pragma unroll
    for (int d = 0; d < 6; ++d) st_out[6 * i + d] = st_in[6 * idx + d];
    z_out[i] = za.zv(idx);
  } else {
#pragma unroll
    for (int d = 0; d < 6; ++d) st_out[6 * i + d] = st_in[6 * i + d];
    z_out[i] = za.zv(i);
  }
}

// phase 11: uniform weights after resampling (all CDF reads are done)
__global__ void __launch_bounds__(256) upd_reset_weights(double* __restrict__ w, long long n,
                                                         const double* __restrict__ trace) {
  const long long i = blockIdx.x * 256LL + threadIdx.x;
  if (i < n && trace[kTrFire] != 0.0) w[i] = rn_div(1.0, (double)n);
}

// phase 12: per-chunk estimate partials (weighted state sums, z sum, z max)
__global__ void __launch_bounds__(kChunkThreads)
    upd_est_chunks(const double* __restrict__ w, const double* __restrict__ st_out,
                   const double* __restrict__ z_out, long long n, double* __restrict__ part) {
  long long lo, hi;
  chunk_range(n, lo, hi);
  const int c = blockIdx.x * kChunkThreads + threadIdx.x;
  for (int d = 0; d < 6; ++d) {
    double e = 0.0;
    for (long long i = lo; i < hi; ++i) e = fma(w[i], st_out[6 * i + d], e);
    part[d * kUpdThreads + c] = e;
  }
  double zs = 0.0, zmax = -INFINITY;
  long long zi = 0;
  for (long long i = lo; i < hi; ++i) {
    zs += z_out[i];
    better(zmax, zi, z_out[i], i);
  }
  part[6 * kUpdThreads + c] = zs;
  part[7 * kUpdThreads + c] = zmax;
  reinterpret_cast<long long*>(part)[8 * kUpdThreads + c] = zi;
}

// phase 13 (one CTA): the estimate and the trace row
__global__ void __launch_bounds__(kUpdThreads)
    upd_est_reduce(const double* __restrict__ part, long long n, int est_best,
                   const er_smc_ctl* __restrict__ ctl, double* __restrict__ trace) {
  __shared__ double sh[33 * 7];
  __shared__ double shv[40];
  __shared__ long long shi[40];
  const int t = threadIdx.x;
  double est[7];
#pragma unroll
  for (int d = 0; d < 7; ++d) est[d] = part[d * kUpdThreads + t];
  block_sum_n(est, sh);
  double zmax = part[7 * kUpdThreads + t];
  long long zi = reinterpret_cast<const long long*>(part)[8 * kUpdThreads + t];
  block_argmax(zmax, zi, shv, shi);
  if (t == 0) {
    const bool use_best = est_best && ctl->has_best;
    for (int d = 0; d < 6; ++d) trace[d] = use_best ? ctl->best_state[d] : est[d];
    trace[6] = rn_div(est[6], (double)n);
    trace[7] = zmax;
    trace[8] = ctl->best_measurement;
    // trace[9..11] (ess, fired, n_degenerate) were written by phase 6
  }
}

template <typename ZA>
void smc_update_multi(const ZA& za, double* w, const double* st_in, double* st_out,
                      double* z_out, double* scratch, long long n, double beta,
                      double ess_frac, uint64_t seed, long long k, int est_best,
                      er_smc_ctl* ctl, double* trace, cudaStream_t st) {
  const unsigned cb = kUpdThreads / kChunkThreads;
  const unsigned pb = (unsigned)((n + 255) / 256);
  double* pre = z_out;     // partials before the resampling writes z_out
  double* post = scratch;  // partials after the CDF has been consumed
  upd_best_chunks<ZA><<<cb, kChunkThreads, 0, st>>>(za, n, pre);
  upd_best_reduce<<<1, kUpdThreads, 0, st>>>(pre, st_in, beta, ctl, trace);
  upd_weight_chunks<ZA><<<cb, kChunkThreads, 0, st>>>(za, w, n, beta, trace, pre);
  upd_total_reduce<<<1, kUpdThreads, 0, st>>>(pre, trace);
  upd_norm_chunks<<<cb, kChunkThreads, 0, st>>>(w, n, trace, pre);
  upd_ess_reduce<<<1, kUpdThreads, 0, st>>>(pre, n, ess_frac, ctl, trace);
  upd_cdf_chunks<<<cb, kChunkThreads, 0, st>>>(w, n, trace, pre);
  upd_cdf_scan<<<1, kUpdThreads, 0, st>>>(pre, trace);
  upd_cdf_fill<<<cb, kChunkThreads, 0, st>>>(w, n, trace, pre, scratch);
  upd_resample<ZA><<<pb, 256, 0, st>>>(za, w, st_in, st_out, z_out, scratch, n, seed, k, trace);
  upd_reset_weights<<<pb, 256, 0, st>>>(w, n, trace);
  upd_est_chunks<<<cb, kChunkThreads, 0, st>>>(w, st_out, z_out, n, post);
  upd_est_reduce<<<1, kUpdThreads, 0, st>>>(post, n, est_best, ctl, trace);
}

// ER_SMC_UPDATE_SINGLE=1 in the environment forces the single-CTA kernel at
// every size (the bit-identity tests compare the two)
bool update_multi(long long n) {
  static const int single = [] {
    const char* e = getenv("ER_SMC_UPDATE_SINGLE");
    return e && e[0] == '1' ? 1 : 0;
  }();
  return n >= kMultiMin && !single;
}

__global__ void argmax_update_kernel(const double* __restrict__ z, long long n,
                                     long long base, double* __restrict__ best) {
  __shared__ double shv[40];
  __shared__ long long shi[40];
  double bv = -INFINITY;
  long long bi = 1LL << 62;
  for (long long i = threadIdx.x; i < n; i += kUpdThreads) better(bv, bi, z[i], i);
  block_argmax(bv, bi, shv, shi);
  if (threadIdx.x == 0 && bv > best[0]) {  // strict '>' across chunks (exhaustive.py:107)
    best[0] = bv;
    best[1] = (double)(base + bi);
  }
}

AffineGeom make_affine_geom(const double center[3], const double tsp[3], const double tor[3],
                            const double ssp[3], const double sor[3]) {
  AffineGeom g;
  for (int d = 0; d < 3; ++d) {
    g.c[d] = center[d];
    g.st[d] = tsp[d];
    g.ot[d] = tor[d];
    g.ss[d] = ssp[d];
    g.os[d] = sor[d];
  }
  return g;
}

}  // namespace

extern "C" int er_smc_init(double* states_dev, int64_t n, uint64_t seed, const double lim[6],
                           void* stream) {
  if (!states_dev || !lim || n < 0) return er_set_error(ER_EINVAL, "er_smc_init: args");
  if (n == 0) return ER_OK;
  // numpy uniform(low=-lim, high=lim): range = high - low (computed in fp64)
  double lo[6], rg[6];
  for (int d = 0; d < 6; ++d) {
    lo[d] = -lim[d];
    rg[d] = lim[d] - (-lim[d]);
  }
  smc_init_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
      states_dev, n, seed, lo[0], lo[1], lo[2], lo[3], lo[4], lo[5], rg[0], rg[1], rg[2],
      rg[3], rg[4], rg[5]);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_smc_predict(const double* states_in_dev, double* states_out_dev, int64_t n,
                              uint64_t seed, int64_t k, const double sigma[6],
                              const double clip[6], void* stream) {
  if (!states_in_dev || !states_out_dev || !sigma || !clip || n < 0)
    return er_set_error(ER_EINVAL, "er_smc_predict: args");
  if (n == 0) return ER_OK;
  Six sg, cl;
  for (int d = 0; d < 6; ++d) {
    sg.v[d] = sigma[d];
    cl.v[d] = clip[d];
  }
  smc_predict_kernel<<<(unsigned)((n + 127) / 128), 128, 0, as_stream(stream)>>>(
      states_in_dev, states_out_dev, n, seed, k, sg, cl, 0, 0, AffineGeom{}, nullptr, nullptr);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_smc_predict_affine(const double* states_in_dev, double* states_out_dev,
                                     int64_t n, uint64_t seed, int64_t k, const double sigma[6],
                                     const double clip[6], int64_t first, int64_t count,
                                     const double center[3], const double tgt_spacing[3],
                                     const double tgt_origin[3], const double src_spacing[3],
                                     const double src_origin[3], double* A_dev, double* b_dev,
                                     void* stream) {
  if (!states_in_dev || !states_out_dev || !sigma || !clip || n < 0 || first < 0 ||
      count < 0 || first + count > n || (count > 0 && (!A_dev || !b_dev)))
    return er_set_error(ER_EINVAL, "er_smc_predict_affine: args");
  if (n == 0) return ER_OK;
  Six sg, cl;
  for (int d = 0; d < 6; ++d) {
    sg.v[d] = sigma[d];
    cl.v[d] = clip[d];
  }
  if (count > 0 && (!center || !tgt_spacing || !tgt_origin || !src_spacing || !src_origin))
    return er_set_error(ER_EINVAL, "er_smc_predict_affine: geometry");
  const AffineGeom g = count > 0 ? make_affine_geom(center, tgt_spacing, tgt_origin,
                                                    src_spacing, src_origin)
                                 : AffineGeom{};
  smc_predict_kernel<<<(unsigned)((n + 127) / 128), 128, 0, as_stream(stream)>>>(
      states_in_dev, states_out_dev, n, seed, k, sg, cl, first, count, g,
      count > 0 ? A_dev : nullptr, b_dev);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_states_to_affine(const double* states_dev, int64_t first, int64_t count,
                                   const double center[3], const double tgt_spacing[3],
                                   const double tgt_origin[3], const double src_spacing[3],
                                   const double src_origin[3], double* A_dev, double* b_dev,
                                   void* stream) {
  if (!states_dev || !A_dev || !b_dev || count < 0 || first < 0)
    return er_set_error(ER_EINVAL, "er_states_to_affine: args");
  if (count == 0) return ER_OK;
  AffineGeom g = make_affine_geom(center, tgt_spacing, tgt_origin, src_spacing, src_origin);
  states_to_affine_kernel<<<(unsigned)((count + 127) / 128), 128, 0, as_stream(stream)>>>(
      states_dev, first, count, g, A_dev, b_dev);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_grid_to_affine(int64_t first, int64_t count, const int32_t half_counts[6],
                                 const double axis_step[6], const double center[3],
                                 const double tgt_spacing[3], const double tgt_origin[3],
                                 const double src_spacing[3], const double src_origin[3],
                                 double* states_dev, double* A_dev, double* b_dev,
                                 void* stream) {
  if (!A_dev || !b_dev || count < 0 || first < 0 || !half_counts || !axis_step)
    return er_set_error(ER_EINVAL, "er_grid_to_affine: args");
  if (count == 0) return ER_OK;
  GridAxes ax;
  for (int a = 0; a < 6; ++a) {
    if (half_counts[a] < 0) return er_set_error(ER_EINVAL, "er_grid_to_affine: half count");
    ax.half[a] = half_counts[a];
    ax.step[a] = axis_step[a];
  }
  AffineGeom g = make_affine_geom(center, tgt_spacing, tgt_origin, src_spacing, src_origin);
  grid_to_affine_kernel<<<(unsigned)((count + 127) / 128), 128, 0, as_stream(stream)>>>(
      first, count, ax, g, states_dev, A_dev, b_dev);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_argmax_update(const double* z_dev, int64_t n, int64_t base_index,
                                double* best_dev, void* stream) {
  if (!z_dev || !best_dev || n < 0) return er_set_error(ER_EINVAL, "er_argmax_update: args");
  if (n == 0) return ER_OK;
  argmax_update_kernel<<<1, kUpdThreads, 0, as_stream(stream)>>>(z_dev, n, base_index, best_dev);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_smc_update(const double* z_dev, const uint8_t* degen_dev, double* weights_dev,
                             const double* states_in_dev, double* states_out_dev,
                             double* z_out_dev, double* scratch_dev, int64_t n, double beta,
                             double ess_fraction, uint64_t seed, int64_t k,
                             int32_t estimate_best, er_smc_ctl* ctl_dev, double* trace_row_dev,
                             void* stream) {
  if (!z_dev || !weights_dev || !states_in_dev || !states_out_dev || !z_out_dev ||
      !scratch_dev || !ctl_dev || !trace_row_dev || n < 1)
    return er_set_error(ER_EINVAL, "er_smc_update: args");
  if (beta < 0) return er_set_error(ER_EINVAL, "er_smc_update: beta must be >= 0");
  if (update_multi(n)) {
    smc_update_multi(ZContig{z_dev, degen_dev}, weights_dev, states_in_dev, states_out_dev,
                     z_out_dev, scratch_dev, n, beta, ess_fraction, seed, k, estimate_best,
                     ctl_dev, trace_row_dev, as_stream(stream));
  } else {
    smc_update_kernel<ZContig><<<1, kUpdThreads, 0, as_stream(stream)>>>(
        ZContig{z_dev, degen_dev}, weights_dev, states_in_dev, states_out_dev, z_out_dev,
        scratch_dev, n, beta, ess_fraction, seed, k, estimate_best, ctl_dev, trace_row_dev);
  }
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_smc_update_gathered(const void* zd_dev, int64_t shard, int64_t block_bytes,
                                      double* weights_dev, const double* states_in_dev,
                                      double* states_out_dev, double* z_out_dev,
                                      double* scratch_dev, int64_t n, double beta,
                                      double ess_fraction, uint64_t seed, int64_t k,
                                      int32_t estimate_best, er_smc_ctl* ctl_dev,
                                      double* trace_row_dev, void* stream) {
  if (!zd_dev || !weights_dev || !states_in_dev || !states_out_dev || !z_out_dev ||
      !scratch_dev || !ctl_dev || !trace_row_dev || n < 1 || shard < 1 ||
      block_bytes < 9 * shard || block_bytes % 8 != 0)
    return er_set_error(ER_EINVAL, "er_smc_update_gathered: args");
  if (beta < 0) return er_set_error(ER_EINVAL, "er_smc_update_gathered: beta must be >= 0");
  const ZPacked za{(const unsigned char*)zd_dev, shard, block_bytes};
  if (update_multi(n)) {
    smc_update_multi(za, weights_dev, states_in_dev, states_out_dev, z_out_dev, scratch_dev, n,
                     beta, ess_fraction, seed, k, estimate_best, ctl_dev, trace_row_dev,
                     as_stream(stream));
  } else {
    smc_update_kernel<ZPacked><<<1, kUpdThreads, 0, as_stream(stream)>>>(
        za, weights_dev, states_in_dev, states_out_dev, z_out_dev, scratch_dev, n, beta,
        ess_fraction, seed, k, estimate_best, ctl_dev, trace_row_dev);
  }
  ER_CHECK_LAUNCH();
  return ER_OK;
}

ER_DEFINE_FAULT_READER(er_faults_smc)
