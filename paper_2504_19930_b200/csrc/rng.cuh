// Counter-based RNG that reproduces, bit for bit, the numpy streams the
// reference draws from:
//   _stream(seed, role, step, index) = Generator(Philox(key=seed,
//       counter=[0, role, step, index]))            (echoreg/smc.py:38-42)
// numpy's Philox4x64-10 pre-increments counter word 0 (with carry) before
// every 4-word block, so block b of that stream is
//   philox4x64_10(ctr = [b+1, role, step, index], key = [seed, 0]).
// Doubles are (u64 >> 11) * 2^-53; Gaussians use numpy's 256-layer ziggurat
// with numpy's own tables (gen_ziggurat.py).  The tail's log1p, whose result
// IS the returned value, is glibc's (er_log1p, restated from its FMA build);
// the wedge test's exp is CUDA's: a 1-ulp difference from glibc could only
// flip an accept test that lands within one ulp of its threshold.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "zig_tables.h"

#if defined(__CUDACC__)
#define ER_HD __host__ __device__ __forceinline__
#else
#define ER_HD inline
#endif

// Device copies of the tables.  The ziggurat indexes them with a random byte
// per lane, so __constant__ storage (broadcast cache) would serialise a warp's
// divergent lookups; ER_ZIG_GLOBAL = 1 keeps them in global memory read
// through the read-only L1 path instead.  (Each translation unit that
// includes this header gets its own copy.)
#ifndef ER_ZIG_GLOBAL
#define ER_ZIG_GLOBAL 1
#endif
#if defined(__CUDACC__)
#if ER_ZIG_GLOBAL
__device__ const uint64_t er_ki_double[256] = ER_KI_INIT;
__device__ const double er_wi_double[256] = ER_WI_INIT;
__device__ const double er_fi_double[256] = ER_FI_INIT;
#else
__constant__ uint64_t er_ki_double[256] = ER_KI_INIT;
__constant__ double er_wi_double[256] = ER_WI_INIT;
__constant__ double er_fi_double[256] = ER_FI_INIT;
#endif
#endif
static const uint64_t er_host_ki_double[256] = ER_KI_INIT;
static const double er_host_wi_double[256] = ER_WI_INIT;
static const double er_host_fi_double[256] = ER_FI_INIT;

#ifdef __CUDA_ARCH__
#if ER_ZIG_GLOBAL
#define ER_KI_AT(i) __ldg(&er_ki_double[(i)])
#define ER_WI_AT(i) __ldg(&er_wi_double[(i)])
#define ER_FI_AT(i) __ldg(&er_fi_double[(i)])
#else
#define ER_KI_AT(i) er_ki_double[(i)]
#define ER_WI_AT(i) er_wi_double[(i)]
#define ER_FI_AT(i) er_fi_double[(i)]
#endif
#else
#define ER_KI_AT(i) er_host_ki_double[(i)]
#define ER_WI_AT(i) er_host_wi_double[(i)]
#define ER_FI_AT(i) er_host_fi_double[(i)]
#endif

struct ErPhilox {
  uint64_t ctr[4];
  uint64_t key[2];
  uint64_t buf[4];
  int pos;
};

ER_HD void er_mulhilo64(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
#ifdef __CUDA_ARCH__
  *lo = a * b;
  *hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
#endif
}

// Philox4x64 with 10 rounds (Salmon et al., SC'11; the Random123 constants).
ER_HD void er_philox4x64_10(const uint64_t in[4], const uint64_t key_in[2], uint64_t out[4]) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
  uint64_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
  uint64_t k0 = key_in[0], k1 = key_in[1];
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    uint64_t hi0, lo0, hi1, lo1;
    er_mulhilo64(M0, c0, &hi0, &lo0);
    er_mulhilo64(M1, c2, &hi1, &lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0;
    uint64_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// Generator(Philox(key=seed, counter=[0, role, step, index])): fresh state,
// empty buffer (numpy sets buffer_pos = 4).
ER_HD void er_stream_init(ErPhilox* s, uint64_t seed, uint64_t role, uint64_t step, uint64_t index) {
  s->ctr[0] = 0;
  s->ctr[1] = role;
  s->ctr[2] = step;
  s->ctr[3] = index;
  s->key[0] = seed;
  s->key[1] = 0;
  s->pos = 4;
}

// Jump straight to block b (0-based) of a fresh stream: used when element e
// of a long draw sequence is wanted without generating 0..e-1.
ER_HD void er_stream_seek_block(ErPhilox* s, uint64_t block) {
  // the stream pre-increments: block b uses ctr[0] = b + 1 (carry into ctr[1..3])
  uint64_t c0 = s->ctr[0] + block;
  uint64_t carry = c0 < s->ctr[0];
  s->ctr[0] = c0;
  if (carry && ++s->ctr[1] == 0 && ++s->ctr[2] == 0) ++s->ctr[3];
  s->pos = 4;
}

ER_HD uint64_t er_next_u64(ErPhilox* s) {
  if (s->pos < 4) return s->buf[s->pos++];
  if (++s->ctr[0] == 0 && ++s->ctr[1] == 0 && ++s->ctr[2] == 0) ++s->ctr[3];
  er_philox4x64_10(s->ctr, s->key, s->buf);
  s->pos = 1;
  return s->buf[0];
}

ER_HD double er_u64_to_double(uint64_t r) {
  return (double)(r >> 11) * (1.0 / 9007199254740992.0);
}

ER_HD double er_next_double(ErPhilox* s) { return er_u64_to_double(er_next_u64(s)); }

#ifdef __CUDA_ARCH__
#define ER_MUL(a, b) __dmul_rn((a), (b))
#define ER_ADD(a, b) __dadd_rn((a), (b))
#define ER_SUB(a, b) __dsub_rn((a), (b))
#else
#define ER_MUL(a, b) ((a) * (b))
#define ER_ADD(a, b) ((a) + (b))
#define ER_SUB(a, b) ((a) - (b))
#endif

#ifdef __CUDA_ARCH__
#define ER_FMA(a, b, c) __fma_rn((a), (b), (c))
#define ER_DIV(a, b) __ddiv_rn((a), (b))
#else
#define ER_FMA(a, b, c) fma((a), (b), (c))
#define ER_DIV(a, b) ((a) / (b))
#endif

ER_HD double er_bits_d(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}
ER_HD uint64_t er_d_bits(double d) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}

// log1p as numpy's ziggurat tail gets it: npy_log1p -> glibc 2.39 log1p,
// whose x86_64 IFUNC picks the FMA build of sysdeps/ieee754/dbl-64/s_log1p.c
// (fdlibm) on FMA/AVX2 hosts.  Restated with that build's fused operations
// (read from its machine code) so tail draws match bit for bit; CUDA's
// log1p differs from it in the last bit on some arguments.
ER_HD double er_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const int32_t hx = (int32_t)(er_d_bits(x) >> 32);
  const int32_t ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {                      // x < 0.41422
    if (ax >= 0x3ff00000) {                   // x <= -1
      if (x == -1.0) return -er_bits_d(0x7ff0000000000000ULL);
      return er_bits_d(0x7ff8000000000000ULL);
    }
    if (ax < 0x3e200000) {                    // |x| < 2^-29
      if (ax < 0x3c900000) return x;
      return ER_FMA(-ER_MUL(x, x), 0.5, x);   // x - x*x*0.5 (fused)
    }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {  // -0.2929 < x < 0.41422
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return ER_ADD(x, x);
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = ER_ADD(1.0, x);
      hu = (int32_t)(er_d_bits(u) >> 32);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? ER_SUB(1.0, ER_SUB(u, x)) : ER_SUB(x, ER_SUB(u, 1.0));
      c = ER_DIV(c, u);
    } else {
      u = x;
      hu = (int32_t)(er_d_bits(u) >> 32);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    const uint64_t lo = er_d_bits(u) & 0xffffffffULL;
    if (hu < 0x6a09e) {
      u = er_bits_d(((uint64_t)(uint32_t)(hu | 0x3ff00000) << 32) | lo);
    } else {
      k += 1;
      u = er_bits_d(((uint64_t)(uint32_t)(hu | 0x3fe00000) << 32) | lo);
      hu = (0x00100000 - hu) >> 2;
    }
    f = ER_SUB(u, 1.0);
  }
  const double hfsq = ER_MUL(ER_MUL(f, 0.5), f);
  const double dk = (double)k;
  if (hu == 0) {                              // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      return ER_FMA(dk, ln2_hi, ER_FMA(dk, ln2_lo, c));
    }
    const double R = ER_MUL(ER_FMA(-f, 0.66666666666666666, 1.0), hfsq);
    if (k == 0) return ER_SUB(f, R);
    return ER_FMA(dk, ln2_hi, -ER_SUB(ER_SUB(R, ER_FMA(dk, ln2_lo, c)), f));
  }
  const double s = ER_DIV(f, ER_ADD(2.0, f));
  const double z = ER_MUL(s, s);
  const double R2 = ER_FMA(z, Lp3, Lp2), R3 = ER_FMA(z, Lp5, Lp4), R4 = ER_FMA(z, Lp7, Lp6);
  const double z2 = ER_MUL(z, z), z4 = ER_MUL(z2, z2), z6 = ER_MUL(z2, z4);
  double R = ER_FMA(z, Lp1, ER_MUL(z2, R2));
  R = ER_FMA(z4, R3, R);
  R = ER_FMA(z6, R4, R);
  const double t = ER_MUL(ER_ADD(R, hfsq), s);
  if (k == 0) return ER_SUB(f, ER_SUB(hfsq, t));
  const double cc = ER_ADD(ER_FMA(dk, ln2_lo, c), t);
  return ER_FMA(dk, ln2_hi, -ER_SUB(ER_SUB(hfsq, cc), f));
}

// Word sources for the ziggurat: the Philox stream itself, or a bounded
// array of pre-generated stream words starting at an arbitrary position (the
// device phantom evaluates "the normal that would start at word q" for every
// q in parallel, then keeps the ones on the actual consumption chain).
struct ErStreamWords {
  ErPhilox* s;
  ER_HD uint64_t next() { return er_next_u64(s); }
  ER_HD bool exhausted() const { return false; }
};
struct ErArrayWords {
  const uint64_t* w;
  long long pos, end;
  ER_HD uint64_t next() { return pos < end ? w[pos++] : (++pos, 0ULL); }
  ER_HD bool exhausted() const { return pos > end; }
};

// numpy random_standard_normal (ziggurat, 256 layers), numpy/random/src/
// distributions/distributions.c; r = [idx:8 | sign:1 | rabs:52 | ...].
// An exhausted array source returns 0.0 (the caller checks exhausted()).
template <class Words>
ER_HD double er_standard_normal_from(Words& s) {
  const double zr = 3.6541528853610087963519472518;      // ziggurat_nor_r
  const double zinv = 0.27366123732975827203338247596;   // ziggurat_nor_inv_r
  for (;;) {
    uint64_t r = s.next();
    if (s.exhausted()) return 0.0;
    int idx = (int)(r & 0xff);
    r >>= 8;
    int sign = (int)(r & 0x1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = ER_MUL((double)rabs, ER_WI_AT(idx));
    if (sign) x = -x;
    if (rabs < ER_KI_AT(idx)) return x;
    if (idx == 0) {
      for (;;) {
        double xx = ER_MUL(-zinv, er_log1p(-er_u64_to_double(s.next())));
        double yy = -er_log1p(-er_u64_to_double(s.next()));
        if (s.exhausted()) return 0.0;
        if (ER_ADD(yy, yy) > ER_MUL(xx, xx))
          return ((rabs >> 8) & 0x1) ? -ER_ADD(zr, xx) : ER_ADD(zr, xx);
      }
    } else {
      double f = ER_ADD(ER_MUL(ER_SUB(ER_FI_AT(idx - 1), ER_FI_AT(idx)),
                               er_u64_to_double(s.next())),
                        ER_FI_AT(idx));
      if (s.exhausted()) return 0.0;
      if (f < exp(ER_MUL(ER_MUL(-0.5, x), x))) return x;
    }
  }
}

ER_HD double er_standard_normal(ErPhilox* s) {
  ErStreamWords w{s};
  return er_standard_normal_from(w);
}

// element drawn from an already generated 64-bit word
ER_HD double er_uniform_from(uint64_t r, double lower, double range) {
  return ER_ADD(lower, ER_MUL(range, er_u64_to_double(r)));
}

// numpy random_uniform: lower + range * next_double (no FMA)
ER_HD double er_uniform(ErPhilox* s, double lower, double range) {
  return ER_ADD(lower, ER_MUL(range, er_next_double(s)));
}
