// numpy's float64 exp on AVX512_SKX hosts, restated bit-exactly.
//
// The reference's phantom speckle is np.exp(sigma * z) (phantom.py:76-77).
// numpy 2.3 dispatches contiguous float64 exp on AVX512_SKX CPUs to the
// bundled Intel SVML routine __svml_exp8_ha (DOUBLE_exp_AVX512_SKX in
// _multiarray_umath), which is NOT correctly rounded (differs from the
// correctly rounded result in ~4.6% of N(0, 0.3^2) arguments), so CUDA's
// exp() cannot reproduce it.  The routine's main path, restated below with
// the same constants (from __svml_dexp_ha_data_internal_avx512) and the same
// rounding of every step:
//   t  = fma_rz(x, 1/ln2, S)  S = 1.5*2^48 (+bias bits): ulp(t) = 1/16,
//                             so k = t - S = floor(16 x / ln2) / 16
//   j  = low 4 bits of t     (k = N + j/16)
//   r  = (x - k*ln2_hi) - k*ln2_lo           (two fused steps)
//   p  = degree-6 minimax polynomial of r    (Estrin-like, fused)
//   e  = T[j] * (1 + (p*r + Tc[j])),  result = e * 2^floor(k)  (vscalefpd)
// |x| >= 707.7 (overflow/underflow/NaN) takes SVML's scalar callout; those
// arguments fall back to exp() here and are outside the phantom's range.
// Verified bit-exact against np.exp on 5.1M arguments on an AVX512 host
// (tests/golden/npexp.npz, tests/test_phantom_device.py).  Hosts whose numpy
// takes the AVX2 path compute a different (also not correctly rounded) exp;
// the reference's phantom is therefore CPU-dependent at the 1-ulp level and
// the goldens pin the AVX512 variant.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifndef ER_HD
#define ER_HD __host__ __device__ __forceinline__
#endif

namespace npexp {

ER_HD double bits(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}
ER_HD uint64_t ubits(double d) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}

#ifdef __CUDA_ARCH__
#define NPX_FMA(a, b, c) __fma_rn((a), (b), (c))
#define NPX_FMA_RZ(a, b, c) __fma_rz((a), (b), (c))
#define NPX_MUL(a, b) __dmul_rn((a), (b))
#define NPX_SUB(a, b) __dsub_rn((a), (b))
#else
// host builds (tests/native): the caller provides fma_rz (fesetround around fma)
double host_fma_rz(double a, double b, double c);
#define NPX_FMA(a, b, c) fma((a), (b), (c))
#define NPX_FMA_RZ(a, b, c) host_fma_rz((a), (b), (c))
#define NPX_MUL(a, b) ((a) * (b))
#define NPX_SUB(a, b) ((a) - (b))
#endif

ER_HD double table_hi(int j) {  // 2^(j/16)
  switch (j) {
    case 0: return bits(0x3ff0000000000000ULL);
    case 1: return bits(0x3ff0b5586cf9890fULL);
    case 2: return bits(0x3ff172b83c7d517bULL);
    case 3: return bits(0x3ff2387a6e756238ULL);
    case 4: return bits(0x3ff306fe0a31b715ULL);
    case 5: return bits(0x3ff3dea64c123422ULL);
    case 6: return bits(0x3ff4bfdad5362a27ULL);
    case 7: return bits(0x3ff5ab07dd485429ULL);
    case 8: return bits(0x3ff6a09e667f3bcdULL);
    case 9: return bits(0x3ff7a11473eb0187ULL);
    case 10: return bits(0x3ff8ace5422aa0dbULL);
    case 11: return bits(0x3ff9c49182a3f090ULL);
    case 12: return bits(0x3ffae89f995ad3adULL);
    case 13: return bits(0x3ffc199bdd85529cULL);
    case 14: return bits(0x3ffd5818dcfba487ULL);
    default: return bits(0x3ffea4afa2a490daULL);
  }
}
ER_HD double table_corr(int j) {  // (2^(j/16) - table_hi(j)) / table_hi(j)
  switch (j) {
    case 0: return bits(0x0000000000000000ULL);
    case 1: return bits(0x3c979aa65d837b6dULL);
    case 2: return bits(0xbc801b15eaa59348ULL);
    case 3: return bits(0x3c968efde3a8a894ULL);
    case 4: return bits(0x3c834d754db0abb6ULL);
    case 5: return bits(0x3c859f48a72a4c6dULL);
    case 6: return bits(0x3c7690cebb7aafb0ULL);
    case 7: return bits(0x3c9063e1e21c5409ULL);
    case 8: return bits(0xbc93b3efbf5e2228ULL);
    case 9: return bits(0xbc7b32dcb94da51dULL);
    case 10: return bits(0x3c8db72fc1f0eab4ULL);
    case 11: return bits(0x3c71affc2b91ce27ULL);
    case 12: return bits(0x3c8c1a7792cb3387ULL);
    case 13: return bits(0x3c736eae30af0cb3ULL);
    case 14: return bits(0x3c74a385a63d07a7ULL);
    default: return bits(0xbc8ff7128fd391f0ULL);
  }
}

ER_HD double exp_svml_ha(double x) {
  const double shifter = bits(0x42f8000000003ff0ULL);
  if (!(fabs(x) < bits(0x40861da04cbafe44ULL))) return exp(x);  // SVML's scalar callout range
  const double t = NPX_FMA_RZ(x, bits(0x3ff71547652b82feULL), shifter);
  const double k = NPX_SUB(t, shifter);
  const int j = (int)(ubits(t) & 15u);
  double r = NPX_FMA(-k, bits(0x3fe62e42fefa39efULL), x);
  r = NPX_FMA(-bits(0x3c7abc9e3b39803fULL), k, r);
  r = bits(ubits(r) & 0xbfffffffffffffffULL);
  const double r2 = NPX_MUL(r, r);
  const double p1 = NPX_FMA(bits(0x3f57411836940c04ULL), r, bits(0x3f81101cbbc265c0ULL));
  const double p2 = NPX_FMA(bits(0x3fa55557242d68feULL), r, bits(0x3fc5555553939732ULL));
  const double p3 = NPX_FMA(bits(0x3fe000000000d008ULL), r, bits(0x3fefffffffffff70ULL));
  double q = NPX_FMA(r2, p1, p2);
  q = NPX_FMA(r2, q, p3);
  const double s = NPX_FMA(q, r, table_corr(j));
  const double th = table_hi(j);
  const double e = NPX_FMA(th, s, th);
  return ldexp(e, (int)floor(k));  // vscalefpd: exact for normal results
}

}  // namespace npexp
