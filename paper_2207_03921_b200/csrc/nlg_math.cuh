// nlg_math.cuh -- x^e for x > 0 (the fractional kernel's r2^(-1-s)).
//
// CUDA's pow() spends ~90 FP64-pipe instructions on special cases and a
// double-double logarithm.  The kernel only ever sees finite, normal,
// positive r2 and a fixed exponent |e| <= 2, where
//     x^e = exp(e * (k ln2 + ln m)),  x = m 2^k,  m in [sqrt(1/2), sqrt(2))
// with ln m = 2 atanh(z), z = (m-1)/(m+1), |z| <= 0.1716 (odd series to
// z^21) and exp by Cody-Waite reduction + degree-12 Taylor.  ~40 FP64 ops,
// relative error ~1e-15 (tests/test_fastpow.py bounds it at 2e-14 against
// libm pow over the whole r2 range the meshes produce), far inside the
// 1e-10 parity bar.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

namespace nlg {

__host__ __device__ __forceinline__ double bits2d(uint64_t b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double d;
  memcpy(&d, &b, 8);
  return d;
#endif
}
__host__ __device__ __forceinline__ uint64_t d2bits(double d) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t b;
  memcpy(&b, &d, 8);
  return b;
#endif
}

// reciprocal to ~1 ulp: hardware seed + two Newton steps
__host__ __device__ __forceinline__ double fast_rcp(double d) {
#ifdef __CUDA_ARCH__
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
#else
  return 1.0 / d;
#endif
}

// series coefficients: atanh (1/21 ... 1/3), exp (1/12! ... 1/2), ln2 hi/lo, 1/ln2.
// On the device they live in constant memory so every FMA takes its
// coefficient as a constant-bank operand (a 64-bit immediate would cost two
// register moves per FMA).
#define NLG_POW_COEFFS                                                                                           \
  {1.0 / 21.0, 1.0 / 19.0, 1.0 / 17.0, 1.0 / 15.0, 1.0 / 13.0, 1.0 / 11.0, 1.0 / 9.0, 1.0 / 7.0, 1.0 / 5.0,       \
   1.0 / 3.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0, 1.0 / 40320.0, 1.0 / 5040.0, \
   1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 0.5, 6.93147180369123816490e-01, 1.90821492927058770002e-10,  \
   1.44269504088896338700e+00}
#ifdef __CUDACC__
__constant__ double c_powk[24] = NLG_POW_COEFFS;
#endif

// coefficient i as a literal (folds to an immediate when i is a constant)
__host__ __device__ constexpr double powk_lit(int i) {
  constexpr double t[24] = NLG_POW_COEFFS;
  return t[i];
}

// CBANK: coefficients from constant memory (loops that are not unrolled, where
// 64-bit immediates are re-materialised per use) or as literals (fully
// unrolled loops, where the compiler keeps them in registers).
template <bool CBANK>
__host__ __device__ __forceinline__ double powk(int i) {
#ifdef __CUDA_ARCH__
  if (CBANK) return c_powk[i];
#endif
  return powk_lit(i);
}

template <bool CBANK = true>
__host__ __device__ __forceinline__ double fast_pow_pos(double x, double e) {
#define K(i) powk<CBANK>(i)
  const uint64_t b = d2bits(x);
  int k = (int)((b >> 52) & 0x7ff) - 1023;
  uint64_t mb = (b & 0x000fffffffffffffull) | 0x3ff0000000000000ull;  // m in [1, 2)
  if ((b & 0x000fffffffffffffull) > 0x6a09e667f3bcdull) {            // m > sqrt(2): halve
    mb = (b & 0x000fffffffffffffull) | 0x3fe0000000000000ull;
    ++k;
  }
  const double m = bits2d(mb);
  const double z = (m - 1.0) * fast_rcp(m + 1.0);
  const double z2 = z * z;
  // atanh series: 2z (1 + z2/3 + z2^2/5 + ... + z2^10/21)
  double s = K(0);
#pragma unroll
  for (int i = 1; i < 10; ++i) s = fma(s, z2, K(i));
  const double lnm = fma(2.0 * z, s * z2, 2.0 * z);
  const double kd = (double)k;
  // t = e * ln x; k*ln2_hi is exact for |k| < 2^11
  const double t = e * (fma(kd, K(21), fma(kd, K(22), lnm)));
  // exp(t) = 2^n exp(r), r = t - n ln2
  const double n = rint(t * K(23));
  const double r = fma(-n, K(22), fma(-n, K(21), t));
  double p = K(10);
#pragma unroll
  for (int i = 11; i < 21; ++i) p = fma(p, r, K(i));
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  return bits2d(d2bits(p) + ((uint64_t)(int64_t)n << 52));
#undef K
}

// Table-driven x^e (x > 0, finite, normal) for the clipped-pair inner loop:
// fewer FP64 ops than fast_pow_pos (about 24 against 40), same accuracy class.
//   ln x = k ln2 + ln c_j + ln(1 + u),  m = x / 2^k in [1, 2),
//          c_j = 1 + (j + 1/2)/128 (j = top 7 mantissa bits), u = (m - c_j)/c_j,
//          |u| < 2^-8, ln(1+u) to u^7
//   exp t = 2^(n >> 6) 2^((n & 63)/64) exp(r),  n = rint(64 t / ln 2),
//          |r| <= ln2/128, exp(r) - 1 to r^6
// Tables (PowTab): 1/c_j and ln c_j for 128 j, 2^(i/64) for 64 i, built by
// pow_tab_fill; the clipped kernel keeps them in shared memory.
struct PowTab {
  double rc[128], lc[128], e2[64];
};

inline void pow_tab_fill(PowTab* t) {
  for (int j = 0; j < 128; ++j) {
    const double c = 1.0 + (j + 0.5) / 128.0;  // exact
    t->rc[j] = 1.0 / c;
    t->lc[j] = std::log(c);
  }
  for (int i = 0; i < 64; ++i) t->e2[i] = std::exp2(i / 64.0);
}

__host__ __device__ __forceinline__ double pow_tab(double x, double e, const double* __restrict__ rc,
                                                   const double* __restrict__ lc, const double* __restrict__ e2) {
  const uint64_t b = d2bits(x);
  const int k = (int)((b >> 52) & 0x7ff) - 1023;
  const int j = (int)((b >> 45) & 127);
  const double m = bits2d((b & 0x000fffffffffffffull) | 0x3ff0000000000000ull);
  const double c = 1.0 + (j + 0.5) * (1.0 / 128.0);
  const double u = (m - c) * rc[j];
  // ln(1+u) = u (1 - u/2 + u^2/3 - ... - u^6/7... ) : P(u) of degree 6
  double s = 1.0 / 7.0;
  s = fma(s, u, -1.0 / 6.0);
  s = fma(s, u, 1.0 / 5.0);
  s = fma(s, u, -1.0 / 4.0);
  s = fma(s, u, 1.0 / 3.0);
  s = fma(s, u, -0.5);
  s = fma(s, u, 1.0);
  const double l1 = u * s;
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double kd = (double)k;
  const double t = e * fma(kd, ln2_hi, lc[j] + fma(kd, ln2_lo, l1));
  const double n = rint(t * (64.0 / 6.93147180559945309417e-01));
  const double r = fma(-n, ln2_lo / 64.0, fma(-n, ln2_hi / 64.0, t));
  double p = 1.0 / 720.0;
  p = fma(p, r, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = p * r;  // exp(r) - 1
  const long long ni = (long long)n;
  const double tj = e2[ni & 63];
  const double v = fma(tj, p, tj);
  return bits2d(d2bits(v) + ((uint64_t)(ni >> 6) << 52));
}

}  // namespace nlg
