/*
 * eq_math.h — the device arithmetic contract shared by the CUDA kernels and the
 * CPU oracle (oracle/eq_oracle.cpp).
 *
 * The reference evaluates its hot path with CPython `math.exp` / `math.log`
 * (pkg/src/eventq/neuro.py:150,169,208, pkg/src/eventq/network.py:527-528,
 * 575-577,599-607).  CUDA's libdevice exp/log and glibc's differ by up to a
 * few ulp, so a GPU result can never be bitwise-compared with a CPU result that
 * used a different libm.  These two functions (per precision) are written only
 * with IEEE-754 primitives that are correctly rounded on both sides (+, -, *,
 * /, fma, rint, exponent bit-splicing), so the same source compiled by gcc
 * (-ffp-contract=off) and nvcc (-fmad=false) yields bit-identical results.
 * Accuracy against libm is tested in tests/test_math.py (<= 2 ulp).
 *
 * Everything else in the oracle is written independently of csrc/.
 */
#pragma once
#include <stdint.h>
#include <string.h>
#include <math.h>

#if defined(__CUDACC__)
#define EQ_HD __host__ __device__ __forceinline__
#else
#define EQ_HD static inline
#endif

EQ_HD double eq_f64_from_bits(int64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(b);
#else
  double d; memcpy(&d, &b, sizeof d); return d;
#endif
}
EQ_HD int64_t eq_f64_bits(double d) {
#if defined(__CUDA_ARCH__)
  return __double_as_longlong(d);
#else
  int64_t b; memcpy(&b, &d, sizeof b); return b;
#endif
}
EQ_HD float eq_f32_from_bits(int32_t b) {
#if defined(__CUDA_ARCH__)
  return __int_as_float(b);
#else
  float f; memcpy(&f, &b, sizeof f); return f;
#endif
}
EQ_HD int32_t eq_f32_bits(float f) {
#if defined(__CUDA_ARCH__)
  return __float_as_int(f);
#else
  int32_t b; memcpy(&b, &f, sizeof b); return b;
#endif
}

/* 2^k for k in the normal range, built from bits. */
EQ_HD double eq_pow2_f64(int k) { return eq_f64_from_bits((int64_t)(k + 1023) << 52); }
EQ_HD float eq_pow2_f32(int k) { return eq_f32_from_bits((int32_t)(k + 127) << 23); }

/* ---------------------------------------------------------------- double */

EQ_HD double eq_exp(double x) {
  if (x != x) return x;
  if (x > 709.782712893384) return (double)INFINITY;
  if (x < -745.1332191019412) return 0.0;
  const double inv_ln2 = 1.4426950408889634;
  const double ln2_hi = 6.93147180369123816490e-01; /* 32 significant bits */
  const double ln2_lo = 1.90821492927058770002e-10;
  double k = rint(x * inv_ln2);
  double r = fma(-k, ln2_hi, x);
  r = fma(-k, ln2_lo, r);
  /* Taylor to r^13 on |r| <= ln2/2: truncation < 5e-18 relative */
  double p = 1.6059043836821613e-10;          /* 1/13! */
  p = fma(p, r, 2.08767569878681e-09);         /* 1/12! */
  p = fma(p, r, 2.505210838544172e-08);        /* 1/11! */
  p = fma(p, r, 2.755731922398589e-07);        /* 1/10! */
  p = fma(p, r, 2.7557319223985893e-06);       /* 1/9!  */
  p = fma(p, r, 2.48015873015873e-05);         /* 1/8!  */
  p = fma(p, r, 1.984126984126984e-04);        /* 1/7!  */
  p = fma(p, r, 1.3888888888888889e-03);       /* 1/6!  */
  p = fma(p, r, 8.333333333333333e-03);        /* 1/5!  */
  p = fma(p, r, 4.1666666666666664e-02);       /* 1/4!  */
  p = fma(p, r, 1.6666666666666666e-01);       /* 1/3!  */
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  int ki = (int)k;
  if (ki > 1023) return (p * eq_pow2_f64(ki - 1)) * 2.0;
  if (ki < -1022) return (p * eq_pow2_f64(ki + 1000)) * eq_pow2_f64(-1000);
  return p * eq_pow2_f64(ki);
}

EQ_HD double eq_log(double x) {
  if (x != x || x < 0.0) return (double)NAN;
  if (x == 0.0) return -(double)INFINITY;
  if (x == (double)INFINITY) return x;
  int64_t bits = eq_f64_bits(x);
  int e = (int)((bits >> 52) & 0x7ff);
  int adj = 0;
  if (e == 0) { /* subnormal: renormalise */
    x = x * 18014398509481984.0; /* 2^54 */
    bits = eq_f64_bits(x);
    e = (int)((bits >> 52) & 0x7ff);
    adj = -54;
  }
  int ex = e - 1023 + adj;
  double m = eq_f64_from_bits((bits & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  if (m > 1.4142135623730951) { m = m * 0.5; ex += 1; }
  double f = m - 1.0;
  double s = f / (2.0 + f);
  double z = s * s;
  /* log(m) = 2 atanh(s) = 2s + s*z*(2/3 + 2z/5 + ... + 2z^10/23) */
  double q = 0.08695652173913043;               /* 2/23 */
  q = fma(q, z, 0.09523809523809523);           /* 2/21 */
  q = fma(q, z, 0.10526315789473684);           /* 2/19 */
  q = fma(q, z, 0.11764705882352941);           /* 2/17 */
  q = fma(q, z, 0.13333333333333333);           /* 2/15 */
  q = fma(q, z, 0.15384615384615385);           /* 2/13 */
  q = fma(q, z, 0.18181818181818182);           /* 2/11 */
  q = fma(q, z, 0.2222222222222222);            /* 2/9  */
  q = fma(q, z, 0.2857142857142857);            /* 2/7  */
  q = fma(q, z, 0.4);                           /* 2/5  */
  q = fma(q, z, 0.6666666666666666);            /* 2/3  */
  double lm = fma(s * z, q, 2.0 * s);
  if (ex == 0) return lm;
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  double de = (double)ex;
  return de * ln2_hi + (fma(de, ln2_lo, lm));
}

/* ----------------------------------------------------------------- float */

EQ_HD float eq_expf(float x) {
  if (x != x) return x;
  if (x > 88.72283f) return (float)INFINITY;
  if (x < -103.972084f) return 0.0f;
  const float inv_ln2 = 1.44269502f;
  const float ln2_hi = 0.693145751953125f;      /* 16 significant bits */
  const float ln2_lo = 1.42860676533018e-06f;
  float k = rintf(x * inv_ln2);
  float r = fmaf(-k, ln2_hi, x);
  r = fmaf(-k, ln2_lo, r);
  float p = 1.98412698e-04f;                    /* 1/7! */
  p = fmaf(p, r, 1.38888889e-03f);              /* 1/6! */
  p = fmaf(p, r, 8.33333333e-03f);              /* 1/5! */
  p = fmaf(p, r, 4.16666667e-02f);              /* 1/4! */
  p = fmaf(p, r, 1.66666667e-01f);              /* 1/3! */
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  int ki = (int)k;
  if (ki > 127) return (p * eq_pow2_f32(ki - 1)) * 2.0f;
  if (ki < -126) return (p * eq_pow2_f32(ki + 100)) * eq_pow2_f32(-100);
  return p * eq_pow2_f32(ki);
}

EQ_HD float eq_logf(float x) {
  if (x != x || x < 0.0f) return (float)NAN;
  if (x == 0.0f) return -(float)INFINITY;
  if (x == (float)INFINITY) return x;
  int32_t bits = eq_f32_bits(x);
  int e = (bits >> 23) & 0xff;
  int adj = 0;
  if (e == 0) {
    x = x * 16777216.0f; /* 2^24 */
    bits = eq_f32_bits(x);
    e = (bits >> 23) & 0xff;
    adj = -24;
  }
  int ex = e - 127 + adj;
  float m = eq_f32_from_bits((bits & 0x007fffff) | 0x3f800000);
  if (m > 1.41421356f) { m = m * 0.5f; ex += 1; }
  float f = m - 1.0f;
  float s = f / (2.0f + f);
  float z = s * s;
  float q = 0.181818182f;                       /* 2/11 */
  q = fmaf(q, z, 0.222222222f);                 /* 2/9 */
  q = fmaf(q, z, 0.285714286f);                 /* 2/7 */
  q = fmaf(q, z, 0.4f);                         /* 2/5 */
  q = fmaf(q, z, 0.666666667f);                 /* 2/3 */
  float lm = fmaf(s * z, q, 2.0f * s);
  if (ex == 0) return lm;
  const float ln2_hi = 0.693145751953125f;
  const float ln2_lo = 1.42860676533018e-06f;
  float de = (float)ex;
  return de * ln2_hi + fmaf(de, ln2_lo, lm);
}

#ifdef __cplusplus
/* precision-generic spellings used by templated code */
EQ_HD double eq_exp_t(double x) { return eq_exp(x); }
EQ_HD float eq_exp_t(float x) { return eq_expf(x); }
EQ_HD double eq_log_t(double x) { return eq_log(x); }
EQ_HD float eq_log_t(float x) { return eq_logf(x); }
#endif
