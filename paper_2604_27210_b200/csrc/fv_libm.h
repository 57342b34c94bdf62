// fv_libm.h -- bit-faithful restatement of the third-party scalar math the
// reference path executes, as __host__ __device__ C++.
//
// The reference (fastvol, pure Python) reaches native arithmetic only through
//   * CPython `math.exp/log/erfc/sqrt` and `float.__pow__` -> glibc 2.39 libm
//     (x86-64 multiarch: the FMA variants __exp_fma/__log_fma/__pow_fma are
//     selected by ifunc on any FMA-capable host; erfc is the plain fdlibm
//     s_erf.c build and calls the same ifunc'd exp), and
//   * `scipy.special.erfcx` (scipy 1.18.1, xsf = S. G. Johnson's Faddeeva
//     package) at fastvol/lbr.py:30,48-49.
// Results must match those bits exactly (~1.2% of
// quotes move sigma by >1e-12 under a 1-ulp perturbation), so each routine
// below restates the published algorithm with the exact operation DAG the
// glibc 2.39 x86-64 build executes: every `fma()` here is a fused op in the
// shipped binary (read from `objdump -d` of libm-2.39.a), every other op is a
// separately rounded IEEE op.  Compile with FMA contraction OFF
// (nvcc -fmad=false, gcc -ffp-contract=off); IEEE div/sqrt are the CUDA
// defaults for fp64.  Constants/tables: fv_tables.h (tools/gen_tables.py).
//
// Verified bit-for-bit against the live glibc / scipy on CPU by
// tests/test_libm_host.py (host build of this same header) and on the B200 by
// tests/test_gpu_parity.py.
#pragma once
#include <stdint.h>
#include <string.h>
#include <math.h>

#if defined(__CUDACC__)
#define FV_HD __host__ __device__ __forceinline__
#define FV_HDM __host__ __device__ __forceinline__
// Out-of-line on the device: the LBR kernel calls these from many sites and
// inlining all of them blows the instruction cache (ncu: stall_no_instruction).
#define FV_HDN __host__ __device__ __noinline__
#else
#define FV_HD static inline
#define FV_HDM inline
#define FV_HDN static
#endif

// ---- tables: host copy (static arrays) + device copy (global memory) -------
#define FV_TABLE_DEFINED_BY_INCLUDER 1
#define FV_TABLE(type, name, n) static const type name##_h[n]
#include "fv_tables.h"
#undef FV_TABLE
#if defined(__CUDACC__)
#define FV_TABLE(type, name, n) static __device__ const type __align__(16) name##_d[n]
#include "fv_tables.h"
#undef FV_TABLE
#endif

#include "fv_consts.h"

#if defined(__CUDA_ARCH__)
#define FV_TAB(name, i) (__ldg(&name##_d[(i)]))
#else
#define FV_TAB(name, i) (name##_h[(i)])
#endif

FV_HD double fv_asdouble(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double d; memcpy(&d, &u, 8); return d;
#endif
}
FV_HD uint64_t fv_asuint64(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u; memcpy(&u, &d, 8); return u;
#endif
}
FV_HD double fv_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return __builtin_fma(a, b, c);
#endif
}
// Correctly rounded x / c for a constant divisor c, given yh = RN(1/c) and
// yl = RN(1/c - yh): q0 = RN(x*yh + x*yl) is within 1 ulp of x/c, the
// remainder r = x - q0*c is exact in one FMA, and Markstein's theorem makes
// RN(q0 + r*yh) the correctly rounded quotient -- i.e. the same bits as the
// IEEE division the reference performs, in 4 FP64 ops instead of a
// reciprocal-iteration division.  Out-of-range x (zero, tiny, huge, inf, nan)
// takes the plain division.  (Checked against x / c on 1.8e9 random inputs
// on CPU and on the B200: tests/test_libm_host.py, tests/test_gpu_parity.py.)
#define FV_DIV_CONST(x, c, yh, yl) fv_div_const((x), (c), (yh), (yl))
FV_HD double fv_div_const(double x, double c, double yh, double yl);
FV_HD uint32_t fv_top12(double x) { return (uint32_t)(fv_asuint64(x) >> 52); }
FV_HD int fv_isnan(double x) { return (fv_asuint64(x) & 0x7fffffffffffffffull) > 0x7ff0000000000000ull; }
FV_HD int fv_isinf(double x) { return (fv_asuint64(x) & 0x7fffffffffffffffull) == 0x7ff0000000000000ull; }
FV_HD int fv_isfinite(double x) { return (fv_asuint64(x) & 0x7ff0000000000000ull) != 0x7ff0000000000000ull; }
FV_HD double fv_fabs(double x) { return fv_asdouble(fv_asuint64(x) & 0x7fffffffffffffffull); }

FV_HDN double fv_div_slow(double x, double c) { return x / c; }   // cold: keep it out of line
FV_HD double fv_div_const(double x, double c, double yh, double yl) {
  double ax = fv_fabs(x);
  if (!(ax > 0x1p-900 && ax < 0x1p+900)) return fv_div_slow(x, c);
  double q0 = fv_fma(x, yh, x * yl);
  double r = fv_fma(-q0, c, x);
  return fv_fma(r, yh, q0);
}
#define FV_DIV_SQRT2(x) fv_div_const((x), FV_DIV_SQRT2_C, FV_DIV_SQRT2_YH, FV_DIV_SQRT2_YL)
#define FV_DIV_INT(x, d) fv_div_const((x), (double)(d), FV_DIV_##d##_YH, FV_DIV_##d##_YL)

// ---------------------------------------------------------------------------
// exp: glibc 2.39 sysdeps/ieee754/dbl-64/e_exp.c as built into __exp_fma.
// exp(x) = 2^(k/128) * exp(r); table scale*(1+tail); degree-5 polynomial.
// ---------------------------------------------------------------------------
FV_HDN double fv_exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {
    // k > 0: the exponent of scale might have overflowed by <= 460.
    sbits -= 1009ull << 52;
    double scale = fv_asdouble(sbits);
    return 0x1p1009 * fv_fma(scale, tmp, scale);
  }
  // k < 0: careful rounding in the subnormal range (not fused in the binary).
  sbits += 1022ull << 52;
  double scale = fv_asdouble(sbits);
  double st = scale * tmp;
  double y = scale + st;
  if (y < 1.0) {
    double lo = (scale - y) + st;
    double hi = 1.0 + y;
    lo = ((1.0 - hi) + y) + lo;
    y = (lo + hi) - 1.0;
    if (y == 0.0) y = 0.0;
  }
  return 0x1p-1022 * y;
}

// Core shared by exp (xtail = 0, sign_bias = 0) and pow's exp_inline.
template <bool kPow>
FV_HD double fv_exp_core(double x, double xtail, uint64_t sign_bias) {
  uint32_t abstop = fv_top12(x) & 0x7ff;
  if (abstop - 0x3c9u >= 0x3fu) {          // top12(0x1p-54), top12(512.0)
    if ((int32_t)(abstop - 0x3c9u) < 0) {  // tiny |x|: 1 + x
      double one = 1.0 + x;
      return sign_bias ? -one : one;
    }
    if (abstop >= 0x409) {                 // |x| >= 1024
      if (!kPow) {
        if (fv_asuint64(x) == 0xfff0000000000000ull) return 0.0;
        if (abstop >= 0x7ff) return 1.0 + x;
      }
      if (fv_asuint64(x) >> 63) return sign_bias ? -0.0 : 0.0;            // __math_uflow
      return sign_bias ? -__builtin_inf() : __builtin_inf();              // __math_oflow
    }
    abstop = 0;                            // large |x|: special-cased below
  }
  double kd = fv_fma(x, FV_EXP_INVLN2N, FV_EXP_SHIFT);
  uint64_t ki = fv_asuint64(kd);
  kd = kd - FV_EXP_SHIFT;
  double r = fv_fma(kd, FV_EXP_NEGLN2HIN, x);
  r = fv_fma(kd, FV_EXP_NEGLN2LON, r);
  if (kPow) r = xtail + r;
  uint32_t idx = 2u * (uint32_t)(ki & 127u);
  uint64_t top = (ki + sign_bias) << 45;
  double tail = fv_asdouble(FV_TAB(fv_exp_tab, idx));
  uint64_t sbits = FV_TAB(fv_exp_tab, idx + 1) + top;
  double p1 = fv_fma(r, FV_EXP_C3, FV_EXP_C2);
  double tr = r + tail;
  double r2 = r * r;
  double p2 = fv_fma(r, FV_EXP_C5, FV_EXP_C4);
  p1 = fv_fma(p1, r2, tr);
  double r4 = r2 * r2;
  double tmp = fv_fma(r4, p2, p1);
  if (abstop == 0) {
    if (!kPow) return fv_exp_specialcase(tmp, sbits, ki);
    // pow.c specialcase: signed scale, |y| < 1 test, sign-of-zero fix.
    if ((ki & 0x80000000ull) == 0) {
      sbits -= 1009ull << 52;
      double scale = fv_asdouble(sbits);
      return 0x1p1009 * fv_fma(scale, tmp, scale);
    }
    sbits += 1022ull << 52;
    double scale = fv_asdouble(sbits);
    double st = scale * tmp;
    double y = scale + st;
    if (fv_fabs(y) < 1.0) {
      double one = (y < 0.0) ? -1.0 : 1.0;
      double lo = (scale - y) + st;
      double hi = y + one;
      lo = ((one - hi) + y) + lo;
      y = (lo + hi) - one;
      if (y == 0.0) y = fv_asdouble(sbits & 0x8000000000000000ull);
    }
    return 0x1p-1022 * y;
  }
  double scale = fv_asdouble(sbits);
  return fv_fma(scale, tmp, scale);
}

FV_HD double fv_exp(double x) { return fv_exp_core<false>(x, 0.0, 0); }

// ---------------------------------------------------------------------------
// log: glibc 2.39 sysdeps/ieee754/dbl-64/e_log.c as built into __log_fma.
// ---------------------------------------------------------------------------
FV_HD double fv_log_i(double x) {
  uint64_t ix = fv_asuint64(x);
  uint32_t top = (uint32_t)(ix >> 48);
  if (ix - 0x3fee000000000000ull < 0x3090000000000ull) {  // |x - 1| < ~0x1p-4
    if (ix == 0x3ff0000000000000ull) return 0.0;
    double r = x - 1.0;
    double r2 = r * r;
    double r3 = r * r2;
    double q1 = fv_fma(r2, FV_LOG_B3, fv_fma(r, FV_LOG_B2, FV_LOG_B1));
    double q2 = fv_fma(r2, FV_LOG_B6, fv_fma(r, FV_LOG_B5, FV_LOG_B4));
    double q3 = fv_fma(r3, FV_LOG_B10, fv_fma(r2, FV_LOG_B9, fv_fma(r, FV_LOG_B8, FV_LOG_B7)));
    double poly = fv_fma(fv_fma(q3, r3, q2), r3, q1);
    double rw = fv_fma(r, 0x1p27, r);          // r + w, w = r*2^27 (fused)
    double rhi = fv_fma(-0x1p27, r, rw);       // (r + w) - w
    double rhi2 = rhi * rhi;
    double rlo = r - rhi;
    double hi = fv_fma(rhi2, FV_LOG_B0, r);    // r + rhi*rhi*B0
    double lo = fv_fma(rhi2, FV_LOG_B0, r - hi);
    lo = fv_fma(FV_LOG_B0 * rlo, rhi + r, lo);
    double y = fv_fma(poly, r3, lo);
    return hi + y;
  }
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
    if ((ix << 1) == 0) return -__builtin_inf();              // __math_divzero(1)
    if (ix == 0x7ff0000000000000ull) return x;                // log(inf) = inf
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u)
      return __builtin_nan("");                               // __math_invalid
    ix = fv_asuint64(x * 0x1p52);                             // subnormal
    ix -= 52ull << 52;
  }
  uint64_t tmp = ix - 0x3fe6000000000000ull;
  int i = (int)((tmp >> 45) & 127u);
  int k = (int)((int64_t)tmp >> 52);
  uint64_t iz = ix - (tmp & (0xfffull << 52));
  double invc = FV_TAB(fv_log_tab, 2 * i);
  double logc = FV_TAB(fv_log_tab, 2 * i + 1);
  double z = fv_asdouble(iz);
  double kd = (double)k;
  double w = fv_fma(kd, FV_LOG_LN2HI, logc);
  double r = fv_fma(z, invc, -1.0);
  double p1 = fv_fma(r, FV_LOG_A2, FV_LOG_A1);
  double hi = r + w;
  double r2 = r * r;
  double lo = fv_fma(kd, FV_LOG_LN2LO, (w - hi) + r);
  double r3 = r * r2;
  double p2 = fv_fma(r, FV_LOG_A4, FV_LOG_A3);
  double lo2 = fv_fma(r2, FV_LOG_A0, lo);
  double q = fv_fma(p2, r2, p1);
  double y = fv_fma(r3, q, lo2);
  return y + hi;
}

// ---------------------------------------------------------------------------
// pow: glibc 2.39 sysdeps/ieee754/dbl-64/e_pow.c as built into __pow_fma,
// for the inputs CPython's float_pow forwards to libm on this path: x finite
// and > 0 (float_pow strips the sign, zero, inf, nan and 1.0 itself) and y a
// small positive integer (2, 3, 4 at lbr.py:298, :342, :369, :376, :386).
// ---------------------------------------------------------------------------
FV_HD double fv_pow_pos_i(double x, double y) {
  uint64_t ix = fv_asuint64(x);
  if ((ix >> 52) == 0) {                       // subnormal x: normalize
    ix = fv_asuint64(x * 0x1p52);
    ix &= 0x7fffffffffffffffull;
    ix -= 52ull << 52;
  }
  // log_inline
  uint64_t tmp = ix - 0x3fe6955500000000ull;
  int i = (int)((tmp >> 45) & 127u);
  int k = (int)((int64_t)tmp >> 52);
  uint64_t iz = ix - (tmp & (0xfffull << 52));
  double z = fv_asdouble(iz);
  double kd = (double)k;
  double invc = FV_TAB(fv_powlog_tab, 3 * i);
  double logc = FV_TAB(fv_powlog_tab, 3 * i + 1);
  double logctail = FV_TAB(fv_powlog_tab, 3 * i + 2);
  double t1 = fv_fma(kd, FV_POW_LN2HI, logc);
  double lo1 = fv_fma(kd, FV_POW_LN2LO, logctail);
  double r = fv_fma(z, invc, -1.0);
  double ar = r * FV_POW_A0;
  double pa = fv_fma(r, FV_POW_A2, FV_POW_A1);
  double pb = fv_fma(r, FV_POW_A4, FV_POW_A3);
  double t2 = r + t1;
  double lo2 = (t1 - t2) + r;
  double ar2 = r * ar;
  double ar3 = r * ar2;
  double lo3 = fv_fma(ar, r, -ar2);
  double hi = t2 + ar2;
  double pc = fv_fma(r, FV_POW_A6, FV_POW_A5);
  double lo4 = (t2 - hi) + ar2;
  pc = fv_fma(pc, ar2, pb);
  pa = fv_fma(ar2, pc, pa);
  double lo = ((lo1 + lo2) + lo3) + lo4;
  lo = fv_fma(ar3, pa, lo);
  double lhi = hi + lo;
  double ltail = (hi - lhi) + lo;
  // y * log(x) as ehi + elo
  double ehi = y * lhi;
  double elo = fv_fma(y, ltail, fv_fma(lhi, y, -ehi));
  return fv_exp_core<true>(ehi, elo, 0);
}

// ---------------------------------------------------------------------------
// erfc: glibc 2.39 sysdeps/ieee754/dbl-64/s_erf.c (fdlibm-derived, Estrin-style
// pairs), built WITHOUT fma; its two exp calls resolve to __exp_fma (fv_exp).
// ---------------------------------------------------------------------------
template <bool kMergeInner, bool kMergeTail>
FV_HD double fv_erfc_t(double x) {
  uint64_t ux = fv_asuint64(x);
  int32_t hx = (int32_t)(ux >> 32);
  int32_t ix = hx & 0x7fffffff;
  if (ix >= 0x7ff00000) {  // erfc(nan) = nan, erfc(+-inf) = 0, 2
    return (double)(((uint32_t)hx >> 31) << 1) + 1.0 / x;
  }
  if (!kMergeInner && ix < 0x3feb0000) {   // |x| < 0.84375
    if (ix < 0x3c700000) return 1.0 - x;
    double z = x * x;
    double r1 = z * FV_ERFC_PP1 + FV_ERFC_PP0;
    double z2 = z * z;
    double r2 = z * FV_ERFC_PP3 + FV_ERFC_PP2;
    double z4 = z2 * z2;
    double s1 = z * FV_ERFC_QQ1 + 1.0;
    double s2 = z * FV_ERFC_QQ3 + FV_ERFC_QQ2;
    double s3 = z * FV_ERFC_QQ5 + FV_ERFC_QQ4;
    double r = (r1 + z2 * r2) + z4 * FV_ERFC_PP4;
    double s = (s1 + z2 * s2) + z4 * s3;
    double y = r / s;
    if (hx < 0x3fd00000) return 1.0 - (x + x * y);
    r = x * y;
    r = r + (x - 0.5);
    return 0.5 - r;
  }
  if (!kMergeInner && ix < 0x3ff40000) {   // 0.84375 <= |x| < 1.25
    double s = fv_fabs(x) - 1.0;
    double P1 = s * FV_ERFC_PA1 + FV_ERFC_PA0;
    double s2 = s * s;
    double Q1 = s * FV_ERFC_QA1 + 1.0;
    double s4 = s2 * s2;
    double P2 = s * FV_ERFC_PA3 + FV_ERFC_PA2;
    double s6 = s4 * s2;
    double Q2 = s * FV_ERFC_QA3 + FV_ERFC_QA2;
    double P3 = s * FV_ERFC_PA5 + FV_ERFC_PA4;
    double Q3 = s * FV_ERFC_QA5 + FV_ERFC_QA4;
    double P = ((P1 + s2 * P2) + s4 * P3) + s6 * FV_ERFC_PA6;
    double Q = ((Q1 + s2 * Q2) + s4 * Q3) + s6 * FV_ERFC_QA6;
    if (hx >= 0) return FV_ERFC_ONE_M_ERX - P / Q;
    double zz = FV_ERFC_ERX + P / Q;
    return 1.0 + zz;
  }
  if (kMergeInner && ix < 0x3ff40000) {   // |x| < 1.25
    if (ix < 0x3c700000) return 1.0 - x;
    // |x| < 0.84375 (pp/qq in u = x^2) and 0.84375 <= |x| < 1.25 (pa/qa in
    // u = |x| - 1) evaluate one shared rational form over a two-row table
    // (zero coefficients add exact +0s), then take their own final formula:
    // bit-identical to glibc's two branches without splitting the warp.
    const bool inner = ix < 0x3feb0000;
    const double u = inner ? x * x : fv_fabs(x) - 1.0;
    const int row = inner ? 0 : 16;
    double n0 = FV_TAB(fv_erfc_mid, row + 0), n1 = FV_TAB(fv_erfc_mid, row + 1);
    double n2 = FV_TAB(fv_erfc_mid, row + 2), n3 = FV_TAB(fv_erfc_mid, row + 3);
    double n4 = FV_TAB(fv_erfc_mid, row + 4), n5 = FV_TAB(fv_erfc_mid, row + 5);
    double n6 = FV_TAB(fv_erfc_mid, row + 6);
    double e1 = FV_TAB(fv_erfc_mid, row + 7), e2 = FV_TAB(fv_erfc_mid, row + 8);
    double e3 = FV_TAB(fv_erfc_mid, row + 9), e4 = FV_TAB(fv_erfc_mid, row + 10);
    double e5 = FV_TAB(fv_erfc_mid, row + 11), e6 = FV_TAB(fv_erfc_mid, row + 12);
    double N1 = u * n1 + n0;
    double u2 = u * u;
    double D1 = u * e1 + 1.0;
    double u4 = u2 * u2;
    double N2 = u * n3 + n2;
    double u6 = u4 * u2;
    double D2 = u * e3 + e2;
    double N3 = u * n5 + n4;
    double D3 = u * e5 + e4;
    double num = ((N1 + u2 * N2) + u4 * N3) + u6 * n6;
    double den = ((D1 + u2 * D2) + u4 * D3) + u6 * e6;
    double y = num / den;
    if (inner) {
      if (hx < 0x3fd00000) return 1.0 - (x + x * y);   // x < 1/4
      double r = x * y;
      r = r + (x - 0.5);
      return 0.5 - r;
    }
    if (hx >= 0) return FV_ERFC_ONE_M_ERX - y;
    double zz = FV_ERFC_ERX + y;
    return 1.0 + zz;
  }
  if (ix < 0x403c0000) {   // |x| < 28
    double ax = fv_fabs(x);
    double s = 1.0 / (x * x);
    // The two tail ranges (|x| < 1/0.35: ra/sa; else rb/sb) share one code
    // path over a two-row coefficient table: the rb row has explicit zeros
    // where rb/sb have no term, which only adds exact +0s, so every result
    // is bit-identical to glibc's two separate branches while neighbouring
    // lanes in different ranges no longer diverge.
    double R, S;
    if (!kMergeTail) {
    if (ix < 0x4006db6d) {
      double R1 = s * FV_ERFC_RA1 + FV_ERFC_RA0;
      double s2 = s * s;
      double S1 = s * FV_ERFC_SA1 + 1.0;
      double s4 = s2 * s2;
      double R2 = s * FV_ERFC_RA3 + FV_ERFC_RA2;
      double s6 = s4 * s2;
      double S2 = s * FV_ERFC_SA3 + FV_ERFC_SA2;
      double s8 = s4 * s4;
      double R3 = s * FV_ERFC_RA5 + FV_ERFC_RA4;
      double S3 = s * FV_ERFC_SA5 + FV_ERFC_SA4;
      double R4 = s * FV_ERFC_RA7 + FV_ERFC_RA6;
      double S4 = s * FV_ERFC_SA7 + FV_ERFC_SA6;
      R = ((R1 + s2 * R2) + s4 * R3) + s6 * R4;
      S = (((S1 + s2 * S2) + s4 * S3) + s6 * S4) + s8 * FV_ERFC_SA8;
    } else {
      if (hx < 0 && ix >= 0x40180000) return FV_K_TWO_M_TINY;
      double R1 = s * FV_ERFC_RB1 + FV_ERFC_RB0;
      double s2 = s * s;
      double S1 = s * FV_ERFC_SB1 + 1.0;
      double s4 = s2 * s2;
      double R2 = s * FV_ERFC_RB3 + FV_ERFC_RB2;
      double s6 = s4 * s2;
      double S2 = s * FV_ERFC_SB3 + FV_ERFC_SB2;
      double R3 = s * FV_ERFC_RB5 + FV_ERFC_RB4;
      double S3 = s * FV_ERFC_SB5 + FV_ERFC_SB4;
      double S4 = s * FV_ERFC_SB7 + FV_ERFC_SB6;
      R = ((R1 + s2 * R2) + s4 * R3) + s6 * FV_ERFC_RB6;
      S = ((S1 + s2 * S2) + s4 * S3) + s6 * S4;
    }
    } else {
    if (ix >= 0x4006db6d && hx < 0 && ix >= 0x40180000) return FV_K_TWO_M_TINY;  // x < -6
    const int row = (ix < 0x4006db6d) ? 0 : 16;
    double c0 = FV_TAB(fv_erfc_tail, row + 0), c1 = FV_TAB(fv_erfc_tail, row + 1);
    double c2 = FV_TAB(fv_erfc_tail, row + 2), c3 = FV_TAB(fv_erfc_tail, row + 3);
    double c4 = FV_TAB(fv_erfc_tail, row + 4), c5 = FV_TAB(fv_erfc_tail, row + 5);
    double c6 = FV_TAB(fv_erfc_tail, row + 6), c7 = FV_TAB(fv_erfc_tail, row + 7);
    double d1 = FV_TAB(fv_erfc_tail, row + 8), d2 = FV_TAB(fv_erfc_tail, row + 9);
    double d3 = FV_TAB(fv_erfc_tail, row + 10), d4 = FV_TAB(fv_erfc_tail, row + 11);
    double d5 = FV_TAB(fv_erfc_tail, row + 12), d6 = FV_TAB(fv_erfc_tail, row + 13);
    double d7 = FV_TAB(fv_erfc_tail, row + 14), d8 = FV_TAB(fv_erfc_tail, row + 15);
    double R1 = s * c1 + c0;
    double s2 = s * s;
    double S1 = s * d1 + 1.0;
    double s4 = s2 * s2;
    double R2 = s * c3 + c2;
    double s6 = s4 * s2;
    double S2 = s * d3 + d2;
    double s8 = s4 * s4;
    double R3 = s * c5 + c4;
    double S3 = s * d5 + d4;
    double R4 = s * c7 + c6;
    double S4 = s * d7 + d6;
    R = ((R1 + s2 * R2) + s4 * R3) + s6 * R4;
    S = (((S1 + s2 * S2) + s4 * S3) + s6 * S4) + s8 * d8;
    }
    double z = fv_asdouble(fv_asuint64(ax) & 0xffffffff00000000ull);
    double e1 = fv_exp(-z * z - 0.5625);
    double e2 = fv_exp((z - ax) * (z + ax) + R / S);
    double r = e1 * e2;
    if (hx > 0) return r / ax;
    return 2.0 - r / ax;
  }
  if (hx > 0) return 0.0;  // tiny*tiny
  return FV_K_TWO_M_TINY;
}

// ---------------------------------------------------------------------------
// erfcx: scipy 1.18.1 scipy.special.erfcx = xsf/Faddeeva erfcx (S. G.
// Johnson): 100-interval Chebyshev fit of erfcx(x) in y = 4/(4+x) for
// 0 <= x <= 50, continued fraction above, 2*exp(x^2) - erfcx(-x) below 0.
// scipy's x86-64 wheel is built without FMA: every op separately rounded.
// ---------------------------------------------------------------------------
FV_HD double fv_erfcx_y100(double y100) {
  int k = (int)y100;
  if (k >= 100) return 1.0;                    // y100 == 100 <=> x == 0
  double t = 2.0 * y100 - (double)(2 * k + 1);
  int b = 7 * k;
  double c0 = FV_TAB(fv_erfcx_tab, b + 0), c1 = FV_TAB(fv_erfcx_tab, b + 1);
  double c2 = FV_TAB(fv_erfcx_tab, b + 2), c3 = FV_TAB(fv_erfcx_tab, b + 3);
  double c4 = FV_TAB(fv_erfcx_tab, b + 4), c5 = FV_TAB(fv_erfcx_tab, b + 5);
  double c6 = FV_TAB(fv_erfcx_tab, b + 6);
  return c0 + (c1 + (c2 + (c3 + (c4 + (c5 + c6 * t) * t) * t) * t) * t) * t;
}

FV_HD double fv_erfcx_i(double x) {
  if (x >= 0.0) {
    if (x > 50.0) {
      const double ispi = FV_K_ISPI;  // 1/sqrt(pi)
      if (x > 5e7) return ispi / x;
      return ispi * ((x * x) * (x * x + 4.5) + 2.0) / (x * ((x * x) * (x * x + 5.0) + 3.75));
    }
    return fv_erfcx_y100(400.0 / (4.0 + x));
  }
  if (fv_isnan(x)) return x;
  if (x < FV_K_M26P7) return __builtin_inf();
  if (x < FV_K_M6P1) return 2.0 * fv_exp(x * x);
  return 2.0 * fv_exp(x * x) - fv_erfcx_y100(400.0 / (4.0 - x));
}

// Out-of-line entry points (the default everywhere: keeps kernels small);
// the *_i forms above are inlined only in the hot far-low solve kernel, where
// inlining lets independent evaluations overlap and constants stay in
// uniform registers.
FV_HDN double fv_log(double x) { return fv_log_i(x); }
FV_HDN double fv_pow_pos(double x, double y) { return fv_pow_pos_i(x, y); }
FV_HDN double fv_erfcx(double x) { return fv_erfcx_i(x); }
// Two builds of erfc: separate fdlibm branches (constants in the constant
// bank; best where neighbouring lanes share a range, e.g. the LBR anchors) and
// the merged-table form (best where lanes' arguments scatter over the ranges:
// pricing, Greeks, Halley).  Bit-identical; chosen per caller.
FV_HD double fv_erfc_i(double x) { return fv_erfc_t<false, false>(x); }
FV_HDN double fv_erfc(double x) { return fv_erfc_t<false, false>(x); }
FV_HDN double fv_erfc_m(double x) { return fv_erfc_t<true, false>(x); }
