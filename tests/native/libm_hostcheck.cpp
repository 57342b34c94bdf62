// Host build of paper_2604_27210_b200/csrc/fv_libm.h for bit-comparison
// against the live glibc libm / scipy on CPU (test infrastructure only; the
// product path is the CUDA build of the same header).
// Build: g++ -O2 -ffp-contract=off -fno-fast-math -shared -fPIC
#include "../../paper_2604_27210_b200/csrc/fv_libm.h"
#include <math.h>
#include <stdint.h>

extern "C" {
#define ARR1(name, expr)                                                     \
  void name(const double* x, int64_t n, double* out) {                      \
    for (int64_t i = 0; i < n; ++i) { double v = x[i]; out[i] = (expr); }   \
  }
ARR1(fvh_exp, fv_exp(v))
ARR1(fvh_log, fv_log(v))
ARR1(fvh_erfc, fv_erfc(v))
ARR1(fvh_erfcx, fv_erfcx(v))
ARR1(glibc_exp, exp(v))
ARR1(glibc_log, log(v))
ARR1(glibc_erfc, erfc(v))
void fvh_pow(const double* x, const double* y, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = fv_pow_pos(x[i], y[i]);
}
void glibc_pow(const double* x, const double* y, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = pow(x[i], y[i]);
}
}

extern "C" {
// fv_div_const against the IEEE division for the constants the path uses
// (returns mismatches).
int64_t fvh_div_const_check(const double* x, int64_t n) {
  struct C { double c, yh, yl; } cs[] = {
      {FV_DIV_SQRT2_C, FV_DIV_SQRT2_YH, FV_DIV_SQRT2_YL},
      {6.0, FV_DIV_6_YH, FV_DIV_6_YL}, {120.0, FV_DIV_120_YH, FV_DIV_120_YL},
      {5040.0, FV_DIV_5040_YH, FV_DIV_5040_YL}, {362880.0, FV_DIV_362880_YH, FV_DIV_362880_YL},
      {39916800.0, FV_DIV_39916800_YH, FV_DIV_39916800_YL},
      {6227020800.0, FV_DIV_6227020800_YH, FV_DIV_6227020800_YL},
      {365.0, FV_DIV_365_YH, FV_DIV_365_YL}, {100.0, FV_DIV_100_YH, FV_DIV_100_YL}};
  int64_t bad = 0;
  for (const C& c : cs)
    for (int64_t i = 0; i < n; ++i) {
      volatile double cc = c.c;
      double a = fv_div_const(x[i], c.c, c.yh, c.yl), b = x[i] / cc;
      uint64_t ua, ub; memcpy(&ua, &a, 8); memcpy(&ub, &b, 8);
      if (ua != ub && !(a != a && b != b)) ++bad;
    }
  return bad;
}
}
extern "C" {
ARR1(fvh_erfc_m, fv_erfc_m(v))
ARR1(fvh_erfc_t11, (fv_erfc_t<true, true>(v)))
ARR1(fvh_erfc_t01, (fv_erfc_t<false, true>(v)))
}
