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
