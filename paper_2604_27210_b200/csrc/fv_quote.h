// fv_quote.h -- per-quote device code for the batched pricing / Greeks /
// implied-vol path, __host__ __device__ (the CUDA kernels in fv_kernels.cu
// instantiate it; tests/native/quote_hostcheck.cpp compiles the same source
// for CPU pre-checks against the oracle).
//
// Restates, bit for bit, the reference's per-row arithmetic:
//   pricing.py:23-61 (black_kernel, price_black76, price_bsm)
//   greeks.py:45-98  (_core)
//   solver.py:40-161 (_raw_vega, implied_vol_halley)
//   lbr.py:48-486    (normalized Black, normalize_quote, anchors/regions,
//                     initial guesses, objective branches, Householder(3))
//   distributions.py:19-95 (norm_cdf, norm_pdf, AS241 inverse)
// on top of fv_libm.h (glibc/scipy-faithful exp/log/pow/erfc/erfcx).
//
// Differences from the Python are restricted to bit-neutral restructuring:
//   * common subexpressions computed once (the second _anchors() call of
//     initial_guess, lbr.py:325; the duplicated normalized_black_log in the
//     far-low Newton step, lbr.py:293/:299; log(F/K) and sqrt(t) inside the
//     Halley loop, solver.py:45/:122; the per-quote constants exp(+-x/2),
//     b_max - beta and ln(beta) of the far-high / far-low objectives; the
//     exp(-(h^2+t^2)/2) shared by normalized_black and normalized_vega);
//   * the discarded LBR residual (lbr.py:429, :484) is not evaluated -- it
//     cannot raise for any quote that reaches it (|x| <= 1419.6 there, so its
//     b_max = exp(x/2) > 0);
//   * Python exceptions are reported as codes (fv_exc) instead of unwinding;
//     every raising site is kept, with the Python-float vs numpy.float64
//     operand typing that decides whether a division by zero raises.
#pragma once
#include "fv_libm.h"

// ---- exception codes (same numbering as oracle/fvoracle.cpp) ---------------
#define FV_EXC_NONE 0
#define FV_EXC_MATH_RANGE 1     // OverflowError('math range error')
#define FV_EXC_MATH_DOMAIN 2    // ValueError('math domain error')
#define FV_EXC_ZERO_DIV 3       // ZeroDivisionError('float division by zero')
#define FV_EXC_POW_RANGE 4      // OverflowError(34, 'Numerical result out of range')
#define FV_EXC_DOM_FK 5         // DomainError('F and K must be positive')
#define FV_EXC_DOM_ATM_BETA 6   // DomainError('atm_inverse requires beta in (0, 1), got ...')
#define FV_EXC_DOM_INVCDF_P 7   // DomainError('inv_norm_cdf requires p in (0, 1), got ...')
#define FV_EXC_DOM_NB_X 8       // DomainError('normalized_black requires x <= 0, got ...')
#define FV_EXC_DOM_NB_S 9       // DomainError('normalized_black requires s > 0, got ...')
#define FV_EXC_DOM_OBJ_S 10     // DomainError('objective_branch requires s > 0, got ...')

// ---- statuses (solver.py:14-19; batch.py:270-274) --------------------------
#define FV_IV_CONVERGED 0
#define FV_IV_FELL_BACK 1
#define FV_IV_BELOW_INTRINSIC 2
#define FV_IV_ABOVE_UPPER 3
#define FV_IV_MAX_ITER 4
#define FV_GK_OK 0
#define FV_GK_EDGE 1

#define FV_REGION_NONE (-1)
#define FV_FAR_LOW 0
#define FV_NEAR_LOW 1
#define FV_NEAR_HIGH 2
#define FV_FAR_HIGH 3

struct FvExc {
  int code;
  int np;      // value is a numpy.float64 (repr "np.float64(...)")
  double val;  // value quoted by DomainError messages
  FV_HDM void raise(int c) { if (code == FV_EXC_NONE) { code = c; } }
  FV_HDM void raise_v(int c, double v, int is_np) {
    if (code == FV_EXC_NONE) { code = c; val = v; np = is_np; }
  }
};

// ---- CPython semantics -----------------------------------------------------
FV_HD double py_exp(double x, FvExc& e) {           // math.exp (math_1, can_overflow)
  double r = fv_exp(x);
  if (fv_isinf(r) && fv_isfinite(x)) e.raise(FV_EXC_MATH_RANGE);
  return r;
}
template <bool kInl>
FV_HD double py_log_t(double x, FvExc& e) {         // math.log (m_log)
  if (fv_isfinite(x)) {
    if (x > 0.0) return kInl ? fv_log_i(x) : fv_log(x);
    e.raise(FV_EXC_MATH_DOMAIN);
    return x == 0.0 ? -__builtin_inf() : __builtin_nan("");
  }
  if (fv_isnan(x) || x > 0.0) return x;
  e.raise(FV_EXC_MATH_DOMAIN);
  return __builtin_nan("");
}
FV_HD double py_log(double x, FvExc& e) { return py_log_t<false>(x, e); }
FV_HD double py_sqrt(double x, FvExc& e) {          // math.sqrt
  double r = sqrt(x);
  if (fv_isnan(r) && !fv_isnan(x)) e.raise(FV_EXC_MATH_DOMAIN);
  return r;
}
// float / float raises on a zero divisor; any numpy.float64 operand does not.
FV_HD double py_div(double a, double b, bool np, FvExc& e) {
  if (!np && b == 0.0) e.raise(FV_EXC_ZERO_DIV);
  return a / b;
}
// x ** n, n in {2,3,4}: float_pow for Python floats (OverflowError on an
// infinite result from finite x), npy_pow for numpy scalars; both reach
// glibc pow for finite x != 0 (|x| via CPython's sign handling).
template <bool kInl>
FV_HD double py_powi_t(double x, int n, bool np, FvExc& e) {
  if (!fv_isfinite(x) || x == 0.0) {
    if (fv_isnan(x)) return x;
    if (x == 0.0) return (n & 1) ? x : 0.0;
    return (x < 0.0 && (n & 1)) ? -__builtin_inf() : __builtin_inf();
  }
  double r = kInl ? fv_pow_pos_i(fv_fabs(x), (double)n) : fv_pow_pos(fv_fabs(x), (double)n);
  if (x < 0.0 && (n & 1)) r = -r;
  if (!np && fv_isinf(r)) e.raise(FV_EXC_POW_RANGE);
  return r;
}
FV_HD double py_powi(double x, int n, bool np, FvExc& e) { return py_powi_t<false>(x, n, np, e); }
FV_HD double py_max(double a, double b) { return (b > a) ? b : a; }   // builtins.max
FV_HD double py_min(double a, double b) { return (b < a) ? b : a; }   // builtins.min

// ---- distributions.py ------------------------------------------------------
FV_HD double fv_norm_cdf(double x) { return 0.5 * fv_erfc(FV_DIV_SQRT2(-x)); }
FV_HD double fv_norm_cdf_i(double x) { return 0.5 * fv_erfc_i(FV_DIV_SQRT2(-x)); }
// pricing / Greeks / Halley: arguments scatter over erfc's ranges across lanes
FV_HD double fv_norm_cdf_m(double x) { return 0.5 * fv_erfc_m(FV_DIV_SQRT2(-x)); }
FV_HD double fv_norm_pdf(double x) { return FV_INV_SQRT_TWO_PI * fv_exp(-0.5 * x * x); }

FV_HD double as241_poly(double c0, double c1, double c2, double c3, double c4, double c5,
                        double c6, double c7, double r) {
  double acc = 0.0;                              // distributions.py:56-60 (Horner from 0.0)
  acc = acc * r + c7; acc = acc * r + c6; acc = acc * r + c5; acc = acc * r + c4;
  acc = acc * r + c3; acc = acc * r + c2; acc = acc * r + c1; acc = acc * r + c0;
  return acc;
}
#define FV_AS241_POLY(L, r) as241_poly(FV_AS241_##L##0, FV_AS241_##L##1, FV_AS241_##L##2, \
  FV_AS241_##L##3, FV_AS241_##L##4, FV_AS241_##L##5, FV_AS241_##L##6, FV_AS241_##L##7, r)

// inv_norm_cdf (distributions.py:63-95).  p_np: p is a numpy scalar.  Out of
// line on the device, so it returns (x, type of x, exception code) by value;
// the DomainError value is p (the caller's).
struct IncRes { double x; int x_np; int code; };
FV_HDN IncRes fv_inv_norm_cdf_impl(double p, bool p_np) {
  IncRes o;
  FvExc e = {0, 0, 0.0};
  if (!(0.0 < p && p < 1.0)) { o.x = __builtin_nan(""); o.x_np = p_np; o.code = FV_EXC_DOM_INVCDF_P; return o; }
  double q = p - 0.5;
  double x;
  bool xnp;
  if (fv_fabs(q) <= FV_K_0P425) {
    double r = FV_K_0P180625 - q * q;
    x = q * FV_AS241_POLY(A, r) / FV_AS241_POLY(B, r);
    xnp = p_np;
  } else {
    double r = (q < 0.0) ? p : (1.0 - p);
    r = py_sqrt(-py_log(r, e), e);
    double val;
    if (r <= 5.0) {
      r = r - FV_K_1P6;
      val = py_div(FV_AS241_POLY(C, r), FV_AS241_POLY(D, r), false, e);
    } else {
      r = r - 5.0;
      val = py_div(FV_AS241_POLY(E, r), FV_AS241_POLY(F, r), false, e);
    }
    x = (q < 0.0) ? -val : val;
    xnp = false;
  }
  double pdf = fv_norm_pdf(x);
  if (pdf > 0.0) {
    double err = fv_norm_cdf(x) - p;
    double u = py_div(err, pdf, p_np, e);
    bool unp = p_np;
    x = x - py_div(u, 1.0 + 0.5 * x * u, unp || xnp, e);
    xnp = xnp || unp;
  }
  o.x = x; o.x_np = xnp; o.code = e.code;
  return o;
}
FV_HD double fv_inv_norm_cdf(double p, bool p_np, bool* x_np, FvExc& e) {
  IncRes o = fv_inv_norm_cdf_impl(p, p_np);
  if (o.code == FV_EXC_DOM_INVCDF_P) e.raise_v(o.code, p, p_np);
  else if (o.code) e.raise(o.code);
  *x_np = o.x_np != 0;
  return o.x;
}

// ---- pricing.py black_kernel (:23-33) ---------------------------------------
// lnFK = log(F/K) computed by the caller (bit-identical each call); fk_bad:
// F/K <= 0 so math.log raises once the kernel reaches it.
FV_HD double fv_black_kernel(double th, double Fw, double K, double disc, double s,
                             double lnFK, bool fk_bad, FvExc& e) {
  double intrinsic = py_max(th * (Fw - K), 0.0);
  double cap = (th > 0.0) ? Fw : K;
  if (s < FV_K_1EM12) return disc * intrinsic;
  if (fk_bad) e.raise(FV_EXC_MATH_DOMAIN);
  double d1 = (lnFK + 0.5 * s * s) / s;
  double d2 = d1 - s;
  double raw = th * (Fw * fv_norm_cdf_m(th * d1) - K * fv_norm_cdf_m(th * d2));
  return disc * py_min(py_max(raw, intrinsic), cap);
}

// math.log(F / K) evaluated once per quote; *bad: the call raises
// ValueError('math domain error') whenever the reference reaches it.
FV_HD double fv_log_fk(double FK, bool* bad) {
  FvExc tmp = {0, 0, 0.0};
  double v = py_log(FK, tmp);
  *bad = tmp.code != FV_EXC_NONE;
  return v;
}

// batch_price row (batch.py:195-198): model 0 = Black-76, else spot (BS/BSM).
FV_HD double fv_price_row(int model, double th, double un, double K, double t, double r,
                          double q, double sigma, FvExc& e) {
  double Fw = un;
  if (model != 0) Fw = un * py_exp((r - q) * t, e);
  double disc = py_exp(-r * t, e);
  double s = sigma * sqrt(t);
  bool bad;
  double lnFK = fv_log_fk(Fw / K, &bad);
  return fv_black_kernel(th, Fw, K, disc, s, lnFK, bad, e);
}

// ---- fused price + Greeks (pricing.py:56-61 + greeks.py:45-98) -------------
// One pass over d1/d2/Phi/phi for both reference calls (batch_price and
// batch_greeks); each keeps its own exception record (ep / eg).
struct FvGreeks { double price, delta, gamma, theta, rho, vega; int status; };

FV_HD FvGreeks fv_price_greeks_row(int model, double th, double un, double K, double t,
                                   double r, double q, double sigma, bool want_price,
                                   bool want_greeks, FvExc& ep, FvExc& eg) {
  FvGreeks o;
  const double nan = __builtin_nan("");
  o.price = nan; o.delta = nan; o.gamma = nan; o.theta = nan; o.rho = nan; o.vega = nan;
  o.status = FV_GK_OK;
  bool fwd = (model == 0);
  double sqrt_t = sqrt(t);
  double s = sigma * sqrt_t;
  // pricing: F (spot), disc ; greeks: disc, edge check, F, carry_disc
  double eFq = 1.0;
  FvExc e0 = {0, 0, 0.0};
  if (!fwd) eFq = py_exp((r - q) * t, e0);          // both reference calls evaluate this
  double disc = fv_exp(-r * t);
  bool disc_ovf = fv_isinf(disc) && fv_isfinite(-r * t);
  double Fw = fwd ? un : un * eFq;
  // batch_price: F (spot) -> disc -> kernel
  if (want_price) {
    if (e0.code) ep.raise(e0.code);
    if (disc_ovf) ep.raise(FV_EXC_MATH_RANGE);
  }
  // batch_greeks: disc -> (edge) -> F -> carry_disc -> log
  bool edge = s < FV_K_1EM12;
  double carry_disc = disc;
  if (want_greeks) {
    if (disc_ovf) eg.raise(FV_EXC_MATH_RANGE);
    if (!edge && !fwd) {
      if (e0.code) eg.raise(e0.code);
      carry_disc = py_exp(-q * t, eg);
    }
    if (edge && eg.code == FV_EXC_NONE) o.status = FV_GK_EDGE;
  }
  double intrinsic = py_max(th * (Fw - K), 0.0);
  double cap = (th > 0.0) ? Fw : K;
  if (s < FV_K_1EM12) {
    o.price = disc * intrinsic;
    return o;
  }
  bool bad;
  double lnFK = fv_log_fk(Fw / K, &bad);
  if (bad) { if (want_price) ep.raise(FV_EXC_MATH_DOMAIN); if (want_greeks) eg.raise(FV_EXC_MATH_DOMAIN); }
  double d1 = (lnFK + 0.5 * s * s) / s;
  double d2 = d1 - s;
  double cdf_td1 = fv_norm_cdf_m(th * d1);
  double cdf_td2 = fv_norm_cdf_m(th * d2);
  double raw = th * (Fw * cdf_td1 - K * cdf_td2);
  o.price = disc * py_min(py_max(raw, intrinsic), cap);
  if (!want_greeks) return o;
  double under = fwd ? Fw : un;
  double pdf_d1 = fv_norm_pdf(d1);
  o.delta = th * carry_disc * cdf_td1;
  o.gamma = carry_disc * pdf_d1 / (under * s);
  double vega = carry_disc * under * pdf_d1 * sqrt_t;
  double theta_cal, rho;
  if (fwd) {
    double value = disc * th * (Fw * cdf_td1 - K * cdf_td2);
    theta_cal = r * value - disc * Fw * pdf_d1 * sigma / (2.0 * sqrt_t);
    rho = -t * value;
  } else {
    theta_cal = (-under * carry_disc * pdf_d1 * sigma / (2.0 * sqrt_t)
                 - th * (r * K * disc * cdf_td2 - q * under * carry_disc * cdf_td1));
    rho = th * K * t * disc * cdf_td2;
  }
  o.theta = FV_DIV_INT(theta_cal, 365);
  o.rho = FV_DIV_INT(rho, 100);
  o.vega = FV_DIV_INT(vega, 100);
  return o;
}

// ---- solver.py implied_vol_halley (:49-161), two phases ---------------------
// Phase 1 (setup + <= 16 Halley steps) either finishes the quote or hands a
// compact state to phase 2 (<= 128 bisection steps), so the ~4% of quotes
// that need the long bisection tail run on their own, warp-dense.
struct FvHalleyCtx {       // per-quote constants
  double th, Fw, K, disc, sqrt_t, lnFK, target, tol_price;
  bool fk_bad;
};
struct FvHalleyState { double sigma, fval, lo, hi; int iterations; };

FV_HD double fv_halley_f(const FvHalleyCtx& c, double sigma, FvExc& e) {
  return fv_black_kernel(c.th, c.Fw, c.K, c.disc, sigma * c.sqrt_t, c.lnFK, c.fk_bad, e) - c.target;
}

// Returns 1 if the quote is finished (status/sigma/iterations set), 0 if it
// needs the bisection phase (ctx/state filled).
FV_HD int fv_halley_phase1(int model, double th, double un, double K, double t, double r,
                           double q, double target, FvHalleyCtx& c, FvHalleyState& st,
                           int* status, double* sigma_out, FvExc& e) {
  const double nan = __builtin_nan("");
  *sigma_out = nan;
  st.iterations = 0;
  double Fw = (model == 0) ? un : un * py_exp((r - q) * t, e);
  double discount = py_exp(-r * t, e);
  double sqrt_t = sqrt(t);
  if (e.code) { *status = FV_IV_MAX_ITER; return 1; }
  double disc_intrinsic = discount * py_max(th * (Fw - K), 0.0);
  double disc_cap = discount * ((th > 0.0) ? Fw : K);
  double tie_tol = FV_K_1EM12 * py_max(1.0, disc_cap);
  if (!fv_isfinite(target)) { *status = FV_IV_BELOW_INTRINSIC; return 1; }
  if (target <= disc_intrinsic + tie_tol) { *status = FV_IV_BELOW_INTRINSIC; return 1; }
  if (target > disc_cap + tie_tol) { *status = FV_IV_ABOVE_UPPER; return 1; }
  double tol_price = py_min(tie_tol, FV_K_1EM10 * (target - disc_intrinsic));
  if (t <= 0.0) { *status = FV_IV_ABOVE_UPPER; return 1; }
  c.th = th; c.Fw = Fw; c.K = K; c.disc = discount; c.sqrt_t = sqrt_t;
  c.lnFK = fv_log_fk(Fw / K, &c.fk_bad);
  c.target = target; c.tol_price = tol_price;

  double lo = FV_K_1EM9, hi = 10.0;
  double f_lo = fv_halley_f(c, lo, e);
  if (e.code) { *status = FV_IV_MAX_ITER; return 1; }
  if (f_lo >= 0.0) {
    if (fv_fabs(f_lo) <= tol_price) { *status = FV_IV_CONVERGED; *sigma_out = lo; return 1; }
    *status = FV_IV_BELOW_INTRINSIC; return 1;
  }
  double f_hi = fv_halley_f(c, hi, e);
  while (f_hi < 0.0 && hi < 100.0) {
    hi = py_min(2.0 * hi, 100.0);
    f_hi = fv_halley_f(c, hi, e);
  }
  if (f_hi < 0.0) { *status = FV_IV_MAX_ITER; return 1; }
  double sigma = sqrt(FV_TWO_PI / t) * target / un;
  sigma = py_min(py_max(sigma, FV_K_0P05), 2.0);
  sigma = py_min(py_max(sigma, lo), hi);
  double fval = fv_halley_f(c, sigma, e);
  if (fval > 0.0) hi = py_min(hi, sigma);
  else if (fval < 0.0) lo = py_max(lo, sigma);
  int iterations = 0;
  for (int it = 0; it < 16; ++it) {
    if (fv_fabs(fval) <= tol_price) {
      *status = FV_IV_CONVERGED; *sigma_out = sigma; st.iterations = iterations; return 1;
    }
    // _raw_vega (solver.py:40-46) and the d1/d2 of :121-123 share s and d1
    double s = sigma * sqrt_t;
    double vega = 0.0, d1 = 0.0;
    if (!(s < FV_K_1EM12)) {
      if (c.fk_bad) e.raise(FV_EXC_MATH_DOMAIN);
      d1 = (c.lnFK + 0.5 * s * s) / s;
      vega = discount * Fw * fv_norm_pdf(d1) * sqrt_t;
    }
    double cand = nan;
    if (vega > 0.0) {
      double d2 = d1 - s;
      double vomma = vega * d1 * d2 / sigma;
      double denom = 2.0 * vega * vega - fval * vomma;
      if (denom != 0.0) cand = sigma - 2.0 * fval * vega / denom;
    }
    bool accepted = false;
    double f_cand = 0.0;
    if (fv_isfinite(cand) && lo < cand && cand < hi) {
      f_cand = fv_halley_f(c, cand, e);
      if (fv_fabs(f_cand) < fv_fabs(fval)) accepted = true;
    }
    if (!accepted) {
      cand = 0.5 * (lo + hi);
      f_cand = fv_halley_f(c, cand, e);
    }
    if (e.code) { *status = FV_IV_MAX_ITER; return 1; }
    if (f_cand > 0.0) hi = cand;
    else if (f_cand < 0.0) lo = cand;
    double step = cand - sigma;
    sigma = cand; fval = f_cand;
    iterations += 1;
    if (fv_fabs(step) <= FV_K_1EM12 * py_max(1.0, sigma)) {
      *status = FV_IV_CONVERGED; *sigma_out = sigma; st.iterations = iterations; return 1;
    }
  }
  st.sigma = sigma; st.fval = fval; st.lo = lo; st.hi = hi; st.iterations = iterations;
  return 0;
}

// Phase 2: solver.py:146-161.
FV_HD void fv_halley_phase2(const FvHalleyCtx& c, FvHalleyState st, int* status,
                            double* sigma_out, FvExc& e) {
  double sigma = st.sigma, fval = st.fval, lo = st.lo, hi = st.hi;
  for (int it = 0; it < 128; ++it) {
    if (fv_fabs(fval) <= c.tol_price || (hi - lo) <= FV_K_1EM12 * py_max(1.0, sigma)) {
      *status = FV_IV_FELL_BACK; *sigma_out = sigma; return;
    }
    sigma = 0.5 * (lo + hi);
    fval = fv_halley_f(c, sigma, e);
    if (fval > 0.0) hi = sigma;
    else lo = sigma;
  }
  if (fv_fabs(fval) <= c.tol_price || (hi - lo) <= FV_K_1EM12 * py_max(1.0, sigma)) {
    *status = FV_IV_FELL_BACK; *sigma_out = sigma; return;
  }
  *status = FV_IV_MAX_ITER; *sigma_out = __builtin_nan("");
}

// ---- solver.py implied_vol_halley as a per-lane state machine ---------------
// The GPU form of :49-161.  Every step of the solver is "decide sigma ->
// evaluate f(sigma) = black_kernel(...) - target -> update"; the kernel runs
// that step for all lanes in lockstep (the expensive black_kernel is the
// shared code) and refills a lane as soon as its quote finishes, so neither
// the spread of Halley iteration counts nor the 51-60-step bisection tail of
// ~4% of quotes leaves lanes idle.  The sequence of f evaluations and every
// value per quote are exactly the reference's.
#define FV_HS_DONE 0
#define FV_HS_LO 1       // f(SIGMA_LO)                      :91-96
#define FV_HS_HI 2       // f(hi), doubling while negative    :97-102
#define FV_HS_GUESS 3    // f(guess)                          :104-112
#define FV_HS_ITER 4     // Halley candidate (needs vega)     :115-135
#define FV_HS_CHECK 5    // f(cand) evaluated: accept?        :129-132
#define FV_HS_MID 6      // rejected: f(mid)                  :133-135
#define FV_HS_BISECT 7   // bisection tail                    :147-157

struct FvHalleySM {
  FvHalleyCtx c;
  double lo, hi, sigma, fval, cand, guess;
  int state, k, iterations, status;
  double out_sigma;
};

FV_HD void fv_hsm_finish(FvHalleySM& m, int status, double sigma) {
  m.state = FV_HS_DONE; m.status = status; m.out_sigma = sigma;
}

// :60-86 (everything before the first f evaluation).  Returns 1 when the
// quote is already finished (bounds / t <= 0 / exception).
FV_HD int fv_hsm_setup(int model, double th, double un, double K, double t, double r, double q,
                       double target, FvHalleySM& m, FvExc& e) {
  const double nan = __builtin_nan("");
  m.iterations = 0; m.k = 0;
  double Fw = (model == 0) ? un : un * py_exp((r - q) * t, e);
  double discount = py_exp(-r * t, e);
  double sqrt_t = sqrt(t);
  if (e.code) { fv_hsm_finish(m, FV_IV_MAX_ITER, nan); return 1; }
  double disc_intrinsic = discount * py_max(th * (Fw - K), 0.0);
  double disc_cap = discount * ((th > 0.0) ? Fw : K);
  double tie_tol = FV_K_1EM12 * py_max(1.0, disc_cap);
  if (!fv_isfinite(target)) { fv_hsm_finish(m, FV_IV_BELOW_INTRINSIC, nan); return 1; }
  if (target <= disc_intrinsic + tie_tol) { fv_hsm_finish(m, FV_IV_BELOW_INTRINSIC, nan); return 1; }
  if (target > disc_cap + tie_tol) { fv_hsm_finish(m, FV_IV_ABOVE_UPPER, nan); return 1; }
  double tol_price = py_min(tie_tol, FV_K_1EM10 * (target - disc_intrinsic));
  if (t <= 0.0) { fv_hsm_finish(m, FV_IV_ABOVE_UPPER, nan); return 1; }
  m.c.th = th; m.c.Fw = Fw; m.c.K = K; m.c.disc = discount; m.c.sqrt_t = sqrt_t;
  m.c.lnFK = fv_log_fk(Fw / K, &m.c.fk_bad);
  m.c.target = target; m.c.tol_price = tol_price;
  m.guess = sqrt(FV_TWO_PI / t) * target / un;            // :105, before clamping
  m.lo = FV_K_1EM9; m.hi = 10.0;
  m.state = FV_HS_LO;
  return 0;
}

// Decide where this step evaluates f.  Returns 0 if the quote finished
// without needing an evaluation (m.state == DONE).
FV_HD int fv_hsm_pre(FvHalleySM& m, double* x, FvExc& e) {
  const double nan = __builtin_nan("");
  switch (m.state) {
    case FV_HS_LO: *x = m.lo; return 1;
    case FV_HS_HI: *x = m.hi; return 1;
    case FV_HS_GUESS: *x = m.sigma; return 1;
    case FV_HS_MID: *x = m.cand; return 1;
    case FV_HS_ITER: {
      if (fv_fabs(m.fval) <= m.c.tol_price) { fv_hsm_finish(m, FV_IV_CONVERGED, m.sigma); return 0; }
      // _raw_vega (:40-46) and the d1/d2 of :121-123 share s and d1
      const double sigma = m.sigma, sqrt_t = m.c.sqrt_t;
      double s = sigma * sqrt_t;
      double vega = 0.0, d1 = 0.0;
      if (!(s < FV_K_1EM12)) {
        if (m.c.fk_bad) { e.raise(FV_EXC_MATH_DOMAIN); fv_hsm_finish(m, FV_IV_MAX_ITER, nan); return 0; }
        d1 = (m.c.lnFK + 0.5 * s * s) / s;
        vega = m.c.disc * m.c.Fw * fv_norm_pdf(d1) * sqrt_t;
      }
      double cand = nan;
      if (vega > 0.0) {
        double d2 = d1 - s;
        double vomma = vega * d1 * d2 / sigma;
        double denom = 2.0 * vega * vega - m.fval * vomma;
        if (denom != 0.0) cand = sigma - 2.0 * m.fval * vega / denom;
      }
      if (fv_isfinite(cand) && m.lo < cand && cand < m.hi) { m.cand = cand; m.state = FV_HS_CHECK; }
      else { m.cand = 0.5 * (m.lo + m.hi); m.state = FV_HS_MID; }
      *x = m.cand;
      return 1;
    }
    case FV_HS_BISECT: {
      if (fv_fabs(m.fval) <= m.c.tol_price || (m.hi - m.lo) <= FV_K_1EM12 * py_max(1.0, m.sigma)) {
        fv_hsm_finish(m, FV_IV_FELL_BACK, m.sigma); return 0;
      }
      m.sigma = 0.5 * (m.lo + m.hi);
      *x = m.sigma;
      return 1;
    }
  }
  return 0;
}

// Consume fx = f(x) for the evaluation decided by fv_hsm_pre.
FV_HD void fv_hsm_post(FvHalleySM& m, double fx, FvExc& e) {
  const double nan = __builtin_nan("");
  if (e.code) { fv_hsm_finish(m, FV_IV_MAX_ITER, nan); return; }
  switch (m.state) {
    case FV_HS_LO:                                         // :92-96
      if (fx >= 0.0) {
        if (fv_fabs(fx) <= m.c.tol_price) fv_hsm_finish(m, FV_IV_CONVERGED, m.lo);
        else fv_hsm_finish(m, FV_IV_BELOW_INTRINSIC, nan);
        return;
      }
      m.state = FV_HS_HI;
      return;
    case FV_HS_HI:                                         // :97-112
      if (fx < 0.0 && m.hi < 100.0) { m.hi = py_min(2.0 * m.hi, 100.0); return; }
      if (fx < 0.0) { fv_hsm_finish(m, FV_IV_MAX_ITER, nan); return; }
      {
        double sigma = py_min(py_max(m.guess, FV_K_0P05), 2.0);
        m.sigma = py_min(py_max(sigma, m.lo), m.hi);
      }
      m.state = FV_HS_GUESS;
      return;
    case FV_HS_GUESS:                                      // :108-112
      m.fval = fx;
      if (fx > 0.0) m.hi = py_min(m.hi, m.sigma);
      else if (fx < 0.0) m.lo = py_max(m.lo, m.sigma);
      m.k = 0; m.iterations = 0;
      m.state = FV_HS_ITER;
      return;
    case FV_HS_CHECK:                                      // :129-132
      if (!(fv_fabs(fx) < fv_fabs(m.fval))) {              // rejected -> f(mid)
        m.cand = 0.5 * (m.lo + m.hi);
        m.state = FV_HS_MID;
        return;
      }
      // fall through: accepted
    case FV_HS_MID: {                                      // :136-144
      const double cand = m.cand;
      if (fx > 0.0) m.hi = cand;
      else if (fx < 0.0) m.lo = cand;
      double step = cand - m.sigma;
      m.sigma = cand; m.fval = fx;
      m.iterations += 1;
      if (fv_fabs(step) <= FV_K_1EM12 * py_max(1.0, m.sigma)) { fv_hsm_finish(m, FV_IV_CONVERGED, m.sigma); return; }
      m.k += 1;
      if (m.k == 16) { m.k = 0; m.state = FV_HS_BISECT; }
      else m.state = FV_HS_ITER;
      return;
    }
    case FV_HS_BISECT:                                     // :151-161
      m.fval = fx;
      if (fx > 0.0) m.hi = m.sigma;
      else m.lo = m.sigma;
      m.iterations += 1;
      m.k += 1;
      if (m.k == 128) {
        if (fv_fabs(m.fval) <= m.c.tol_price || (m.hi - m.lo) <= FV_K_1EM12 * py_max(1.0, m.sigma))
          fv_hsm_finish(m, FV_IV_FELL_BACK, m.sigma);
        else fv_hsm_finish(m, FV_IV_MAX_ITER, nan);
      }
      return;
  }
}

// Whole solver for one row through the state machine (host checks, explain).
FV_HD void fv_halley_row_sm(int model, double th, double un, double K, double t, double r,
                            double q, double target, int* status, double* sigma, FvExc& e) {
  FvHalleySM m;
  if (!fv_hsm_setup(model, th, un, K, t, r, q, target, m, e)) {
    for (;;) {
      double x;
      if (!fv_hsm_pre(m, &x, e)) break;
      double fx = fv_halley_f(m.c, x, e);
      fv_hsm_post(m, fx, e);
      if (m.state == FV_HS_DONE) break;
    }
  }
  *status = m.status;
  *sigma = (m.status == FV_IV_CONVERGED || m.status == FV_IV_FELL_BACK) ? m.out_sigma : __builtin_nan("");
}

// ---- lbr.py: normalized Black --------------------------------------------
// normalized_black (:112-129) for Python-float x (x_work) and s of numpy-ness
// s_np.  *E (if non-null) receives exp(-(h^2+t^2)/2) -- the factor
// normalized_vega (:152-156) shares -- computed here when the branch needs it.
#ifndef FV_NB_INLINE_ERFCX
#define FV_NB_INLINE_ERFCX 0
#endif
#if FV_NB_INLINE_ERFCX
#define FV_NB_ERFCX(x) fv_erfcx_i(x)
#else
#define FV_NB_ERFCX(x) fv_erfcx(x)
#endif
struct NbRes { double b; double E; int code; int branch; };
FV_HDN NbRes fv_normalized_black_impl(double x, double s, bool s_np) {
  NbRes o;
  o.E = 0.0; o.code = 0; o.branch = -1;
  FvExc e = {0, 0, 0.0};
  if (x > 0.0) { o.b = __builtin_nan(""); o.code = FV_EXC_DOM_NB_X; return o; }
  if (!(s > 0.0)) { o.b = __builtin_nan(""); o.code = FV_EXC_DOM_NB_S; return o; }
  double h = py_div(x, s, s_np, e);
  double t = 0.5 * s;
  if (h < -10.0 && t < FV_SMALL_T_THRESHOLD + (-10.0 - h)) {
    // _asymptotic_black (:65-71)
    o.branch = 0;
    double th_ = py_div(t, h, s_np, e);
    double ee = th_ * th_;
    double rr = (h + t) * (h - t);
    double hr = py_div(h, rr, s_np, e);
    double qq = hr * hr;
    double c0 = 0.0;
    for (int j = 17; j >= 0; --j) {
      // column j of _ASYM_PASCAL: P[0..j][j] (zeros above the diagonal are
      // bit-neutral in numpy's Horner since e is finite and >= 0)
      int base = j * (j + 1) / 2;
      double cj = FV_TAB(fv_asym_pascal, base + j) + ee * 0.0;
      for (int i = j - 1; i >= 0; --i) cj = FV_TAB(fv_asym_pascal, base + i) + cj * ee;
      double wj = FV_TAB(fv_asym_facts, j) * cj;
      c0 = (j == 17) ? (wj + qq * 0.0) : (wj + c0 * qq);
    }
    double Ev = fv_exp(-0.5 * (h * h + t * t));
    o.E = Ev;
    double b = FV_INV_SQRT_TWO_PI * Ev * py_div(t, rr, s_np, e) * c0;
    o.b = py_max(b, 0.0); o.code = e.code; return o;
  }
  if (t < FV_SMALL_T_THRESHOLD) {
    // _small_t_black (:74-103)
    o.branch = 1;
    double a = 1.0 + h * FV_HALF_SQRT_TWO_PI * FV_NB_ERFCX(FV_DIV_SQRT2(-h));
    double w = t * t;
    double h2 = h * h;
    double c1 = FV_DIV_INT(-1.0 + 3.0 * a + a * h2, 6);
    double c2 = FV_DIV_INT(-7.0 + 15.0 * a + h2 * (-1.0 + 10.0 * a + a * h2), 120);
    double c3 = FV_DIV_INT(-57.0 + 105.0 * a + h2 * (-18.0 + 105.0 * a + h2 * (-1.0 + 21.0 * a + a * h2)), 5040);
    double c4 = FV_DIV_INT(-561.0 + 945.0 * a + h2 * (-285.0 + 1260.0 * a + h2 * (-33.0 + 378.0 * a
                 + h2 * (-1.0 + 36.0 * a + a * h2))), 362880);
    double c5 = FV_DIV_INT(-6555.0 + 10395.0 * a + h2 * (-4680.0 + 17325.0 * a + h2 * (-840.0 + 6930.0 * a
                 + h2 * (-52.0 + 990.0 * a + h2 * (-1.0 + 55.0 * a + a * h2)))), 39916800);
    double c6 = FV_DIV_INT(-89055.0 + 135135.0 * a + h2 * (-82845.0 + 270270.0 * a + h2 * (-20370.0 + 135135.0 * a
                 + h2 * (-1926.0 + 25740.0 * a + h2 * (-75.0 + 2145.0 * a
                 + h2 * (-1.0 + 78.0 * a + a * h2))))), 6227020800);
    double expansion = 2.0 * t * (a + w * (c1 + w * (c2 + w * (c3 + w * (c4 + w * (c5 + w * c6))))));
    double Ev = fv_exp(-0.5 * (h * h + t * t));
    o.E = Ev;
    double b = FV_INV_SQRT_TWO_PI * Ev * expansion;
    o.b = py_max(b, 0.0); o.code = e.code; return o;
  }
  if (h + t > FV_K_0P85) {
    o.branch = 2;
    double b_max = fv_exp(0.5 * x);
    double b = fv_norm_cdf(h + t) * b_max - py_div(fv_norm_cdf(h - t), b_max, false, e);
    o.E = fv_exp(-0.5 * (h * h + t * t));
    o.b = py_max(b, 0.0); o.code = e.code; return o;
  }
  // _erfcx_black (:106-109)
  o.branch = 3;
  double Ev = fv_exp(-0.5 * (h * h + t * t));
  o.E = Ev;
  double b = 0.5 * Ev * (FV_NB_ERFCX(FV_DIV_SQRT2(-(h + t))) - FV_NB_ERFCX(FV_DIV_SQRT2(-(h - t))));
  o.b = py_max(b, 0.0); o.code = e.code; return o;
}

FV_HD double fv_normalized_black(double x, double s, bool s_np, FvExc& e, double* E, int* branch) {
  NbRes o = fv_normalized_black_impl(x, s, s_np);
  if (o.code == FV_EXC_DOM_NB_X) e.raise_v(o.code, x, 0);
  else if (o.code == FV_EXC_DOM_NB_S) e.raise_v(o.code, s, s_np);
  else if (o.code) e.raise(o.code);
  if (E) *E = o.E;
  if (branch) *branch = o.branch;
  return o.b;
}

// normalized_black_log (:140-149)
struct DRes { double v; int code; };
FV_HDN DRes fv_normalized_black_log_impl(double x, double s, bool s_np) {
  FvExc e = {0, 0, 0.0};
  DRes o;
  double h = py_div(x, s, s_np, e);
  double t = 0.5 * s;
  double diff = fv_erfcx(FV_DIV_SQRT2(-(h + t))) - fv_erfcx(FV_DIV_SQRT2(-(h - t)));
  if (diff <= 0.0) { o.v = -__builtin_inf(); o.code = e.code; return o; }
  o.v = -0.5 * (h * h + t * t) + py_log(0.5 * diff, e);
  o.code = e.code;
  return o;
}
FV_HD double fv_normalized_black_log(double x, double s, bool s_np, FvExc& e) {
  DRes o = fv_normalized_black_log_impl(x, s, s_np);
  if (o.code) e.raise(o.code);
  return o.v;
}
// Inline form for the far-low kernel, with h = x / s supplied by the caller
// (the same division the caller needs anyway; its ZeroDivisionError check is
// the caller's).
template <bool kInl>
FV_HD double fv_nbl_h(double h, double s, FvExc& e) {
  double t = 0.5 * s;
  double a1 = FV_DIV_SQRT2(-(h + t)), a2 = FV_DIV_SQRT2(-(h - t));
  double diff = kInl ? (fv_erfcx_i(a1) - fv_erfcx_i(a2)) : (fv_erfcx(a1) - fv_erfcx(a2));
  if (diff <= 0.0) return -__builtin_inf();
  return -0.5 * (h * h + t * t) + py_log_t<kInl>(0.5 * diff, e);
}

// normalized_black_complement (:132-137) with the per-quote exp(+-x/2)
FV_HDN DRes fv_complement_impl(double x, double s, bool s_np, double ep, double em) {
  FvExc e = {0, 0, 0.0};
  DRes o;
  double h = py_div(x, s, s_np, e);
  double t = 0.5 * s;
  o.v = ep * fv_norm_cdf(-h - t) + em * fv_norm_cdf(h - t);
  o.code = e.code;
  return o;
}
FV_HD double fv_complement(double x, double s, bool s_np, double ep, double em, FvExc& e) {
  DRes o = fv_complement_impl(x, s, s_np, ep, em);
  if (o.code) e.raise(o.code);
  return o.v;
}

// ---- lbr.py: implied_vol_lbr (:410-486) -----------------------------------
// Split in two so the GPU can run it as a classify pass plus region-uniform
// solve passes (csrc/fv_kernels.cu); fv_lbr_row glues them back together in
// the reference's order for single-row use.
struct FvLbrOut { double sigma; int status; int region; int iterations; };

// Per-quote state handed from classify to solve (anchors computed once).
struct FvLbrState {
  double x, beta, sqrt_t, s_c;   // x = x_work, beta = beta_work, s_c = sqrt(2|x|)
  double b0, b1, E0, E1;         // NEAR_LOW: (b_lo, b_c, E_lo, E_c); NEAR_HIGH: (b_c, b_hi, E_c, E_hi)
};

// normalize_quote + ATM shortcut (:416-430).  Returns 1 when the quote is
// finished (o filled: bounds, ATM, exception), else 0 with st.x / st.beta /
// st.sqrt_t set for fv_lbr_anchors.
FV_HD int fv_lbr_normalize(double th, double Fw, double K, double t, double r, double px,
                           FvLbrState& st, FvLbrOut& o, FvExc& e) {
  const double nan = __builtin_nan("");
  o.sigma = nan; o.status = FV_IV_MAX_ITER; o.region = FV_REGION_NONE; o.iterations = 0;
  // normalize_quote (:174-207); F, K, t, price are numpy scalars
  if (!(Fw > 0.0 && K > 0.0)) { e.raise(FV_EXC_DOM_FK); return 1; }
  double xq = py_log(Fw / K, e);
  double beta0 = px * py_exp(r * t, e) / sqrt(Fw * K);
  double e_hx = py_exp(0.5 * xq, e);
  double e_mhx = py_exp(-0.5 * xq, e);
  if (e.code) return 1;
  double parity = e_hx - e_mhx;
  double beta;
  if (th > 0.0) beta = (xq > 0.0) ? beta0 - parity : beta0;
  else beta = (xq < 0.0) ? beta0 + parity : beta0;
  double x = -fv_fabs(xq);
  double b_max = fv_exp(0.5 * x);
  if (beta <= FV_K_1EM300) { o.status = FV_IV_BELOW_INTRINSIC; return 1; }
  if (beta >= b_max * FV_K_ONE_M_1EM15) { o.status = FV_IV_ABOVE_UPPER; return 1; }
  double sqrt_t = sqrt(t);
  py_exp(-r * t, e);                             // scale = sqrt(F K) exp(-r t): only its overflow
  if (e.code) return 1;

  if (fv_fabs(x) < FV_K_1EM12) {                      // ATM shortcut (:427-430)
    if (!(0.0 < beta && beta < 1.0)) { e.raise_v(FV_EXC_DOM_ATM_BETA, beta, 1); return 1; }
    bool znp;
    double z = fv_inv_norm_cdf(0.5 * (1.0 - beta), true, &znp, e);
    if (e.code) return 1;
    double s = -2.0 * z;
    o.sigma = s / sqrt_t; o.status = FV_IV_CONVERGED;
    return 1;
  }
  st.x = x; st.beta = beta; st.sqrt_t = sqrt_t;
  return 0;
}

// anchors (:231-238) + _region (:241-248), computed once (initial_guess
// recomputes them, :325) and LAZILY: _region compares beta with b_lo, then
// b_c, then b_hi, and each anchor is needed only if the comparison chain
// reaches it.  Skipping the ones it does not reach is bit-neutral because the
// anchors are pure: normalized_black cannot raise for x <= 0 < s (its only
// raising sites are the x / s, t / h, h / rr divisions, none of which can
// divide by zero there, and an exp of a non-positive argument), and nothing
// else in _anchors can raise.  A far-low quote -- the bulk of an OTM chain --
// therefore costs one normalized_black instead of three.
//
// First stage: s_c, b_lo (-> st.b0, st.E0) and the far-low test.  Returns
// FV_FAR_LOW, FV_NEAR_LOW ("the rest of the chain is needed") or -1 if an
// exception was raised.
FV_HD int fv_lbr_anchor_lo(FvLbrState& st, FvExc& e) {
  const double x = st.x;
  st.s_c = py_sqrt(2.0 * fv_fabs(x), e);
  double E_lo = 0.0;
  st.b0 = fv_normalized_black(x, st.s_c * 0.5, false, e, &E_lo, nullptr);
  st.E0 = E_lo;
  if (e.code) return -1;
  return st.beta < st.b0 ? FV_FAR_LOW : FV_NEAR_LOW;
}
// Second stage, for quotes not in the far-low region (st.b0 / st.E0 hold
// b_lo / E_lo): b_c, then b_hi only if beta >= b_c.  Returns the region (or
// -1 on an exception) with the anchor pair the solve needs in b0/b1/E0/E1:
// NEAR_LOW (b_lo, b_c), NEAR_HIGH (b_c, b_hi).
FV_HD int fv_lbr_anchor_rest(FvLbrState& st, FvExc& e) {
  const double x = st.x, beta = st.beta, s_c = st.s_c;
  double E_c = 0.0;
  const double b_c = fv_normalized_black(x, s_c, false, e, &E_c, nullptr);
  if (e.code) return -1;
  if (beta < b_c) { st.b1 = b_c; st.E1 = E_c; return FV_NEAR_LOW; }
  double E_hi = 0.0;
  const double b_hi = fv_normalized_black(x, s_c / 0.5, false, e, &E_hi, nullptr);
  if (e.code) return -1;
  st.b0 = b_c; st.E0 = E_c; st.b1 = b_hi; st.E1 = E_hi;
  return beta < b_hi ? FV_NEAR_HIGH : FV_FAR_HIGH;
}
// Both stages.  Returns 1 if an exception was raised.
FV_HD int fv_lbr_anchors(FvLbrState& st, FvLbrOut& o, FvExc& e) {
  int region = fv_lbr_anchor_lo(st, e);
  if (region == FV_NEAR_LOW) region = fv_lbr_anchor_rest(st, e);
  if (region < 0) return 1;
  o.region = region;
  return 0;
}

FV_HD int fv_lbr_classify(double th, double Fw, double K, double t, double r, double px,
                          FvLbrState& st, FvLbrOut& o, FvExc& e) {
  if (fv_lbr_normalize(th, Fw, K, t, r, px, st, o, e)) return 1;
  return fv_lbr_anchors(st, o, e);
}

// Bracket, initial guess and Householder(3) iterations for one region
// (:434-486).  R is the region (NEAR_LOW stands for both near regions, whose
// code is identical; `region` then picks the anchor pair at run time).
template <int R>
FV_HD FvLbrOut fv_lbr_solve(int region, const FvLbrState& st, FvExc& e) {
  // far-low (the bulk of a chain's OTM quotes) inlines its libm calls
  constexpr bool kInl = (R == FV_FAR_LOW);
  const double nan = __builtin_nan("");
  FvLbrOut o;
  o.sigma = nan; o.status = FV_IV_MAX_ITER; o.region = region; o.iterations = 0;
  const double x = st.x, beta = st.beta, s_c = st.s_c;
  const double s_lo = s_c * 0.5;
  const double s_hi = s_c / 0.5;

  double lo, hi;
  double ep = 0.0, em = 0.0, comp_beta = 0.0, b_max = 0.0;
  if (R == FV_FAR_LOW) { lo = 0.0; hi = s_lo; }
  else if (R == FV_FAR_HIGH) {
    b_max = fv_exp(0.5 * x);                      // quote.b_max, exp(0.5 x)
    ep = b_max;
    comp_beta = b_max - beta;
    lo = s_hi; hi = 2.0 * s_hi;
    em = py_exp(-0.5 * x, e);
    while (fv_complement(x, hi, false, ep, em, e) > comp_beta && hi < 1e6) hi *= 2.0;
    if (e.code) return o;
  } else if (region == FV_NEAR_LOW) { lo = s_lo; hi = s_c; }
  else { lo = s_c; hi = s_hi; }
  lo *= FV_K_ONE_M_1EM6;
  hi *= FV_K_ONE_P_1EM6;
  bool lo_np = false, hi_np = false;

  // initial_guess (:321-332)
  double s;
  bool s_np = false;
  double ln_beta = 0.0;
  if (R == FV_FAR_LOW) {
    // _far_low_guess (:283-309)
    ln_beta = py_log(beta, e);
    double s_cap = s_lo;
    s = py_div(fv_fabs(x), py_sqrt(-2.0 * ln_beta, e), false, e);
    s = py_min(py_max(s, FV_K_1EM6 * s_cap), FV_K_0P999 * s_cap);
    double v = py_log(s, e);
    double v_hi = py_log(s_cap, e);
    for (int it = 0; it < 5; ++it) {
      if (e.code) return o;
      double xs = py_div(x, s, false, e);        // h of normalized_black_log == x / s of :298
      double ln_b = fv_nbl_h<kInl>(xs, s, e);
      double g = ln_b - ln_beta;
      if (g > 0.0) v_hi = py_min(v_hi, v);
      double arg = FV_LOG_INV_SQRT_TWO_PI - 0.5 * (py_powi_t<kInl>(xs, 2, false, e) + 0.25 * s * s) - ln_b;
      double dg_dv = s * py_exp(arg, e);
      if (e.code) return o;
      if (!(fv_isfinite(dg_dv) && dg_dv > 0.0)) break;
      double v_new = v - g / dg_dv;
      if (!fv_isfinite(v_new)) break;
      if (v_new >= v_hi) v_new = 0.5 * (v + v_hi);
      v = v_new;
      s = py_exp(v, e);
    }
  } else if (R == FV_FAR_HIGH) {
    // _far_high_guess (:312-318)
    double p = (b_max - beta) / (2.0 * b_max);    // numpy scalar (beta)
    bool p_np = true;
    if (FV_K_MIN_SUB > p) { p = FV_K_MIN_SUB; p_np = false; }
    if (FV_HALF_ONE_MINUS_EPS < p) { p = FV_HALF_ONE_MINUS_EPS; p_np = false; }
    bool z_np;
    double z = fv_inv_norm_cdf(p, p_np, &z_np, e);
    if (e.code) return o;
    s = -z + py_sqrt(z * z + 2.0 * fv_fabs(x), e);
    s_np = z_np;
  } else {
    // _hermite_inverse (:265-280), all Python floats
    const double b0 = st.b0, b1 = st.b1, E0 = st.E0, E1 = st.E1;
    const double s0 = (region == FV_NEAR_LOW) ? s_lo : s_c;
    const double s1 = (region == FV_NEAR_LOW) ? s_c : s_hi;
    double m0 = py_div(b0, FV_INV_SQRT_TWO_PI * E0, false, e);
    double m1 = py_div(b1, FV_INV_SQRT_TWO_PI * E1, false, e);
    double lb1 = py_log(b1, e);
    double lb0 = py_log(b0, e);
    double du = lb1 - lb0;
    double u = py_div(py_log(beta, e) - lb0, du, false, e);
    if (e.code) return o;
    double u2 = u * u;
    double u3 = u2 * u;
    s = ((2.0 * u3 - 3.0 * u2 + 1.0) * s0 + (u3 - 2.0 * u2 + u) * du * m0
         + (-2.0 * u3 + 3.0 * u2) * s1 + (u3 - u2) * du * m1);
    if (!(py_min(s0, s1) <= s && s <= py_max(s0, s1))) s = s0 + u * (s1 - s0);
  }
  if (!(lo < s && s < hi)) { s = 0.5 * (lo + hi); s_np = false; }

  // Householder(3) iterations (:454-483)
  const bool increasing = R != FV_FAR_LOW;
  double ln_comp_beta = 0.0;
  bool comp_beta_bad = false;
  if (R == FV_FAR_HIGH) {
    FvExc tmp = {0, 0, 0.0};
    ln_comp_beta = py_log(comp_beta, tmp);
    comp_beta_bad = tmp.code != 0;
  }
  const double inv_ln_beta = (R == FV_FAR_LOW) ? 1.0 / ln_beta : 0.0;
  int iterations = 0;
  bool converged = false;
  for (int it = 0; it < 8; ++it) {
    // objective_branch (:346-389)
    if (!(s > 0.0)) { e.raise_v(FV_EXC_DOM_OBJ_S, s, s_np); return o; }
    double h = py_div(x, s, s_np, e);
    double t = 0.5 * s;
    double s3 = s * s * s;
    double r2 = py_div(x * x, s3, s_np, e) - 0.25 * s;
    double s4 = py_powi_t<kInl>(s, 4, s_np, e);
    double r3 = r2 * r2 - py_div(3.0 * x * x, s4, s_np, e) - 0.25;
    double g, g1, g2, g3;
    bool g_np, g1_np, g23_np;
    if (R == FV_FAR_LOW) {
      double ln_b = fv_nbl_h<kInl>(h, s, e);      // its h = x / s is the h above
      double ln_bp = FV_LOG_INV_SQRT_TWO_PI - 0.5 * (h * h + 0.25 * s * s);
      double up = py_exp(ln_bp - ln_b, e);
      double up3 = py_powi_t<kInl>(up, 3, false, e);
      double upp = up * r2 - up * up;
      double uppp = up * r3 - 3.0 * up * up * r2 + 2.0 * up3;
      double inv = py_div(1.0, ln_b, false, e);
      double inv2 = inv * inv;
      if (ln_beta == 0.0) e.raise(FV_EXC_ZERO_DIV);
      g = inv - inv_ln_beta;                      // 1.0 / ln_beta, loop-invariant
      g1 = -up * inv2;
      g2 = -upp * inv2 + 2.0 * up * up * inv2 * inv;
      g3 = (-uppp * inv2 + 6.0 * up * upp * inv2 * inv - 6.0 * up3 * inv2 * inv2);
      g_np = false; g1_np = false; g23_np = s_np;
    } else if (R == FV_FAR_HIGH) {
      double bp = FV_INV_SQRT_TWO_PI * fv_exp(-0.5 * (h * h + t * t));
      double comp = ep * fv_norm_cdf(-h - t) + em * fv_norm_cdf(h - t);
      double w = py_div(bp, comp, false, e);
      if (comp_beta_bad) e.raise(FV_EXC_MATH_DOMAIN);
      double lcomp = py_log(comp, e);
      double w3 = py_powi(w, 3, false, e);
      g = ln_comp_beta - lcomp;
      g1 = w;
      g2 = w * r2 + w * w;
      g3 = w * r3 + 3.0 * w * w * r2 + 2.0 * w3;
      g_np = false; g1_np = false; g23_np = s_np;
    } else {
      double Ev = 0.0;
      double b = fv_normalized_black(x, s, s_np, e, &Ev, nullptr);
      double bp = FV_INV_SQRT_TWO_PI * Ev;
      g = b - beta; g1 = bp; g2 = bp * r2; g3 = bp * r3;
      g_np = true; g1_np = false; g23_np = s_np;
    }
    if (e.code) return o;
    if (g == 0.0) { converged = true; break; }
    bool below = increasing ? (g < 0.0) : (g > 0.0);
    if (below) { if (s > lo) { lo = s; lo_np = s_np; } }
    else { if (s < hi) { hi = s; hi_np = s_np; } }
    // householder3_step (:392-402)
    double ds;
    bool ds_np;
    if (g1 == 0.0 || !fv_isfinite(g1)) { ds = nan; ds_np = false; }
    else {
      double nu = -g / g1;
      double eta = g2 / g1;
      double gam = py_div(g3, 6.0 * g1, g23_np || g1_np, e);
      bool num_np = g_np || g1_np || g23_np;
      ds = py_div(nu * (1.0 + 0.5 * nu * eta), 1.0 + nu * (eta + nu * gam), num_np, e);
      ds_np = num_np;
      if (e.code) return o;
    }
    if (fv_isfinite(ds) && fv_fabs(ds) <= FV_K_1EM14 * py_max(1.0, s)) {
      s = s + ds; s_np = s_np || ds_np;
      iterations += 1;
      converged = true;
      break;
    }
    double cand = s + ds;
    bool cand_np = s_np || ds_np;
    if (!fv_isfinite(cand) || !(lo < cand && cand < hi)) {
      cand = 0.5 * (lo + hi);
      cand_np = lo_np || hi_np;
      ds = cand - s;
    }
    s = cand; s_np = cand_np;
    iterations += 1;
    if (fv_fabs(ds) <= FV_K_1EM14 * py_max(1.0, s)) { converged = true; break; }
  }
  o.sigma = s / st.sqrt_t;
  o.status = converged ? FV_IV_CONVERGED : FV_IV_MAX_ITER;
  o.iterations = iterations;
  return o;
}

// Far-low region (:434-486 with _far_low_guess :283-309 and the 1/ln b
// objective :362-377), restructured for the GPU's instruction cache: the five
// safeguarded Newton steps of the guess and the <= 8 Householder(3) steps run
// as ONE step loop, so each heavy routine (normalized_black_log, pow, exp) has
// a single inlined call site and the loop body stays a few KB.  Every value is
// computed by the same expression as in the reference; where the two phases
// check exceptions in different orders, each check keeps its own record and
// they are merged in the reference's order.  Bit-identical to
// fv_lbr_solve<FV_FAR_LOW> (tests/test_quote_host.py checks both).
FV_HD FvLbrOut fv_lbr_far_low_fused(const FvLbrState& st, FvExc& e) {
  const double nan = __builtin_nan("");
  FvLbrOut o;
  o.sigma = nan; o.status = FV_IV_MAX_ITER; o.region = FV_FAR_LOW; o.iterations = 0;
  const double x = st.x, beta = st.beta;
  const double s_lo = st.s_c * 0.5;
  double lo = 0.0, hi = s_lo;
  lo *= FV_K_ONE_M_1EM6;
  hi *= FV_K_ONE_P_1EM6;
  // _far_low_guess prologue (:286-291)
  const double ln_beta = py_log_t<true>(beta, e);
  const double s_cap = s_lo;
  double s = py_div(fv_fabs(x), py_sqrt(-2.0 * ln_beta, e), false, e);
  s = py_min(py_max(s, FV_K_1EM6 * s_cap), FV_K_0P999 * s_cap);
  double v = py_log_t<true>(s, e);
  double v_hi = py_log_t<true>(s_cap, e);
  if (e.code) return o;
  const double xx = x * x;
  const double x3 = 3.0 * x * x;
  const double inv_ln_beta = 1.0 / ln_beta;
  int nk = 0;                 // Newton steps taken
  bool newton = true;
  int iterations = 0;
  bool converged = false;
  for (int step = 0; step < 13; ++step) {
    if (!newton) {
      if (iterations == 8) break;
      if (!(s > 0.0)) { e.raise_v(FV_EXC_DOM_OBJ_S, s, 0); return o; }     // :358-359
    }
    FvExc e_h = {0, 0, 0.0}, e_r = {0, 0, 0.0}, e_nb = {0, 0, 0.0}, e_pw = {0, 0, 0.0};
    const double h = py_div(x, s, false, e_h);                 // x / s (:144 / :298 / :154)
    double r2 = 0.0, r3 = 0.0;
    if (!newton) r2 = py_div(xx, s * s * s, false, e_r) - 0.25 * s;   // :341
    // pow site: (x/s)**2 (:298) or s**4 (:342)
    const double pw = py_powi_t<true>(newton ? h : s, newton ? 2 : 4, false, e_pw);
    if (!newton) r3 = r2 * r2 - py_div(x3, pw, false, e_pw) - 0.25;  // :342
    const double ln_b = fv_nbl_h<true>(h, s, e_nb);            // normalized_black_log(x, s)
    // reference order: Newton = nbl, (x/s)**2 ; iteration = x/s, ratios, nbl
    e.raise(e_h.code);
    if (newton) { e.raise(e_nb.code); e.raise(e_pw.code); }
    else { e.raise(e_r.code); e.raise(e_pw.code); e.raise(e_nb.code); }
    if (e.code) return o;
    // exp site: dg_dv's exponent (:297-299) or b'/b (:366-367)
    const double q = newton ? pw : h * h;
    const double ex = py_exp(FV_LOG_INV_SQRT_TWO_PI - 0.5 * (q + 0.25 * s * s) - ln_b, e);
    if (e.code) return o;
    if (newton) {
      // rest of the Newton step (:293-308)
      const double g = ln_b - ln_beta;
      if (g > 0.0) v_hi = py_min(v_hi, v);
      const double dg_dv = s * ex;
      bool stop = !(fv_isfinite(dg_dv) && dg_dv > 0.0);
      if (!stop) {
        double v_new = v - g / dg_dv;
        if (!fv_isfinite(v_new)) stop = true;
        else {
          if (v_new >= v_hi) v_new = 0.5 * (v + v_hi);
          v = v_new;
          s = py_exp(v, e);
          if (e.code) return o;
        }
      }
      if (stop || ++nk == 5) {
        newton = false;                                         // initial_guess done
        if (!(lo < s && s < hi)) s = 0.5 * (lo + hi);           // :451-452
      }
      continue;
    }
    // Householder(3) step on the far-low objective (:363-377, :457-483)
    const double up = ex;
    const double up3 = py_powi_t<true>(up, 3, false, e);
    const double upp = up * r2 - up * up;
    const double uppp = up * r3 - 3.0 * up * up * r2 + 2.0 * up3;
    const double inv = py_div(1.0, ln_b, false, e);
    const double inv2 = inv * inv;
    if (ln_beta == 0.0) e.raise(FV_EXC_ZERO_DIV);
    const double g = inv - inv_ln_beta;
    const double g1 = -up * inv2;
    const double g2 = -upp * inv2 + 2.0 * up * up * inv2 * inv;
    const double g3 = (-uppp * inv2 + 6.0 * up * upp * inv2 * inv - 6.0 * up3 * inv2 * inv2);
    if (e.code) return o;
    if (g == 0.0) { converged = true; break; }
    if (g > 0.0) { if (s > lo) lo = s; }                        // decreasing objective
    else { if (s < hi) hi = s; }
    double ds;
    if (g1 == 0.0 || !fv_isfinite(g1)) ds = nan;
    else {
      const double nu = -g / g1;
      const double eta = g2 / g1;
      const double gam = py_div(g3, 6.0 * g1, false, e);
      ds = py_div(nu * (1.0 + 0.5 * nu * eta), 1.0 + nu * (eta + nu * gam), false, e);
      if (e.code) return o;
    }
    if (fv_isfinite(ds) && fv_fabs(ds) <= FV_K_1EM14 * py_max(1.0, s)) {
      s = s + ds;
      iterations += 1;
      converged = true;
      break;
    }
    double cand = s + ds;
    if (!fv_isfinite(cand) || !(lo < cand && cand < hi)) {
      cand = 0.5 * (lo + hi);
      ds = cand - s;
    }
    s = cand;
    iterations += 1;
    if (fv_fabs(ds) <= FV_K_1EM14 * py_max(1.0, s)) { converged = true; break; }
  }
  o.sigma = s / st.sqrt_t;
  o.status = converged ? FV_IV_CONVERGED : FV_IV_MAX_ITER;
  o.iterations = iterations;
  return o;
}

FV_HD FvLbrOut fv_lbr_row(double th, double Fw, double K, double t, double r, double px, FvExc& e) {
  FvLbrState st;
  FvLbrOut o;
  if (fv_lbr_classify(th, Fw, K, t, r, px, st, o, e)) return o;
  if (o.region == FV_FAR_LOW) return fv_lbr_far_low_fused(st, e);
  if (o.region == FV_FAR_HIGH) return fv_lbr_solve<FV_FAR_HIGH>(o.region, st, e);
  return fv_lbr_solve<FV_NEAR_LOW>(o.region, st, e);
}

// batch_iv LBR row (batch.py:227-238): spot models forward the underlying.
FV_HD FvLbrOut fv_lbr_batch_row(int model, double th, double un, double K, double t, double r,
                                double q, double px, FvExc& e) {
  FvLbrOut o;
  o.sigma = __builtin_nan(""); o.status = FV_IV_MAX_ITER; o.region = FV_REGION_NONE; o.iterations = 0;
  double Fw = un;
  if (model != 0) {
    Fw = un * py_exp((r - q) * t, e);
    if (e.code) return o;
  }
  if (!(t > 0.0)) { o.status = FV_IV_BELOW_INTRINSIC; return o; }
  o = fv_lbr_row(th, Fw, K, t, r, px, e);
  if (o.status != FV_IV_CONVERGED && o.status != FV_IV_FELL_BACK) o.sigma = __builtin_nan("");
  return o;
}
