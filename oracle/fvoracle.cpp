// oracle/fvoracle.cpp -- TEST INFRASTRUCTURE ONLY (never shipped, never on the
// product path).  A CPU restatement of the reference's batched pricing /
// Greeks / implied-vol path (fastvol 0.1.0, /root/reference/pkg/src/fastvol),
// statement for statement, used as the parity checker for the CUDA kernels and
// as the CPU baseline timed by bench.py.
//
// What makes it faithful:
//   * the scalar math is the REAL third-party code the reference calls:
//     glibc libm exp/log/erfc/pow/sqrt (what CPython's math module and
//     float.__pow__ call) and scipy's own compiled erfcx (function pointer from
//     scipy.special.cython_special, installed by oracle/fvoracle.py);
//   * every value carries the Python type that the reference's value has at
//     that point (Python float vs numpy.float64 scalar -- batch.py passes
//     numpy scalars into the scalar solvers, batch.py:229-234), because the two
//     differ in exception behaviour: float/0.0 raises ZeroDivisionError and
//     float**n overflow raises OverflowError, numpy scalars return inf/nan;
//   * math.exp/log/sqrt raise exactly as CPython 3.12 does (math_1, m_log);
//   * Python max()/min() keep the first argument unless the second compares
//     strictly greater/smaller (NaN and -0.0 behaviour), and return the chosen
//     OBJECT (type included);
//   * no FMA contraction (-ffp-contract=off): CPython evaluates a*b+c as two
//     rounded operations.
// Pinned against the live reference by tests/golden/ (gen_golden.py) and
// tests/test_oracle_golden.py.
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

namespace orc {

// ---------------------------------------------------------------------------
// Exceptions (first raised wins; Python stops at the first raise)
// ---------------------------------------------------------------------------
enum Exc : int {
  EXC_NONE = 0,
  EXC_MATH_RANGE = 1,      // OverflowError('math range error')           (math.exp)
  EXC_MATH_DOMAIN = 2,     // ValueError('math domain error')             (math.log / math.sqrt)
  EXC_ZERO_DIV = 3,        // ZeroDivisionError('float division by zero')
  EXC_POW_RANGE = 4,       // OverflowError((34, 'Numerical result out of range'))  (float.__pow__)
  EXC_DOM_FK = 5,          // DomainError('F and K must be positive')     lbr.py:183-184
  EXC_DOM_ATM_BETA = 6,    // DomainError(f'atm_inverse requires beta in (0, 1), got {beta!r}')  lbr.py:260-261
  EXC_DOM_INVCDF_P = 7,    // DomainError(f'inv_norm_cdf requires p in (0, 1), got {p!r}')       distributions.py:85-86
  EXC_DOM_NB_X = 8,        // DomainError(f'normalized_black requires x <= 0, got {x!r}')        lbr.py:114-115
  EXC_DOM_NB_S = 9,        // DomainError(f'normalized_black requires s > 0, got {s!r}')         lbr.py:116-117
  EXC_DOM_OBJ_S = 10,      // DomainError(f'objective_branch requires s > 0, got {s!r}')         lbr.py:358-359
};

struct State {
  int exc = EXC_NONE;
  double exc_val = 0.0;
  int exc_np = 0;
};
static thread_local State S;

// Optional value trace for debugging parity (tests only): TRACE(v) appends.
static thread_local double* g_trace = nullptr;
static thread_local int g_trace_n = 0;
#define TRACE(v) do { if (g_trace && g_trace_n < 256) g_trace[g_trace_n++] = (v); } while (0)

static inline void raise(int code, double val = 0.0, int np = 0) {
  if (S.exc == EXC_NONE) { S.exc = code; S.exc_val = val; S.exc_np = np; }
}
#define RAISED (S.exc != EXC_NONE)

// ---------------------------------------------------------------------------
// Py: a Python float or numpy.float64 scalar
// ---------------------------------------------------------------------------
struct Py {
  double v;
  bool np;
};
static inline Py F(double v) { return Py{v, false}; }   // Python float / int literal
static inline Py N(double v) { return Py{v, true}; }    // numpy.float64
static inline Py operator+(Py a, Py b) { return Py{a.v + b.v, a.np || b.np}; }
static inline Py operator-(Py a, Py b) { return Py{a.v - b.v, a.np || b.np}; }
static inline Py operator*(Py a, Py b) { return Py{a.v * b.v, a.np || b.np}; }
static inline Py operator-(Py a) { return Py{-a.v, a.np}; }
static inline Py operator/(Py a, Py b) {
  if (!a.np && !b.np && b.v == 0.0) raise(EXC_ZERO_DIV);
  return Py{a.v / b.v, a.np || b.np};
}
static inline Py operator+(Py a, double b) { return a + F(b); }
static inline Py operator+(double a, Py b) { return F(a) + b; }
static inline Py operator-(Py a, double b) { return a - F(b); }
static inline Py operator-(double a, Py b) { return F(a) - b; }
static inline Py operator*(Py a, double b) { return a * F(b); }
static inline Py operator*(double a, Py b) { return F(a) * b; }
static inline Py operator/(Py a, double b) { return a / F(b); }
static inline Py operator/(double a, Py b) { return F(a) / b; }
static inline bool operator<(Py a, Py b) { return a.v < b.v; }
static inline bool operator>(Py a, Py b) { return a.v > b.v; }
static inline bool operator<=(Py a, Py b) { return a.v <= b.v; }
static inline bool operator>=(Py a, Py b) { return a.v >= b.v; }
static inline bool operator<(Py a, double b) { return a.v < b; }
static inline bool operator>(Py a, double b) { return a.v > b; }
static inline bool operator<=(Py a, double b) { return a.v <= b; }
static inline bool operator>=(Py a, double b) { return a.v >= b; }
static inline bool operator==(Py a, double b) { return a.v == b; }
static inline bool operator!=(Py a, double b) { return a.v != b; }
static inline bool operator<(double a, Py b) { return a < b.v; }
static inline Py py_abs(Py a) { return Py{fabs(a.v), a.np}; }
// builtins max/min (bltinmodule.c min_max): keep the first item unless the
// next compares strictly greater (max) / smaller (min).
static inline Py py_max(Py a, Py b) { return (b.v > a.v) ? b : a; }
static inline Py py_min(Py a, Py b) { return (b.v < a.v) ? b : a; }
static inline bool isfin(Py a) { return isfinite(a.v); }

// math module (CPython 3.12 Modules/mathmodule.c)
static inline Py m_exp(Py x) {      // math_1(x, exp, can_overflow=1)
  double r = exp(x.v);
  if (isinf(r) && isfinite(x.v)) raise(EXC_MATH_RANGE);
  return F(r);
}
static inline Py m_log(Py x) {      // m_log + loghelper
  double v = x.v;
  if (isfinite(v)) {
    if (v > 0.0) return F(log(v));
    raise(EXC_MATH_DOMAIN);
    return F(v == 0.0 ? -INFINITY : NAN);
  }
  if (isnan(v)) return F(v);
  if (v > 0.0) return F(v);
  raise(EXC_MATH_DOMAIN);
  return F(NAN);
}
static inline Py m_sqrt(Py x) {     // math_1(x, sqrt, can_overflow=0)
  double r = sqrt(x.v);
  if (isnan(r) && !isnan(x.v)) raise(EXC_MATH_DOMAIN);
  return F(r);
}
static inline Py m_erfc(Py x) { return F(erfc(x.v)); }   // never raises
// x ** n for a small positive integer n: float_pow (Objects/floatobject.c)
// for Python floats, npy_pow for numpy scalars.
static inline Py py_pow(Py x, int n) {
  double r = pow(x.v, (double)n);
  if (!x.np && isfinite(x.v) && isinf(r)) raise(EXC_POW_RANGE);
  return Py{r, x.np};
}

// scipy.special.erfcx via scipy.special.cython_special (__pyx_fuse_1erfcx)
typedef double (*erfcx_fn)(double, int);
static erfcx_fn g_erfcx = nullptr;
static double g_asym_facts[18];
static double g_asym_pascal[18][18];

static const double SQRT_TWO = 1.4142135623730951;          // distributions.py:14 (math.sqrt(2.0))
static double INV_SQRT_TWO_PI;                               // distributions.py:16
static double SMALL_T_THRESHOLD;                             // lbr.py:40
static const double DBL_EPS = 2.220446049250313e-16;        // lbr.py:37
static const double ASYMPTOTIC_H_THRESHOLD = -10.0;          // lbr.py:42
static const double ATM_X_CUTOFF = 1e-12;                    // lbr.py:43
static const double REGION_RATIO = 0.5;                      // lbr.py:44
static const double STEP_TOLERANCE = 1e-14;                  // lbr.py:45
static const double VOL_TIME_CUTOFF = 1e-12;                 // pricing.py:20

static void init_constants() {
  double sqrt_two_pi = sqrt(2.0 * M_PI);                     // distributions.py:15
  INV_SQRT_TWO_PI = 1.0 / sqrt_two_pi;
  SMALL_T_THRESHOLD = 2.0 * pow(DBL_EPS, 0.0625);            // lbr.py:40
}

// ---------------------------------------------------------------------------
// distributions.py
// ---------------------------------------------------------------------------
static Py norm_cdf(Py x) { return 0.5 * m_erfc(-x / SQRT_TWO); }                 // :19-21
static Py norm_pdf(Py x) { return INV_SQRT_TWO_PI * m_exp(-0.5 * x * x); }       // :24-26

static const double AS_A[8] = {3.3871328727963666080e0, 1.3314166789178437745e2,
    1.9715909503065514427e3, 1.3731693765509461125e4, 4.5921953931549871457e4,
    6.7265770927008700853e4, 3.3430575583588128105e4, 2.5090809287301226727e3};
static const double AS_B[8] = {1.0, 4.2313330701600911252e1, 6.8718700749205790830e2,
    5.3941960214247511077e3, 2.1213794301586595867e4, 3.9307895800092710610e4,
    2.8729085735721942674e4, 5.2264952788528545610e3};
static const double AS_C[8] = {1.42343711074968357734e0, 4.63033784615654529590e0,
    5.76949722146069140550e0, 3.64784832476320460504e0, 1.27045825245236838258e0,
    2.41780725177450611770e-1, 2.27238449892691845833e-2, 7.74545014278341407640e-4};
static const double AS_D[8] = {1.0, 2.05319162663775882187e0, 1.67638483018380384940e0,
    6.89767334985100004550e-1, 1.48103976427480074590e-1, 1.51986665636164571966e-2,
    5.47593808499534494600e-4, 1.05075007164441684324e-9};
static const double AS_E[8] = {6.65790464350110377720e0, 5.46378491116411436990e0,
    1.78482653991729133580e0, 2.96560571828504891230e-1, 2.65321895265761230930e-2,
    1.24266094738807843860e-3, 2.71155556874348757815e-5, 2.01033439929228813265e-7};
static const double AS_F[8] = {1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1,
    1.48753612908506148525e-2, 7.86869131145613259100e-4, 1.84631831751005468180e-5,
    1.42151175831644588870e-7, 2.04426310338993978564e-15};

static Py poly(const double* c, Py r) {                      // :56-60
  Py acc = F(0.0);
  for (int i = 7; i >= 0; --i) acc = acc * r + c[i];
  return acc;
}

static Py ppnd16(Py p) {                                     // :63-76
  Py q = p - 0.5;
  if (py_abs(q) <= 0.425) {
    Py r = 0.180625 - q * q;
    return q * poly(AS_A, r) / poly(AS_B, r);
  }
  Py r = (q < 0.0) ? p : (1.0 - p);
  r = m_sqrt(-m_log(r));
  Py val;
  if (r <= 5.0) {
    r = r - 1.6;
    val = poly(AS_C, r) / poly(AS_D, r);
  } else {
    r = r - 5.0;
    val = poly(AS_E, r) / poly(AS_F, r);
  }
  return (q < 0.0) ? -val : val;
}

static Py inv_norm_cdf(Py p) {                               // :79-95
  if (!(0.0 < p.v && p.v < 1.0)) { raise(EXC_DOM_INVCDF_P, p.v, p.np); return F(NAN); }
  Py x = ppnd16(p);
  Py pdf = norm_pdf(x);
  if (pdf > 0.0) {
    Py err = norm_cdf(x) - p;
    Py u = err / pdf;
    x = x - u / (1.0 + 0.5 * x * u);
  }
  return x;
}

// ---------------------------------------------------------------------------
// pricing.py
// ---------------------------------------------------------------------------
static Py black_kernel(int theta, Py Fw, Py K, Py discount, Py s) {   // :23-33
  Py th = F((double)theta);
  Py intrinsic = py_max(th * (Fw - K), F(0.0));
  Py cap = (theta > 0) ? Fw : K;
  if (s < VOL_TIME_CUTOFF) return discount * intrinsic;
  Py d1 = (m_log(Fw / K) + 0.5 * s * s) / s;
  Py d2 = d1 - s;
  Py raw = th * (Fw * norm_cdf(th * d1) - K * norm_cdf(th * d2));
  return discount * py_min(py_max(raw, intrinsic), cap);
}

static Py price_black76(int theta, Py Fw, Py K, Py t, Py r, Py sigma) {   // :49-53 (_check pre-validated)
  Py disc = m_exp(-r * t);
  Py s = sigma * m_sqrt(t);
  return black_kernel(theta, Fw, K, disc, s);
}

static Py price_bsm(int theta, Py Sp, Py K, Py t, Py r, Py q, Py sigma) {   // :56-61
  Py Fw = Sp * m_exp((r - q) * t);
  Py disc = m_exp(-r * t);
  Py s = sigma * m_sqrt(t);
  return black_kernel(theta, Fw, K, disc, s);
}

// ---------------------------------------------------------------------------
// greeks.py _core (:45-98); returns 0 = ok, 1 = StepFunctionEdge
// ---------------------------------------------------------------------------
static int greeks_core(int theta, bool forward_model, Py under_in, Py K, Py t, Py r, Py q,
                       Py sigma, double out[5]) {
  Py th = F((double)theta);
  Py sqrt_t = m_sqrt(t);
  Py s = sigma * sqrt_t;
  Py disc = m_exp(-r * t);
  if (RAISED) return 0;
  if (s < VOL_TIME_CUTOFF) return 1;
  Py Fw, carry_disc, under;
  if (forward_model) {
    Fw = under_in; carry_disc = disc; under = Fw;
  } else {
    Py Sp = under_in;
    Fw = Sp * m_exp((r - q) * t);
    carry_disc = m_exp(-q * t);
    under = Sp;
  }
  Py d1 = (m_log(Fw / K) + 0.5 * s * s) / s;
  if (RAISED) return 0;
  Py d2 = d1 - s;
  Py cdf_td1 = norm_cdf(th * d1);
  Py cdf_td2 = norm_cdf(th * d2);
  Py pdf_d1 = norm_pdf(d1);
  Py delta = th * carry_disc * cdf_td1;
  Py gamma = carry_disc * pdf_d1 / (under * s);
  Py vega = carry_disc * under * pdf_d1 * sqrt_t;
  Py theta_cal, rho;
  if (forward_model) {
    Py value = disc * th * (Fw * cdf_td1 - K * cdf_td2);
    theta_cal = r * value - disc * Fw * pdf_d1 * sigma / (2.0 * sqrt_t);
    rho = -t * value;
  } else {
    theta_cal = (-under * carry_disc * pdf_d1 * sigma / (2.0 * sqrt_t)
                 - th * (r * K * disc * cdf_td2 - q * under * carry_disc * cdf_td1));
    rho = th * K * t * disc * cdf_td2;
  }
  theta_cal = theta_cal / 365.0;
  rho = rho / 100.0;
  vega = vega / 100.0;
  out[0] = delta.v; out[1] = gamma.v; out[2] = theta_cal.v; out[3] = rho.v; out[4] = vega.v;
  return 0;
}

// ---------------------------------------------------------------------------
// solver.py: statuses and Halley+bisection (:49-161)
// ---------------------------------------------------------------------------
enum Status : int { CONVERGED = 0, FELL_BACK = 1, BELOW_INTRINSIC = 2, ABOVE_UPPER = 3, MAX_ITER = 4 };
struct Result { Py sigma; int iterations; int status; };

static Py raw_vega(Py Fw, Py K, Py t, Py discount, Py sigma) {   // :40-46
  Py s = sigma * m_sqrt(t);
  if (s < VOL_TIME_CUTOFF) return F(0.0);
  Py d1 = (m_log(Fw / K) + 0.5 * s * s) / s;
  return discount * Fw * norm_pdf(d1) * m_sqrt(t);
}

static Result implied_vol_halley(Py target, int theta, bool b76, Py under, Py K, Py t, Py r, Py q) {
  const Py nan = F(NAN);
  const double SIGMA_LO = 1e-9, SIGMA_HI = 10.0, SIGMA_HI_CAP = 100.0;   // :35-37
  const double tol_sigma = 1e-12;
  const int max_halley = 16, max_bisect = 128;
  Py Fw = b76 ? under : under * m_exp((r - q) * t);
  Py discount = m_exp(-r * t);
  Py sqrt_t = m_sqrt(t);
  if (RAISED) return Result{nan, 0, MAX_ITER};
  Py th = F((double)theta);
  Py disc_intrinsic = discount * py_max(th * (Fw - K), F(0.0));
  Py disc_cap = discount * ((theta > 0) ? Fw : K);
  Py tie_tol = 1e-12 * py_max(F(1.0), disc_cap);
  if (!isfin(target)) return Result{nan, 0, BELOW_INTRINSIC};
  if (target <= disc_intrinsic + tie_tol) return Result{nan, 0, BELOW_INTRINSIC};
  if (target > disc_cap + tie_tol) return Result{nan, 0, ABOVE_UPPER};
  Py tol_price = py_min(tie_tol, 1e-10 * (target - disc_intrinsic));
  if (t <= 0.0) return Result{nan, 0, ABOVE_UPPER};

  auto f = [&](Py sigma) -> Py {
    return black_kernel(theta, Fw, K, discount, sigma * sqrt_t) - target;
  };
  Py lo = F(SIGMA_LO), hi = F(SIGMA_HI);
  Py f_lo = f(lo);
  if (RAISED) return Result{nan, 0, MAX_ITER};
  if (f_lo >= 0.0) {
    if (py_abs(f_lo) <= tol_price) return Result{lo, 0, CONVERGED};
    return Result{nan, 0, BELOW_INTRINSIC};
  }
  Py f_hi = f(hi);
  while (f_hi < 0.0 && hi < SIGMA_HI_CAP) {
    hi = py_min(2.0 * hi, F(SIGMA_HI_CAP));
    f_hi = f(hi);
  }
  if (f_hi < 0.0) return Result{nan, 0, MAX_ITER};
  Py sigma = m_sqrt(2.0 * M_PI / t) * target / under;
  sigma = py_min(py_max(sigma, F(0.05)), F(2.0));
  sigma = py_min(py_max(sigma, lo), hi);
  Py fval = f(sigma);
  if (RAISED) return Result{nan, 0, MAX_ITER};
  if (fval > 0.0) hi = py_min(hi, sigma);
  else if (fval < 0.0) lo = py_max(lo, sigma);
  int iterations = 0;
  for (int it = 0; it < max_halley; ++it) {
    if (py_abs(fval) <= tol_price) return Result{sigma, iterations, CONVERGED};
    Py vega = raw_vega(Fw, K, t, discount, sigma);
    if (RAISED) return Result{nan, 0, MAX_ITER};
    Py cand = nan;
    if (vega > 0.0) {
      Py s = sigma * sqrt_t;
      Py d1 = (m_log(Fw / K) + 0.5 * s * s) / s;
      Py d2 = d1 - s;
      Py vomma = vega * d1 * d2 / sigma;
      Py denom = 2.0 * vega * vega - fval * vomma;
      if (denom != 0.0) cand = sigma - 2.0 * fval * vega / denom;
      if (RAISED) return Result{nan, 0, MAX_ITER};
    }
    bool accepted = false;
    Py f_cand = F(0.0);
    if (isfin(cand) && lo < cand && cand < hi) {
      f_cand = f(cand);
      if (py_abs(f_cand) < py_abs(fval)) accepted = true;
    }
    if (!accepted) {
      cand = 0.5 * (lo + hi);
      f_cand = f(cand);
    }
    if (RAISED) return Result{nan, 0, MAX_ITER};
    if (f_cand > 0.0) hi = cand;
    else if (f_cand < 0.0) lo = cand;
    Py step = cand - sigma;
    sigma = cand; fval = f_cand;
    iterations += 1;
    if (py_abs(step) <= tol_sigma * py_max(F(1.0), sigma))
      return Result{sigma, iterations, CONVERGED};
  }
  for (int it = 0; it < max_bisect; ++it) {
    if (py_abs(fval) <= tol_price || (hi - lo) <= tol_sigma * py_max(F(1.0), sigma))
      return Result{sigma, iterations, FELL_BACK};
    sigma = 0.5 * (lo + hi);
    fval = f(sigma);
    if (RAISED) return Result{nan, 0, MAX_ITER};
    if (fval > 0.0) hi = sigma;
    else lo = sigma;
    iterations += 1;
  }
  if (py_abs(fval) <= tol_price || (hi - lo) <= tol_sigma * py_max(F(1.0), sigma))
    return Result{sigma, iterations, FELL_BACK};
  return Result{nan, iterations, MAX_ITER};
}

// ---------------------------------------------------------------------------
// lbr.py
// ---------------------------------------------------------------------------
static Py erfcx_(Py z) { return F(g_erfcx(z.v, 0)); }     // :48-49

static Py asymptotic_black(Py h, Py t) {                   // :65-71
  Py e = (t / h) * (t / h);
  Py r = (h + t) * (h - t);
  Py q = (h / r) * (h / r);
  // polyval(e, _ASYM_PASCAL): column-wise Horner, c0 = c[-1] + x*0
  double inner[18];
  for (int j = 0; j < 18; ++j) {
    Py c0 = F(g_asym_pascal[17][j]) + e * 0.0;
    for (int i = 16; i >= 0; --i) c0 = F(g_asym_pascal[i][j]) + c0 * e;
    inner[j] = c0.v;
  }
  Py c0 = F(g_asym_facts[17] * inner[17]) + q * 0.0;
  for (int i = 16; i >= 0; --i) c0 = F(g_asym_facts[i] * inner[i]) + c0 * q;
  Py total = F(c0.v);
  Py b = INV_SQRT_TWO_PI * m_exp(-0.5 * (h * h + t * t)) * (t / r) * total;
  return py_max(b, F(0.0));
}

static Py small_t_black(Py h, Py t) {                      // :74-103
  Py a = 1.0 + h * (0.5 * sqrt(2.0 * M_PI)) * erfcx_(-h / SQRT_TWO);
  Py w = t * t;
  Py h2 = h * h;
  Py c1 = (-1.0 + 3.0 * a + a * h2) / 6.0;
  Py c2 = (-7.0 + 15.0 * a + h2 * (-1.0 + 10.0 * a + a * h2)) / 120.0;
  Py c3 = (-57.0 + 105.0 * a + h2 * (-18.0 + 105.0 * a + h2 * (-1.0 + 21.0 * a + a * h2))) / 5040.0;
  Py c4 = (-561.0 + 945.0 * a
           + h2 * (-285.0 + 1260.0 * a
                   + h2 * (-33.0 + 378.0 * a
                           + h2 * (-1.0 + 36.0 * a + a * h2)))) / 362880.0;
  Py c5 = (-6555.0 + 10395.0 * a
           + h2 * (-4680.0 + 17325.0 * a
                   + h2 * (-840.0 + 6930.0 * a
                           + h2 * (-52.0 + 990.0 * a
                                   + h2 * (-1.0 + 55.0 * a + a * h2))))) / 39916800.0;
  Py c6 = (-89055.0 + 135135.0 * a
           + h2 * (-82845.0 + 270270.0 * a
                   + h2 * (-20370.0 + 135135.0 * a
                           + h2 * (-1926.0 + 25740.0 * a
                                   + h2 * (-75.0 + 2145.0 * a
                                           + h2 * (-1.0 + 78.0 * a + a * h2)))))) / 6227020800.0;
  Py expansion = 2.0 * t * (a + w * (c1 + w * (c2 + w * (c3 + w * (c4 + w * (c5 + w * c6))))));
  Py b = INV_SQRT_TWO_PI * m_exp(-0.5 * (h * h + t * t)) * expansion;
  return py_max(b, F(0.0));
}

static Py erfcx_black(Py h, Py t) {                        // :106-109
  Py b = 0.5 * m_exp(-0.5 * (h * h + t * t)) *
         (erfcx_(-(h + t) / SQRT_TWO) - erfcx_(-(h - t) / SQRT_TWO));
  return py_max(b, F(0.0));
}

// branch code for tests: 0 asymptotic, 1 small-t, 2 direct, 3 erfcx
static Py normalized_black(Py x, Py s, int* branch = nullptr) {   // :112-129
  if (x > 0.0) { raise(EXC_DOM_NB_X, x.v, x.np); return F(NAN); }
  if (!(s > 0.0)) { raise(EXC_DOM_NB_S, s.v, s.np); return F(NAN); }
  Py h = x / s;
  Py t = 0.5 * s;
  if (h < ASYMPTOTIC_H_THRESHOLD && t < SMALL_T_THRESHOLD + (ASYMPTOTIC_H_THRESHOLD - h)) {
    if (branch) *branch = 0;
    return asymptotic_black(h, t);
  }
  if (t < SMALL_T_THRESHOLD) { if (branch) *branch = 1; return small_t_black(h, t); }
  if (h + t > 0.85) {
    if (branch) *branch = 2;
    Py b_max = m_exp(0.5 * x);
    Py b = norm_cdf(h + t) * b_max - norm_cdf(h - t) / b_max;
    return py_max(b, F(0.0));
  }
  if (branch) *branch = 3;
  return erfcx_black(h, t);
}

static Py normalized_black_complement(Py x, Py s) {        // :132-137
  Py h = x / s;
  Py t = 0.5 * s;
  return m_exp(0.5 * x) * norm_cdf(-h - t) + m_exp(-0.5 * x) * norm_cdf(h - t);
}

static Py normalized_black_log(Py x, Py s) {               // :140-149
  Py h = x / s;
  Py t = 0.5 * s;
  Py diff = erfcx_(-(h + t) / SQRT_TWO) - erfcx_(-(h - t) / SQRT_TWO);
  if (diff <= 0.0) return F(-INFINITY);
  return -0.5 * (h * h + t * t) + m_log(0.5 * diff);
}

static Py normalized_vega(Py x, Py s) {                    // :152-156
  Py h = x / s;
  Py t = 0.5 * s;
  return INV_SQRT_TWO_PI * m_exp(-0.5 * (h * h + t * t));
}

struct Anchors { Py s_lo, s_c, s_hi, b_lo, b_c, b_hi; };
enum Region : int { FAR_LOW = 0, NEAR_LOW = 1, NEAR_HIGH = 2, FAR_HIGH = 3 };

static Anchors anchors_(Py x) {                            // :231-238
  Anchors a;
  a.s_c = m_sqrt(2.0 * py_abs(x));
  a.s_lo = a.s_c * REGION_RATIO;
  a.s_hi = a.s_c / REGION_RATIO;
  a.b_lo = normalized_black(x, a.s_lo);
  a.b_c = normalized_black(x, a.s_c);
  a.b_hi = normalized_black(x, a.s_hi);
  return a;
}

static int region_(Py beta, const Anchors& a) {            // :241-248
  if (beta < a.b_lo) return FAR_LOW;
  if (beta < a.b_c) return NEAR_LOW;
  if (beta < a.b_hi) return NEAR_HIGH;
  return FAR_HIGH;
}

static Py atm_inverse(Py beta) {                           // :258-262
  if (!(0.0 < beta.v && beta.v < 1.0)) { raise(EXC_DOM_ATM_BETA, beta.v, beta.np); return F(NAN); }
  return -2.0 * inv_norm_cdf(0.5 * (1.0 - beta));
}

static Py hermite_inverse(Py beta, Py b0, Py b1, Py s0, Py s1, Py x) {   // :265-280
  Py m0 = b0 / normalized_vega(x, s0);
  Py m1 = b1 / normalized_vega(x, s1);
  Py du = m_log(b1) - m_log(b0);
  Py u = (m_log(beta) - m_log(b0)) / du;
  Py u2 = u * u;
  Py u3 = u2 * u;
  Py s = ((2.0 * u3 - 3.0 * u2 + 1.0) * s0 + (u3 - 2.0 * u2 + u) * du * m0
          + (-2.0 * u3 + 3.0 * u2) * s1 + (u3 - u2) * du * m1);
  if (!(py_min(s0, s1) <= s && s <= py_max(s0, s1))) s = s0 + u * (s1 - s0);
  return s;
}

static Py far_low_guess(Py x, Py beta, const Anchors& a) {   // :283-309
  Py ln_beta = m_log(beta);
  Py s_cap = a.s_lo;
  Py s = py_abs(x) / m_sqrt(-2.0 * ln_beta);
  s = py_min(py_max(s, 1e-6 * s_cap), 0.999 * s_cap);
  Py v = m_log(s);
  Py v_hi = m_log(s_cap);
  for (int it = 0; it < 5; ++it) {
    if (RAISED) return F(NAN);
    Py g = normalized_black_log(x, s) - ln_beta;
    if (g > 0.0) v_hi = py_min(v_hi, v);
    Py dg_dv = s * m_exp(F(log(INV_SQRT_TWO_PI))
                         - 0.5 * (py_pow(x / s, 2) + 0.25 * s * s)
                         - normalized_black_log(x, s));
    if (RAISED) return F(NAN);
    if (!(isfin(dg_dv) && dg_dv > 0.0)) break;
    Py v_new = v - g / dg_dv;
    if (!isfin(v_new)) break;
    if (v_new >= v_hi) v_new = 0.5 * (v + v_hi);
    v = v_new;
    s = m_exp(v);
  }
  return s;
}

static Py far_high_guess(Py x, Py beta, Py b_max) {        // :312-318
  Py p = (b_max - beta) / (2.0 * b_max);
  p = py_min(py_max(p, F(5e-324)), F(0.5 * (1.0 - DBL_EPS)));
  Py z = inv_norm_cdf(p);
  return -z + m_sqrt(z * z + 2.0 * py_abs(x));
}

static Py initial_guess(Py x, Py beta, int region) {       // :321-332
  if (py_abs(x) < ATM_X_CUTOFF) return atm_inverse(beta);
  Anchors a = anchors_(x);
  if (region == FAR_LOW) return far_low_guess(x, beta, a);
  if (region == NEAR_LOW) return hermite_inverse(beta, a.b_lo, a.b_c, a.s_lo, a.s_c, x);
  if (region == NEAR_HIGH) return hermite_inverse(beta, a.b_c, a.b_hi, a.s_c, a.s_hi, x);
  return far_high_guess(x, beta, m_exp(0.5 * x));
}

static void vega_ratios(Py x, Py s, Py* r2, Py* r3) {      // :339-343
  *r2 = x * x / (s * s * s) - 0.25 * s;
  *r3 = (*r2) * (*r2) - 3.0 * x * x / py_pow(s, 4) - 0.25;
}

static void objective_branch(Py x, Py s, Py beta, int region, Py g[4]) {   // :346-389
  if (!(s > 0.0)) { raise(EXC_DOM_OBJ_S, s.v, s.np); return; }
  Py bp = normalized_vega(x, s);
  Py r2, r3;
  vega_ratios(x, s, &r2, &r3);
  if (region == FAR_LOW) {
    Py ln_b = normalized_black_log(x, s);
    Py ln_beta = m_log(beta);
    Py h = x / s;
    Py ln_bp = F(log(INV_SQRT_TWO_PI)) - 0.5 * (h * h + 0.25 * s * s);
    Py up = m_exp(ln_bp - ln_b);
    Py upp = up * r2 - up * up;
    Py uppp = up * r3 - 3.0 * up * up * r2 + 2.0 * py_pow(up, 3);
    Py inv = 1.0 / ln_b;
    Py inv2 = inv * inv;
    g[0] = inv - 1.0 / ln_beta;
    g[1] = -up * inv2;
    g[2] = -upp * inv2 + 2.0 * up * up * inv2 * inv;
    g[3] = (-uppp * inv2 + 6.0 * up * upp * inv2 * inv - 6.0 * py_pow(up, 3) * inv2 * inv2);
    return;
  }
  if (region == FAR_HIGH) {
    Py b_max = m_exp(0.5 * x);
    Py comp = normalized_black_complement(x, s);
    Py comp_beta = b_max - beta;
    Py w = bp / comp;
    g[0] = m_log(comp_beta) - m_log(comp);
    g[1] = w;
    g[2] = w * r2 + w * w;
    g[3] = w * r3 + 3.0 * w * w * r2 + 2.0 * py_pow(w, 3);
    return;
  }
  Py b = normalized_black(x, s);
  g[0] = b - beta; g[1] = bp; g[2] = bp * r2; g[3] = bp * r3;
}

static Py householder3_step(Py g, Py g1, Py g2, Py g3) {   // :392-402
  if (g == 0.0) return F(0.0);
  if (g1 == 0.0 || !isfin(g1)) return F(NAN);
  Py nu = -g / g1;
  Py eta = g2 / g1;
  Py gam = g3 / (6.0 * g1);
  return nu * (1.0 + 0.5 * nu * eta) / (1.0 + nu * (eta + nu * gam));
}

// implied_vol_lbr (:410-486); region_out = -1 when no region was selected.
static Result implied_vol_lbr(Py target, int theta, Py Fw, Py K, Py t, Py r, int* region_out) {
  const Py nan = F(NAN);
  const int max_iter = 8;
  *region_out = -1;
  // normalize_quote (:174-207)
  if (!(Fw > 0.0 && K > 0.0)) { raise(EXC_DOM_FK); return Result{nan, 0, MAX_ITER}; }
  Py xq = m_log(Fw / K);
  Py beta0 = target * m_exp(r * t) / m_sqrt(Fw * K);
  Py parity = m_exp(0.5 * xq) - m_exp(-0.5 * xq);
  if (RAISED) return Result{nan, 0, MAX_ITER};
  Py beta_work;
  if (theta > 0) beta_work = (xq > 0.0) ? beta0 - parity : beta0;
  else beta_work = (xq < 0.0) ? beta0 + parity : beta0;
  Py x_work = -py_abs(xq);
  Py b_max = m_exp(0.5 * x_work);
  if (beta_work <= 1e-300) return Result{nan, 0, BELOW_INTRINSIC};
  if (beta_work >= b_max * (1.0 - 1e-15)) return Result{nan, 0, ABOVE_UPPER};

  Py x = x_work;
  Py beta = beta_work;
  Py sqrt_t = m_sqrt(t);
  Py scale = m_sqrt(Fw * K) * m_exp(-r * t);
  (void)scale;   // only feeds the residual, which batch_iv discards
  if (RAISED) return Result{nan, 0, MAX_ITER};

  if (py_abs(x) < ATM_X_CUTOFF) {
    Py s = atm_inverse(beta);
    if (RAISED) return Result{nan, 0, MAX_ITER};
    normalized_black(py_min(x, F(0.0)), s);      // residual (:429): only its exceptions matter
    if (RAISED) return Result{nan, 0, MAX_ITER};
    return Result{s / sqrt_t, 0, CONVERGED};
  }

  Anchors an = anchors_(x);
  if (RAISED) return Result{nan, 0, MAX_ITER};
  int region = region_(beta, an);
  *region_out = region;
  Py lo, hi;
  if (region == FAR_LOW) { lo = F(0.0); hi = an.s_lo; }
  else if (region == NEAR_LOW) { lo = an.s_lo; hi = an.s_c; }
  else if (region == NEAR_HIGH) { lo = an.s_c; hi = an.s_hi; }
  else {
    lo = an.s_hi; hi = 2.0 * an.s_hi;
    Py comp_beta = b_max - beta;
    while (normalized_black_complement(x, hi) > comp_beta && hi < 1e6) {
      if (RAISED) return Result{nan, 0, MAX_ITER};
      hi = hi * 2.0;
    }
    if (RAISED) return Result{nan, 0, MAX_ITER};
  }
  lo = lo * (1.0 - 1e-6);
  hi = hi * (1.0 + 1e-6);

  Py s = initial_guess(x, beta, region);
  if (RAISED) return Result{nan, 0, MAX_ITER};
  TRACE(s.v);
  if (!(lo < s && s < hi)) s = 0.5 * (lo + hi);

  bool increasing = region != FAR_LOW;
  int iterations = 0;
  bool converged = false;
  for (int it = 0; it < max_iter; ++it) {
    Py g[4];
    objective_branch(x, s, beta, region, g);
    if (RAISED) return Result{nan, 0, MAX_ITER};
    TRACE(s.v); TRACE(g[0].v); TRACE(g[1].v); TRACE(g[2].v); TRACE(g[3].v);
    if (g[0] == 0.0) { converged = true; break; }
    bool below = increasing ? (g[0] < 0.0) : (g[0] > 0.0);
    if (below) lo = py_max(lo, s);
    else hi = py_min(hi, s);
    Py ds = householder3_step(g[0], g[1], g[2], g[3]);
    if (RAISED) return Result{nan, 0, MAX_ITER};
    if (isfin(ds) && py_abs(ds) <= STEP_TOLERANCE * py_max(F(1.0), s)) {
      s = s + ds;
      iterations += 1;
      converged = true;
      break;
    }
    Py cand = s + ds;
    if (!isfin(cand) || !(lo < cand && cand < hi)) {
      cand = 0.5 * (lo + hi);
      ds = cand - s;
    }
    s = cand;
    iterations += 1;
    if (py_abs(ds) <= STEP_TOLERANCE * py_max(F(1.0), s)) { converged = true; break; }
  }
  normalized_black(x, s);                       // residual (:484): only its exceptions matter
  if (RAISED) return Result{nan, 0, MAX_ITER};
  return Result{s / sqrt_t, iterations, converged ? CONVERGED : MAX_ITER};
}

}  // namespace orc

// ===========================================================================
// C ABI used by oracle/fvoracle.py (ctypes).  Columns are full-length,
// already broadcast and validated (batch.py:_assemble); per-row exception
// codes are returned so the Python side can reproduce the batch-level
// "first raising row aborts the batch" behaviour (batch.py:_run_chunked).
// model: 0 = BLACK76, 1 = BLACK_SCHOLES, 2 = BLACK_SCHOLES_MERTON.
// ===========================================================================
using namespace orc;

extern "C" {

int orc_init(void* erfcx_ptr, const double* facts18, const double* pascal324) {
  init_constants();
  g_erfcx = (erfcx_fn)erfcx_ptr;
  for (int i = 0; i < 18; ++i) g_asym_facts[i] = facts18[i];
  for (int i = 0; i < 18; ++i)
    for (int j = 0; j < 18; ++j) g_asym_pascal[i][j] = pascal324[i * 18 + j];
  return 0;
}

static inline void take_exc(int64_t i, int8_t* exc, double* exc_val, int8_t* exc_np) {
  exc[i] = (int8_t)S.exc;
  if (exc_val) exc_val[i] = S.exc_val;
  if (exc_np) exc_np[i] = (int8_t)S.exc_np;
  S = State();
}

// batch.py:181-203
void orc_batch_price(int model, const int8_t* flag, const double* un, const double* k,
                     const double* t, const double* r, const double* q, const double* sg,
                     int64_t n, double* out, int8_t* exc, double* exc_val, int8_t* exc_np) {
#pragma omp parallel for schedule(dynamic, 2048)
  for (int64_t i = 0; i < n; ++i) {
    S = State();
    Py v = (model == 0)
        ? price_black76(flag[i], N(un[i]), N(k[i]), N(t[i]), N(r[i]), N(sg[i]))
        : price_bsm(flag[i], N(un[i]), N(k[i]), N(t[i]), N(r[i]), N(q[i]), N(sg[i]));
    out[i] = v.v;
    take_exc(i, exc, exc_val, exc_np);
  }
}

// batch.py:250-280 (status 0 = ok, 1 = step_function_edge)
void orc_batch_greeks(int model, const int8_t* flag, const double* un, const double* k,
                      const double* t, const double* r, const double* q, const double* sg,
                      int64_t n, double* delta, double* gamma, double* theta, double* rho,
                      double* vega, int8_t* status, int8_t* exc, double* exc_val, int8_t* exc_np) {
#pragma omp parallel for schedule(dynamic, 2048)
  for (int64_t i = 0; i < n; ++i) {
    S = State();
    double g[5] = {NAN, NAN, NAN, NAN, NAN};
    int st = greeks_core(flag[i], model == 0, N(un[i]), N(k[i]), N(t[i]), N(r[i]), N(q[i]),
                         N(sg[i]), g);
    if (st == 1) { for (int j = 0; j < 5; ++j) g[j] = NAN; }
    delta[i] = g[0]; gamma[i] = g[1]; theta[i] = g[2]; rho[i] = g[3]; vega[i] = g[4];
    status[i] = (int8_t)st;
    take_exc(i, exc, exc_val, exc_np);
  }
}

// batch.py:206-247; method 0 = halley, 1 = lbr.  region may be NULL.
void orc_batch_iv(int model, int method, const int8_t* flag, const double* un, const double* k,
                  const double* t, const double* r, const double* q, const double* px,
                  int64_t n, double* iv, int8_t* status, int32_t* iters, int8_t* region,
                  int8_t* exc, double* exc_val, int8_t* exc_np) {
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < n; ++i) {
    S = State();
    Result res;
    int reg = -1;
    if (method == 1) {
      Py Fw = (model == 0) ? N(un[i]) : N(un[i]) * m_exp((N(r[i]) - N(q[i])) * N(t[i]));
      if (RAISED) res = Result{F(NAN), 0, MAX_ITER};
      else if (t[i] > 0.0) res = implied_vol_lbr(N(px[i]), flag[i], Fw, N(k[i]), N(t[i]), N(r[i]), &reg);
      else res = Result{F(NAN), 0, BELOW_INTRINSIC};
    } else {
      res = implied_vol_halley(N(px[i]), flag[i], model == 0, N(un[i]), N(k[i]), N(t[i]),
                               N(r[i]), N(q[i]));
    }
    bool ok = res.status == CONVERGED || res.status == FELL_BACK;
    iv[i] = ok ? res.sigma.v : NAN;
    status[i] = (int8_t)res.status;
    if (iters) iters[i] = res.iterations;
    if (region) region[i] = (int8_t)reg;
    take_exc(i, exc, exc_val, exc_np);
  }
}

// Debug: one LBR row with its value trace (guess, then s, g0..g3 per iteration).
int orc_trace_lbr(int theta, double Fw, double K, double t, double r, double px, double* trace) {
  S = State();
  g_trace = trace; g_trace_n = 0;
  int reg = -1;
  implied_vol_lbr(N(px), theta, N(Fw), N(K), N(t), N(r), &reg);
  g_trace = nullptr;
  return g_trace_n;
}

// Scalar probes for the reference's own known-answer tests (test_iv_lbr.py).
double orc_normalized_black(double x, double s, int* branch) {
  S = State();
  return normalized_black(F(x), F(s), branch).v;
}
double orc_norm_cdf(double x) { S = State(); return norm_cdf(F(x)).v; }
double orc_inv_norm_cdf(double p) { S = State(); return inv_norm_cdf(F(p)).v; }

}  // extern "C"
