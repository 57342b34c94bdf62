// Host build of paper_2604_27210_b200/csrc/fv_quote.h (the device per-quote
// code) for CPU pre-checks against the oracle / golden fixtures.  Test
// infrastructure only: the product runs the CUDA build of the same header.
// Build: g++ -O2 -ffp-contract=off -fno-fast-math -shared -fPIC
#include "../../paper_2604_27210_b200/csrc/fv_fast.h"

extern "C" {

void qh_price(int model, const int8_t* flag, const double* un, const double* k, const double* t,
              const double* r, const double* q, const double* sg, int64_t n, double* out,
              int8_t* exc) {
  for (int64_t i = 0; i < n; ++i) {
    FvExc e = {0, 0, 0.0};
    out[i] = fv_price_row(model, (double)flag[i], un[i], k[i], t[i], r[i], q[i], sg[i], e);
    exc[i] = (int8_t)e.code;
  }
}

void qh_price_greeks(int model, const int8_t* flag, const double* un, const double* k,
                     const double* t, const double* r, const double* q, const double* sg,
                     int64_t n, double* price, double* g5, int8_t* status, int8_t* excp,
                     int8_t* excg) {
  for (int64_t i = 0; i < n; ++i) {
    FvExc ep = {0, 0, 0.0}, eg = {0, 0, 0.0};
    FvGreeks o = fv_price_greeks_row(model, (double)flag[i], un[i], k[i], t[i], r[i], q[i], sg[i],
                                     true, true, ep, eg);
    price[i] = o.price;
    g5[5 * i + 0] = o.delta; g5[5 * i + 1] = o.gamma; g5[5 * i + 2] = o.theta;
    g5[5 * i + 3] = o.rho; g5[5 * i + 4] = o.vega;
    status[i] = (int8_t)o.status;
    excp[i] = (int8_t)ep.code; excg[i] = (int8_t)eg.code;
  }
}

void qh_iv(int model, int method, const int8_t* flag, const double* un, const double* k,
           const double* t, const double* r, const double* q, const double* px, int64_t n,
           double* iv, int8_t* status, int8_t* region, int8_t* exc, double* exc_val,
           int8_t* exc_np) {
  for (int64_t i = 0; i < n; ++i) {
    FvExc e = {0, 0, 0.0};
    if (method == 1) {
      FvLbrOut o = fv_lbr_batch_row(model, (double)flag[i], un[i], k[i], t[i], r[i], q[i], px[i], e);
      iv[i] = o.sigma; status[i] = (int8_t)o.status; region[i] = (int8_t)o.region;
    } else {
      int status_; double sig;
      fv_halley_row_sm(model, (double)flag[i], un[i], k[i], t[i], r[i], q[i], px[i], &status_, &sig, e);
      iv[i] = sig;
      status[i] = (int8_t)status_; region[i] = -1;
    }
    exc[i] = (int8_t)e.code; exc_val[i] = e.val; exc_np[i] = (int8_t)e.np;
  }
}

double qh_normalized_black(double x, double s, int* branch) {
  FvExc e = {0, 0, 0.0};
  return fv_normalized_black(x, s, false, e, nullptr, branch);
}
}

extern "C" {
// Bit-compare the fused far-low solver against the reference-order one on
// the far-low quotes of a batch; returns the number of mismatching rows.
int64_t qh_far_low_fused_check(const int8_t* flag, const double* F, const double* k,
                               const double* t, const double* r, const double* px, int64_t n,
                               int64_t* nfar) {
  int64_t bad = 0, nf = 0;
  for (int64_t i = 0; i < n; ++i) {
    FvExc e = {0, 0, 0.0};
    FvLbrState st; FvLbrOut o;
    if (!(t[i] > 0.0)) continue;
    if (fv_lbr_classify((double)flag[i], F[i], k[i], t[i], r[i], px[i], st, o, e)) continue;
    if (o.region != FV_FAR_LOW) continue;
    ++nf;
    FvExc e1 = {0, 0, 0.0}, e2 = {0, 0, 0.0};
    FvLbrOut a = fv_lbr_solve<FV_FAR_LOW>(FV_FAR_LOW, st, e1);
    FvLbrOut b = fv_lbr_far_low_fused(st, e2);
    uint64_t ua, ub; memcpy(&ua, &a.sigma, 8); memcpy(&ub, &b.sigma, 8);
    bool same = (ua == ub || (a.sigma != a.sigma && b.sigma != b.sigma)) && a.status == b.status &&
                a.iterations == b.iterations && e1.code == e2.code;
    if (!same) ++bad;
  }
  *nfar = nf;
  return bad;
}

// The straight-line first pass (fx_lbr_classify_lo) against the careful one
// (batch.py fill's forward + fv_lbr_normalize + fv_lbr_anchor_lo): returns
// mismatching unflagged rows; *nflag gets the flagged ones.
int64_t qh_classify_fast_check(int model, const int8_t* flag, const double* un, const double* k,
                               const double* t, const double* r, const double* q, const double* px,
                               int64_t n, int64_t* nflag) {
  int64_t bad = 0, nb = 0;
  for (int64_t i = 0; i < n; ++i) {
    FxBad flagged;
    FvLbrState sf; FvLbrOut of;
    sf.x = sf.beta = sf.sqrt_t = sf.s_c = sf.b0 = sf.E0 = 0.0;
    const int cf = fx_lbr_classify_lo(model, (double)flag[i], un[i], k[i], t[i], r[i], q[i], px[i], sf, of, flagged);
    if (flagged) { ++nb; continue; }
    // careful
    FvExc e = {0, 0, 0.0};
    FvLbrState sc; FvLbrOut oc;
    sc.x = sc.beta = sc.sqrt_t = sc.s_c = sc.b0 = sc.E0 = 0.0;
    oc.sigma = __builtin_nan(""); oc.status = FV_IV_MAX_ITER;
    double Fw = un[i];
    bool done = true;
    if (model != 0) Fw = un[i] * py_exp((r[i] - q[i]) * t[i], e);
    if (e.code) {
    } else if (!(t[i] > 0.0)) {
      oc.status = FV_IV_BELOW_INTRINSIC;
    } else {
      done = fv_lbr_normalize((double)flag[i], Fw, k[i], t[i], r[i], px[i], sc, oc, e) != 0;
    }
    int cc = FV_REGION_NONE;
    if (!(done || e.code)) cc = fv_lbr_anchor_lo(sc, e);
    if (e.code) { ++bad; continue; }                 // unflagged but the careful path raises
    bool same = cf == cc;
    if (same && cc == FV_REGION_NONE) {
      uint64_t ua, ub; memcpy(&ua, &of.sigma, 8); memcpy(&ub, &oc.sigma, 8);
      same = of.status == oc.status && (oc.status != FV_IV_CONVERGED || ua == ub);
    } else if (same) {
      // (sqrt_t is recomputed by the solves, not handed on by this pass)
      const double fa[5] = {sf.x, sf.beta, sf.s_c, sf.b0, sf.E0};
      const double ca[5] = {sc.x, sc.beta, sc.s_c, sc.b0, sc.E0};
      same = memcmp(fa, ca, sizeof(fa)) == 0;
    }
    if (!same) ++bad;
  }
  *nflag = nb;
  return bad;
}

// Straight-line price / fused price+Greeks rows against the careful rows:
// mismatching unflagged rows (any output bit, status, or a careful-path
// exception); *nflag gets the flagged ones.
int64_t qh_price_greeks_fast_check(int model, const int8_t* flag, const double* un, const double* k,
                                   const double* t, const double* r, const double* q, const double* sg,
                                   int64_t n, int64_t* nflag) {
  int64_t bad = 0, nb = 0;
  for (int64_t i = 0; i < n; ++i) {
    FxBad f1, f2;
    const double pf = fx_price_row(model, (double)flag[i], un[i], k[i], t[i], r[i], q[i], sg[i], f1);
    const FvGreeks gf = fx_price_greeks_row(model, (double)flag[i], un[i], k[i], t[i], r[i], q[i], sg[i], true, f2);
    if (f1 || f2) { ++nb; }
    FvExc e = {0, 0, 0.0}, ep = {0, 0, 0.0}, eg = {0, 0, 0.0};
    const double pc = fv_price_row(model, (double)flag[i], un[i], k[i], t[i], r[i], q[i], sg[i], e);
    const FvGreeks gc = fv_price_greeks_row(model, (double)flag[i], un[i], k[i], t[i], r[i], q[i], sg[i],
                                            true, true, ep, eg);
    if (!f1 && (memcmp(&pf, &pc, 8) != 0 || e.code)) ++bad;
    if (!f2) {
      const double a[6] = {gf.price, gf.delta, gf.gamma, gf.theta, gf.rho, gf.vega};
      const double b[6] = {gc.price, gc.delta, gc.gamma, gc.theta, gc.rho, gc.vega};
      if (memcmp(a, b, sizeof(a)) != 0 || gf.status != gc.status || ep.code || eg.code) ++bad;
    }
  }
  *nflag = nb;
  return bad;
}

// The straight-line Halley state machine (fx_hsm_pre / fx_halley_f) against
// the careful solver (fv_halley_row_sm): mismatching unflagged rows; *nflag
// gets the flagged ones.
int64_t qh_halley_fast_check(int model, const int8_t* flag, const double* un, const double* k,
                             const double* t, const double* r, const double* q, const double* px,
                             int64_t n, int64_t* nflag) {
  int64_t bad = 0, nb = 0;
  for (int64_t i = 0; i < n; ++i) {
    FvExc e0 = {0, 0, 0.0};
    FvHalleySM m;
    int st_c; double sg_c;
    FvExc ec = {0, 0, 0.0};
    fv_halley_row_sm(model, (double)flag[i], un[i], k[i], t[i], r[i], q[i], px[i], &st_c, &sg_c, ec);
    if (fv_hsm_setup(model, (double)flag[i], un[i], k[i], t[i], r[i], q[i], px[i], m, e0)) continue;
    FxBad flagged;
    for (;;) {
      double x;
      if (!fx_hsm_pre(m, &x, flagged)) break;
      const double fx = fx_halley_f(m.c, x, flagged);
      if (flagged) break;
      FvExc e = {0, 0, 0.0};
      fv_hsm_post(m, fx, e);
      if (m.state == FV_HS_DONE) break;
    }
    if (flagged) { ++nb; continue; }
    const double sg = (m.status == FV_IV_CONVERGED || m.status == FV_IV_FELL_BACK) ? m.out_sigma : __builtin_nan("");
    uint64_t ua, ub; memcpy(&ua, &sg, 8); memcpy(&ub, &sg_c, 8);
    if (m.status != st_c || !(ua == ub || (sg != sg && sg_c != sg_c)) || ec.code) ++bad;
  }
  *nflag = nb;
  return bad;
}

// The straight-line second anchor stage (fx_lbr_anchor_rest) against the
// careful one on the non-far-low quotes of a batch.
int64_t qh_anchor_rest_fast_check(const int8_t* flag, const double* F, const double* k, const double* t,
                                  const double* r, const double* px, int64_t n, int64_t* nseen, int64_t* nflag) {
  int64_t bad = 0, ns = 0, nb = 0;
  for (int64_t i = 0; i < n; ++i) {
    FvExc e = {0, 0, 0.0};
    FvLbrState st; FvLbrOut o;
    if (!(t[i] > 0.0)) continue;
    if (fv_lbr_normalize((double)flag[i], F[i], k[i], t[i], r[i], px[i], st, o, e)) continue;
    if (fv_lbr_anchor_lo(st, e) != FV_NEAR_LOW) continue;
    ++ns;
    FvLbrState sf = st, sc = st;
    FxBad flagged;
    FvExc e2 = {0, 0, 0.0};
    const int rf = fx_lbr_anchor_rest(sf, flagged);
    const int rc = fv_lbr_anchor_rest(sc, e2);
    if (flagged) { ++nb; continue; }
    bool same = rf == rc && e2.code == 0;
    if (same && rc != FV_FAR_HIGH) {
      const double fa[4] = {sf.b0, sf.b1, sf.E0, sf.E1}, ca[4] = {sc.b0, sc.b1, sc.E0, sc.E1};
      same = memcmp(fa, ca, sizeof(fa)) == 0;
    }
    if (!same) ++bad;
  }
  *nseen = ns;
  *nflag = nb;
  return bad;
}

// The straight-line near-region solver (fx_lbr_near) against the careful one
// on the near-region quotes of a batch: mismatching unflagged rows; *nflag
// gets the flagged ones, *nnear the near quotes seen.
int64_t qh_near_fast_check(const int8_t* flag, const double* F, const double* k, const double* t,
                           const double* r, const double* px, int64_t n, int64_t* nnear, int64_t* nflag) {
  int64_t bad = 0, nn = 0, nb = 0;
  for (int64_t i = 0; i < n; ++i) {
    FvExc e = {0, 0, 0.0};
    FvLbrState st; FvLbrOut o;
    if (!(t[i] > 0.0)) continue;
    if (fv_lbr_classify((double)flag[i], F[i], k[i], t[i], r[i], px[i], st, o, e)) continue;
    if (o.region != FV_NEAR_LOW && o.region != FV_NEAR_HIGH) continue;
    ++nn;
    FvExc e2 = {0, 0, 0.0};
    FxBad flagged;
    FvLbrOut a = fx_lbr_near(o.region, st, flagged);
    FvLbrOut c = fv_lbr_solve<FV_NEAR_LOW>(o.region, st, e2);
    if (flagged) { ++nb; continue; }
    uint64_t ua, uc; memcpy(&ua, &a.sigma, 8); memcpy(&uc, &c.sigma, 8);
    bool same = (ua == uc || (a.sigma != a.sigma && c.sigma != c.sigma)) && a.status == c.status &&
                a.iterations == c.iterations && e2.code == 0;
    if (!same) ++bad;
  }
  *nnear = nn;
  *nflag = nb;
  return bad;
}

// The straight-line far-low solver (fv_fast.h) against the careful one on the
// far-low quotes of a batch: returns mismatching unflagged rows; *nflag gets
// the flagged (handed-back) ones.
int64_t qh_far_low_fast_check(const int8_t* flag, const double* F, const double* k,
                              const double* t, const double* r, const double* px, int64_t n,
                              int64_t* nfar, int64_t* nflag) {
  int64_t bad = 0, nf = 0, nb = 0;
  for (int64_t i = 0; i < n; ++i) {
    FvExc e = {0, 0, 0.0};
    FvLbrState st; FvLbrOut o;
    if (!(t[i] > 0.0)) continue;
    if (fv_lbr_classify((double)flag[i], F[i], k[i], t[i], r[i], px[i], st, o, e)) continue;
    if (o.region != FV_FAR_LOW) continue;
    ++nf;
    FvExc e2 = {0, 0, 0.0};
    FxBad flagged;
    FvLbrOut a = fx_lbr_far_low(st, flagged);
    FvLbrOut b = fv_lbr_far_low_fused(st, e2);
    if (flagged) { ++nb; continue; }
    uint64_t ua, ub; memcpy(&ua, &a.sigma, 8); memcpy(&ub, &b.sigma, 8);
    bool same = (ua == ub || (a.sigma != a.sigma && b.sigma != b.sigma)) && a.status == b.status &&
                a.iterations == b.iterations && e2.code == 0;
    if (!same) ++bad;
  }
  *nfar = nf;
  *nflag = nb;
  return bad;
}
}

extern "C" {
// fx_erfc_u2 (all ranges through one rational form) on pairs (x[i],
// x[n-1-i]): every unflagged value must carry fv_erfc_i's bits, and the
// flags must be fx_erfc's.  Returns mismatches; *nflag = flagged values.
int64_t qh_erfc_u_check(const double* x, int64_t n, int64_t* nflag) {
  int64_t bad = 0, nb = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double xa = x[i], xb = x[n - 1 - i];
    for (int mode = 0; mode < 3; ++mode) {           // both wanted, only a, only b
      const bool va = mode != 2, vb = mode != 1;
      double ra, rb;
      FxBad f;
      fx_erfc_u2(xa, xb, va, vb, ra, rb, f);
      FxBad fa, fb;
      const double ca = fx_erfc(xa, fa), cb = fx_erfc(xb, fb);
      const bool want_flag = (va && fa) || (vb && fb);
      if ((bool)f != want_flag) { ++bad; continue; }
      if (f) { ++nb; continue; }
      const double ea = fv_erfc_i(xa), eb = fv_erfc_i(xb);
      uint64_t u0, u1;
      if (va) { memcpy(&u0, &ra, 8); memcpy(&u1, &ea, 8); if (u0 != u1) ++bad; memcpy(&u1, &ca, 8); if (u0 != u1) ++bad; }
      if (vb) { memcpy(&u0, &rb, 8); memcpy(&u1, &eb, 8); if (u0 != u1) ++bad; memcpy(&u1, &cb, 8); if (u0 != u1) ++bad; }
    }
  }
  *nflag = nb;
  return bad;
}
}

extern "C" {
// fx_halley_sign (fp32 with a margin) against the sign of the careful f(sigma)
// at the bracket's sigma values: returns rows where a decided sign differs;
// *undecided = rows it left to the exact evaluation.
int64_t qh_halley_sign_check(int model, const int8_t* flag, const double* un, const double* k,
                             const double* t, const double* r, const double* q, const double* px,
                             int64_t n, const double* sigmas, int nsig, int64_t* undecided) {
  int64_t bad = 0, und = 0;
  for (int64_t i = 0; i < n; ++i) {
    FvExc e = {0, 0, 0.0};
    FvHalleySM m;
    if (fv_hsm_setup(model, (double)flag[i], un[i], k[i], t[i], r[i], q[i], px[i], m, e)) continue;
    if (m.c.fk_bad) continue;
    for (int j = 0; j < nsig; ++j) {
      FvExc e2 = {0, 0, 0.0};
      const double f = fv_halley_f(m.c, sigmas[j], e2);
      const int sg = fx_halley_sign(m.c, sigmas[j]);
      if (sg == 0) { ++und; continue; }
      if (e2.code || (sg > 0 && !(f > 0.0)) || (sg < 0 && !(f < 0.0))) ++bad;
    }
  }
  *undecided = und;
  return bad;
}
}
