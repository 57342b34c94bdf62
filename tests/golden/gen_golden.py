#!/usr/bin/env python3
"""Generate the golden parity fixtures in tests/golden/ by running the REAL
reference implementation (fastvol 0.1.0, /root/reference/pkg/src, imported
read-only) on seeded inputs.  Run in the build container (the reference does
not exist on the GPU box); the .npz/.json outputs are committed.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_golden.py

Fixtures (inputs + reference outputs, statuses as int8 codes):
  lbr_c1.npz      C1 draws, Black-76 LBR           (bench.py:19-31 generator)
  lbr_c4.npz      strided sample of the 100M C4 chain, Black-76 LBR
  lbr_c5.npz      C5 wing-stress set, Black-76 LBR
  lbr_bsm.npz     C2 draws, BSM LBR (spot -> forward in batch.py:229)
  lbr_grid.npz    the acceptance LBR round-trip grid (test_acceptance.py:98-120)
  halley_c2.npz   C2 draws, BSM Halley with q
  halley_c5.npz   C5 wing-stress set, Black-76 Halley
  halley_grid.npz the acceptance Halley grid, all 3 models (test_acceptance.py:37-62)
  price_greeks.npz C3 draws priced + Greeks for BSM, BS, Black-76
  nb_points.npz   normalized_black / norm_cdf / inv_norm_cdf point values
  exceptions.json fuzzed extreme rows, one reference call per row: value or
                  the exception type + message the reference raises
  validation.json batches the front end rejects: BatchError kind/index/detail
"""

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from fastvol import batch as B  # noqa: E402
from fastvol import lbr as L  # noqa: E402
from fastvol import distributions as D  # noqa: E402
from fastvol.models import Model  # noqa: E402
import workloads as W  # noqa: E402

IV_CODES = {"converged": 0, "fell_back_to_bisection": 1, "below_intrinsic": 2,
            "above_upper_bound": 3, "max_iterations": 4}
GK_CODES = {"ok": 0, "step_function_edge": 1}
REGION_CODES = {"far_low": 0, "near_low": 1, "near_high": 2, "far_high": 3}


def chars(flag):
    return list(W.flag_chars(flag))


def lbr_regions(flag, F, K, t, r, px):
    """Reference region per row (-1 when the quote is rejected or ATM)."""
    out = np.full(len(flag), -1, np.int8)
    for i in range(len(flag)):
        if not t[i] > 0.0:
            continue
        try:
            q = L.normalize_quote(int(flag[i]), F[i], K[i], t[i], r[i], px[i])
        except (L.BelowIntrinsicError, L.AboveUpperBoundError):
            continue
        if abs(q.x_work) < L.ATM_X_CUTOFF:
            continue
        out[i] = REGION_CODES[L.select_region(q.x_work, q.beta_work).value]
    return out


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, {k: v.shape for k, v in arrays.items()})


def iv_fixture(name, model, method, flag, un, K, t, r, q, px, with_region):
    tb = B.batch_iv(model, method, chars(flag), un, K, t, r, price=px, q=q)
    st = np.array([IV_CODES[s] for s in tb["status"]], np.int8)
    extra = {}
    if with_region:
        F = un if model is Model.BLACK76 else un * np.exp((r - q) * t)
        if model is Model.BLACK76:
            extra["region"] = lbr_regions(flag, un, K, t, r, px)
    save(name, model=np.array(model.value), method=np.array(method), flag=flag,
         underlying=un, strike=K, t=t, r=r, q=np.broadcast_to(np.asarray(q, float), un.shape).copy(),
         price=px, iv=np.asarray(tb["iv"], np.float64), status=st, **extra)


def b76_prices(flag, F, K, t, r, sigma):
    return np.asarray(B.batch_price(Model.BLACK76, chars(flag), F, K, t, r, sigma=sigma)["price"])


def main():
    # ---- C1: synthetic_chain draws read as Black-76 forwards ---------------
    flag, S, K, t, r, q, sig = W.chain_draws(6000, seed=0)
    px = b76_prices(flag, S, K, t, r, sig)
    iv_fixture("lbr_c1.npz", Model.BLACK76, "lbr", flag, S, K, t, r, 0.0, px, True)

    # ---- C4 strided sample -------------------------------------------------
    rows = np.arange(0, W.C4_ROWS, W.C4_ROWS // 4000 + 7)
    parts = [W.c4_params(int(i), int(i) + 1) for i in rows]
    flag4, F4, K4, t4, r4, s4 = (np.concatenate([p[j] for p in parts]) for j in range(6))
    px4 = b76_prices(flag4, F4, K4, t4, r4, s4)
    iv_fixture("lbr_c4.npz", Model.BLACK76, "lbr", flag4, F4, K4, t4, r4, 0.0, px4, True)

    # ---- C5 wing stress -----------------------------------------------------
    flag5, F5, K5, t5, r5, s5, kind5, side5 = W.c5_params(6000, seed=5)
    px5 = W.c5_prices(flag5, F5, K5, t5, r5, kind5, side5, b76_prices(flag5, F5, K5, t5, r5, s5))
    iv_fixture("lbr_c5.npz", Model.BLACK76, "lbr", flag5, F5, K5, t5, r5, 0.0, px5, True)
    iv_fixture("halley_c5.npz", Model.BLACK76, "halley", flag5[:3000], F5[:3000], K5[:3000],
               t5[:3000], r5[:3000], 0.0, px5[:3000], False)

    # ---- C2: BSM with dividend yield ---------------------------------------
    flag2, S2, K2, t2, r2, q2, s2 = W.chain_draws(3000, seed=0)
    px2 = np.asarray(B.batch_price(Model.BLACK_SCHOLES_MERTON, chars(flag2), S2, K2, t2, r2,
                                   q2, sigma=s2)["price"])
    iv_fixture("halley_c2.npz", Model.BLACK_SCHOLES_MERTON, "halley", flag2, S2, K2, t2, r2,
               q2, px2, False)
    iv_fixture("lbr_bsm.npz", Model.BLACK_SCHOLES_MERTON, "lbr", flag2[:2000], S2[:2000],
               K2[:2000], t2[:2000], r2[:2000], q2[:2000], px2[:2000], False)

    # ---- acceptance LBR grid (test_acceptance.py:98-120) --------------------
    xs = np.concatenate([[0.0], -np.logspace(-3, 1.0, 20)])
    ss = np.logspace(-3, math.log10(5.0), 30)
    g_flag, g_F, g_K, g_px = [], [], [], []
    for x in xs:
        for s in ss:
            beta = L.normalized_black(float(x), float(s))
            for th in (1, -1):
                Fv = 100.0
                Kv = Fv * math.exp(-float(x) * th)
                g_flag.append(th); g_F.append(Fv); g_K.append(Kv)
                g_px.append(beta * math.sqrt(Fv * Kv))
    g_flag = np.array(g_flag, np.int8)
    g_F, g_K, g_px = (np.array(a, np.float64) for a in (g_F, g_K, g_px))
    ones = np.ones_like(g_F)
    iv_fixture("lbr_grid.npz", Model.BLACK76, "lbr", g_flag, g_F, g_K, ones, 0.0 * ones, 0.0,
               g_px, True)

    # ---- acceptance Halley grid, three models -------------------------------
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import halley_grid
    from fastvol.models import PricingInputs
    from fastvol.pricing import price as ref_price
    arrs = {k: [] for k in ("model", "flag", "underlying", "strike", "t", "r", "q", "price")}
    for mi, model in enumerate((Model.BLACK76, Model.BLACK_SCHOLES, Model.BLACK_SCHOLES_MERTON)):
        for x, sg, tt, rr, th in halley_grid():
            qq = 0.01 if model is Model.BLACK_SCHOLES_MERTON else 0.0
            under = 100.0
            Kv = under * math.exp(-x) if model is Model.BLACK76 else under * math.exp((rr - qq) * tt - x)
            target = ref_price(th, PricingInputs(model, under, Kv, tt, rr, qq, sg))
            for k, v in zip(arrs, (mi, th, under, Kv, tt, rr, qq, target)):
                arrs[k].append(v)
    out = {}
    for mi, model in enumerate((Model.BLACK76, Model.BLACK_SCHOLES, Model.BLACK_SCHOLES_MERTON)):
        sel = [i for i, m in enumerate(arrs["model"]) if m == mi]
        cols = {k: np.array([arrs[k][i] for i in sel]) for k in arrs}
        tb = B.batch_iv(model, "halley", chars(cols["flag"]), cols["underlying"], cols["strike"],
                        cols["t"], cols["r"], price=cols["price"], q=cols["q"])
        for k in ("flag", "underlying", "strike", "t", "r", "q", "price"):
            out[f"{model.value}_{k}"] = cols[k].astype(np.int8 if k == "flag" else np.float64)
        out[f"{model.value}_iv"] = np.asarray(tb["iv"], np.float64)
        out[f"{model.value}_status"] = np.array([IV_CODES[s] for s in tb["status"]], np.int8)
    save("halley_grid.npz", **out)

    # ---- C3: price + Greeks, all three models -------------------------------
    flag3, S3, K3, t3, r3, q3, s3 = W.chain_draws(4000, seed=3)
    # sprinkle zero-vol / zero-time rows (step_function_edge, discounted intrinsic)
    s3[::97] = 0.0
    t3[::89] = 0.0
    out = {}
    for model in (Model.BLACK_SCHOLES_MERTON, Model.BLACK_SCHOLES, Model.BLACK76):
        qq = q3 if model is Model.BLACK_SCHOLES_MERTON else 0.0
        p = B.batch_price(model, chars(flag3), S3, K3, t3, r3, qq, sigma=s3)
        g = B.batch_greeks(model, chars(flag3), S3, K3, t3, r3, qq, sigma=s3)
        out[f"{model.value}_price"] = np.asarray(p["price"], np.float64)
        for gname in B.GREEK_COLUMNS:
            out[f"{model.value}_{gname}"] = np.asarray(g[gname], np.float64)
        out[f"{model.value}_status"] = np.array([GK_CODES[s] for s in g["status"]], np.int8)
    save("price_greeks.npz", flag=flag3, underlying=S3, strike=K3, t=t3, r=r3, q=q3, sigma=s3,
         **out)

    # ---- scalar point values -------------------------------------------------
    rng = np.random.default_rng(11)
    nb_x = np.concatenate([-10 ** rng.uniform(-4, 1.3, 6000), -rng.uniform(0, 3, 2000),
                           np.array([p[0] for p in [(-0.5, 0.3), (-0.02, 0.1), (-0.5, 1.0),
                                                    (-0.3, 0.6), (-1.5, 0.9), (-1.0, 3.0),
                                                    (-2.0, 0.15), (-4.0, 0.35), (-8.0, 0.3)]])])
    nb_s = np.concatenate([10 ** rng.uniform(-3, 1.2, 6000), 10 ** rng.uniform(-3, 0.7, 2000),
                           np.array([0.3, 0.1, 1.0, 0.6, 0.9, 3.0, 0.15, 0.35, 0.3])])
    nb = np.array([L.normalized_black(float(a), float(b)) for a, b in zip(nb_x, nb_s)])
    cx = rng.uniform(-40, 40, 4000)
    cdf = np.array([D.norm_cdf(float(v)) for v in cx])
    pp = np.concatenate([rng.uniform(1e-9, 1 - 1e-9, 3000), 10 ** rng.uniform(-300, -1, 1000)])
    icdf = np.array([D.inv_norm_cdf(float(v)) for v in pp])
    save("nb_points.npz", nb_x=nb_x, nb_s=nb_s, nb=nb, cdf_x=cx, cdf=cdf, icdf_p=pp, icdf=icdf)

    gen_exceptions()
    gen_validation()


def _outcome(fn):
    try:
        tb = fn()
    except Exception as exc:  # noqa: BLE001 -- we record exactly what is raised
        name = type(exc).__name__
        if name == "DomainError":
            name = "DomainError"
        return {"exc": name, "msg": str(exc)}
    return {k: (None if v is None else v) for k, v in tb.items()}


def gen_exceptions():
    """Extreme-but-finite rows, one reference call per row."""
    rng = np.random.default_rng(2024)
    n = 700
    cases = []

    def draw():
        lf = rng.uniform(-300, 300, n)
        F = 10.0 ** lf
        x = np.where(rng.random(n) < 0.5, rng.uniform(-1500, 1500, n), rng.uniform(-20, 20, n))
        x = np.where(rng.random(n) < 0.2, rng.uniform(690, 1500, n) * np.sign(rng.uniform(-1, 1, n)), x)
        K = F * np.exp(np.clip(-x, -700, 700))
        K = np.where(rng.random(n) < 0.3, 10.0 ** rng.uniform(-300, 300, n), K)
        t = 10.0 ** rng.uniform(-9, 3.5, n)
        r = np.where(rng.random(n) < 0.5, rng.uniform(-5, 5, n), rng.uniform(-0.1, 0.1, n))
        q = np.where(rng.random(n) < 0.5, rng.uniform(-5, 5, n), 0.0)
        sig = 10.0 ** rng.uniform(-15, 3, n)
        lp = rng.uniform(-320, 300, n)
        price = 10.0 ** lp
        flag = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
        ok = np.isfinite(F) & (F > 0) & np.isfinite(K) & (K > 0) & np.isfinite(price)
        return flag[ok], F[ok], K[ok], t[ok], r[ok], q[ok], sig[ok], price[ok]

    for model in (Model.BLACK76, Model.BLACK_SCHOLES_MERTON):
        flag, F, K, t, r, q, sig, price = draw()
        qq = q if model is Model.BLACK_SCHOLES_MERTON else np.zeros_like(q)
        for i in range(len(flag)):
            args = dict(model=model.value, flag=int(flag[i]), underlying=F[i], strike=K[i],
                        t=t[i], r=r[i], q=qq[i], sigma=sig[i], price=price[i])
            fl = chars(flag[i:i + 1])
            o_p = _outcome(lambda: {"price": float(B.batch_price(model, fl, F[i:i+1], K[i:i+1], t[i:i+1], r[i:i+1], qq[i:i+1], sigma=sig[i:i+1])["price"][0])})
            o_g = _outcome(lambda: {g: float(v) for g, v in ((g, B.batch_greeks(model, fl, F[i:i+1], K[i:i+1], t[i:i+1], r[i:i+1], qq[i:i+1], sigma=sig[i:i+1])[g][0]) for g in B.GREEK_COLUMNS)})
            o_l = _outcome(lambda: (lambda tb: {"iv": float(tb["iv"][0]), "status": str(tb["status"][0])})(B.batch_iv(model, "lbr", fl, F[i:i+1], K[i:i+1], t[i:i+1], r[i:i+1], price=price[i:i+1], q=qq[i:i+1])))
            o_h = _outcome(lambda: (lambda tb: {"iv": float(tb["iv"][0]), "status": str(tb["status"][0])})(B.batch_iv(model, "halley", fl, F[i:i+1], K[i:i+1], t[i:i+1], r[i:i+1], price=price[i:i+1], q=qq[i:i+1])))
            cases.append({"in": {k: (float(v) if not isinstance(v, str) else v) for k, v in args.items()},
                          "price": o_p, "greeks": o_g, "lbr": o_l, "halley": o_h})
    # deep-wing rows near |x| ~ 700..1420 with in-band prices (NEAR_LOW hermite, parity overflow)
    for xv in list(np.linspace(600, 1450, 60)):
        for th in (1, -1):
            for lb in (-305.0, -250.0, -160.0, -100.0, -40.0):
                # log(F/K) = xv*th with F, K representable (|x| up to ~1450)
                lf = 709.0 if th > 0 else -744.0
                Fv = math.exp(lf)
                Kv = math.exp(lf - xv * th)
                if not (Fv > 0 and Kv > 0 and math.isfinite(Kv)):
                    continue
                args = dict(model="black", flag=th, underlying=Fv, strike=Kv, t=1.0, r=0.0, q=0.0,
                            sigma=1.0, price=10.0 ** lb)
                fl = ["c" if th > 0 else "p"]
                o_l = _outcome(lambda: (lambda tb: {"iv": float(tb["iv"][0]), "status": str(tb["status"][0])})(B.batch_iv(Model.BLACK76, "lbr", fl, [Fv], [Kv], [1.0], [0.0], price=[10.0 ** lb])))
                cases.append({"in": args, "lbr": o_l})
    path = os.path.join(HERE, "exceptions.json")
    with open(path, "w") as f:
        json.dump(cases, f, allow_nan=True)
    kinds = {}
    for c in cases:
        for key in ("price", "greeks", "lbr", "halley"):
            if key in c and "exc" in c[key]:
                kinds[(key, c[key]["exc"], c[key]["msg"][:40])] = kinds.get((key, c[key]["exc"], c[key]["msg"][:40]), 0) + 1
    print("wrote", path, len(cases), "cases;", kinds)


def gen_validation():
    cases = []

    def case(fn_name, model, kwargs):
        fn = getattr(B, fn_name)
        try:
            fn(Model(model), **kwargs)
            out = {"ok": True}
        except B.BatchError as e:
            out = {"kind": e.kind, "index": e.index, "detail": e.detail, "msg": str(e)}
        except Exception as e:  # noqa: BLE001
            out = {"exc": type(e).__name__, "msg": str(e)}
        cases.append({"fn": fn_name, "model": model, "kwargs": kwargs, "out": out})

    nan, inf = float("nan"), float("inf")
    base = dict(flag=["c", "p", "c", "p"], underlying=[100.0, 101.0, 99.0, 100.0],
                strike=[100.0, 95.0, 105.0, 110.0], t=[1.0, 0.5, 0.25, 2.0], r=[0.01, 0.02, 0.0, -0.01])
    for fn_name, extra in (("batch_price", {"sigma": [0.2, 0.3, 0.25, 0.4]}),
                           ("batch_greeks", {"sigma": [0.2, 0.3, 0.25, 0.4]}),
                           ("batch_iv", {"price": [8.0, 3.0, 2.0, 12.0]})):
        for model in ("black", "bs", "bsm"):
            kw = dict(base, **extra)
            if fn_name == "batch_iv":
                for method in ("lbr", "halley", "newton"):
                    k2 = dict(kw, method=method)
                    case(fn_name, model, k2)
                kw["method"] = "lbr"
            case(fn_name, model, kw)
            for col in ("underlying", "strike", "t", "r"):
                for bad in (nan, inf, -1.0, 0.0):
                    k2 = dict(kw)
                    v = list(k2[col]); v[2] = bad; k2[col] = v
                    case(fn_name, model, k2)
            k2 = dict(kw, q=[0.0, 0.01, 0.0, 0.0]); case(fn_name, model, k2)
            k2 = dict(kw, q=0.02); case(fn_name, model, k2)
            k2 = dict(kw, q=[0.0, nan, 0.0, 0.0]); case(fn_name, model, k2)
            k2 = dict(kw, flag=["c", "x", "p", "C"]); case(fn_name, model, k2)
            k2 = dict(kw, flag="P"); case(fn_name, model, k2)
            k2 = dict(kw, strike=[100.0, 95.0]); case(fn_name, model, k2)
            k2 = dict(kw, strike=[]); case(fn_name, model, k2)
            k2 = dict(kw, t=[1.0, nan, 0.5, 0.1], strike=[100.0, 95.0, -3.0, 1.0]); case(fn_name, model, k2)
            if fn_name != "batch_iv":
                k2 = dict(kw, sigma=[0.2, -0.1, 0.3, 0.2]); case(fn_name, model, k2)
                k2 = dict(kw, sigma=None); case(fn_name, model, k2)
            else:
                k2 = dict(kw, price=[1.0, nan, 2.0, 3.0]); case(fn_name, model, k2)
                k2 = dict(kw, price=None); case(fn_name, model, k2)
    path = os.path.join(HERE, "validation.json")
    with open(path, "w") as f:
        json.dump(cases, f, allow_nan=True)
    print("wrote", path, len(cases), "cases")


if __name__ == "__main__":
    main()
