"""CPU pre-check of the device per-quote code (csrc/fv_quote.h compiled for
the host): bit-identical to the live reference's golden outputs (IV + NaN
mask, status, LBR region, prices, Greeks), to the reference's exception
behaviour on fuzzed extreme rows, and the GPU's fused far-low solver
identical to the reference-order one.  The kernels compile this same header;
tests/test_gpu_parity.py re-checks everything on the B200."""
import ctypes
import glob
import json
import os
import sys

import numpy as np
import pytest

from _helpers import assert_bits, bits_equal, load
from conftest import GOLDEN

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "native"))
import build as native_build  # noqa: E402

MID = {"black": 0, "bs": 1, "bsm": 2}
P = ctypes.c_void_p


@pytest.fixture(scope="module")
def Q():
    return ctypes.CDLL(native_build.build("quote_hostcheck"))


def _p(a):
    return P(a.ctypes.data)


def _iv(Q, model, method, flag, un, k, t, r, q, px):
    n = len(flag)
    cols = [np.ascontiguousarray(flag, np.int8)] + [np.ascontiguousarray(c, np.float64)
                                                    for c in (un, k, t, r, q, px)]
    iv, st, reg = np.empty(n), np.empty(n, np.int8), np.empty(n, np.int8)
    exc, ev, en = np.empty(n, np.int8), np.empty(n), np.empty(n, np.int8)
    Q.qh_iv(MID[model], 1 if method == "lbr" else 0, *[_p(c) for c in cols], ctypes.c_int64(n),
            _p(iv), _p(st), _p(reg), _p(exc), _p(ev), _p(en))
    return iv, st, reg, exc, ev, en


FIX = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "lbr_*.npz"))
             + glob.glob(os.path.join(GOLDEN, "halley_c*.npz")))


@pytest.mark.parametrize("name", FIX)
def test_iv_golden(Q, name):
    g = load(os.path.join(GOLDEN, name))
    iv, st, reg, exc, _, _ = _iv(Q, str(g["model"]), str(g["method"]), g["flag"], g["underlying"],
                                 g["strike"], g["t"], g["r"], g["q"], g["price"])
    assert not exc.any()
    assert_bits(st, g["status"], name + " status")
    assert_bits(iv, g["iv"], name + " iv")
    if "region" in g:
        assert_bits(reg, g["region"], name + " region")


@pytest.mark.parametrize("model", ["bsm", "bs", "black"])
def test_price_greeks_golden(Q, model):
    g = load(os.path.join(GOLDEN, "price_greeks.npz"))
    n = len(g["flag"])
    q = g["q"] if model == "bsm" else np.zeros(n)
    cols = [np.ascontiguousarray(a) for a in (g["flag"], g["underlying"], g["strike"], g["t"], g["r"], q, g["sigma"])]
    pr, g5, st = np.empty(n), np.empty(5 * n), np.empty(n, np.int8)
    ep, eg = np.empty(n, np.int8), np.empty(n, np.int8)
    Q.qh_price_greeks(MID[model], *[_p(c) for c in cols], ctypes.c_int64(n), _p(pr), _p(g5), _p(st), _p(ep), _p(eg))
    g5 = g5.reshape(n, 5)
    assert_bits(pr, g[f"{model}_price"], "price")
    assert_bits(st, g[f"{model}_status"], "status")
    for j, nm in enumerate(("delta", "gamma", "theta", "rho", "vega")):
        assert_bits(g5[:, j], g[f"{model}_{nm}"], nm)
    pr2, ex = np.empty(n), np.empty(n, np.int8)
    Q.qh_price(MID[model], *[_p(c) for c in cols], ctypes.c_int64(n), _p(pr2), _p(ex))
    assert_bits(pr2, g[f"{model}_price"], "price-only kernel")


def test_exception_rows(Q):
    from oracle import fvoracle as O
    cases = json.load(open(os.path.join(GOLDEN, "exceptions.json")))
    by = {}
    for c in cases:
        by.setdefault(c["in"]["model"], []).append(c)
    checked = 0
    for m, cs in by.items():
        col = {k: np.array([c["in"][k] for c in cs]) for k in
               ("flag", "underlying", "strike", "t", "r", "q", "sigma", "price")}
        n = len(cs)
        base = [np.ascontiguousarray(a) for a in (col["flag"].astype(np.int8), col["underlying"],
                                                 col["strike"], col["t"], col["r"], col["q"])]
        sg = np.ascontiguousarray(col["sigma"])
        pr, g5, st = np.empty(n), np.empty(5 * n), np.empty(n, np.int8)
        ep, eg = np.empty(n, np.int8), np.empty(n, np.int8)
        Q.qh_price_greeks(MID[m], *[_p(c) for c in base], _p(sg), ctypes.c_int64(n), _p(pr), _p(g5), _p(st), _p(ep), _p(eg))
        g5 = g5.reshape(n, 5)
        res = {meth: _iv(Q, m, meth, *base, col["price"]) for meth in ("lbr", "halley")}
        for i, c in enumerate(cs):
            for key in ("price", "greeks", "lbr", "halley"):
                if key not in c:
                    continue
                want = c[key]
                if key == "price":
                    code, val, np_ = ep[i], 0.0, 0
                    gv = {"price": pr[i]}
                elif key == "greeks":
                    code, val, np_ = eg[i], 0.0, 0
                    gv = dict(zip(("delta", "gamma", "theta", "rho", "vega"), g5[i]))
                else:
                    iv, st2, _, exc, ev, en = res[key]
                    code, val, np_ = exc[i], ev[i], en[i]
                    gv = {"iv": iv[i], "status": list(O.IV_STATUS)[st2[i]]}
                if code:
                    e = O.exception_for(code, val, bool(np_))
                    name = "DomainError" if isinstance(e, O.OracleDomainError) else type(e).__name__
                    assert want.get("exc") == name and want.get("msg") == str(e), (key, c["in"], want, str(e))
                else:
                    assert "exc" not in want, (key, c["in"], want, gv)
                    for k, v in want.items():
                        assert (v == gv[k]) if isinstance(v, str) else bits_equal(gv[k], v), (key, c["in"], want, gv)
                checked += 1
    assert checked > 5000


def test_fused_far_low_matches_reference_order(Q):
    from oracle import fvoracle as O
    import workloads as W
    Q.qh_far_low_fused_check.restype = ctypes.c_int64
    flag, S, K, t, r, q, sig = W.chain_draws(100_000, seed=3)
    px = O.rows_price("black", flag, S, K, t, r, 0.0, sig)["price"]
    cols = [np.ascontiguousarray(a) for a in (flag, S, K, t, r, px)]
    nf = ctypes.c_int64(0)
    bad = Q.qh_far_low_fused_check(*[_p(c) for c in cols], ctypes.c_int64(len(flag)), ctypes.byref(nf))
    assert nf.value > 30_000 and bad == 0


@pytest.mark.parametrize("seed", [3, 4])
def test_straight_line_far_low_matches_careful(Q, seed):
    """fv_fast.h's far-low solver, host build: every quote it does not hand
    back to the careful solver is bit-identical to it (sigma, status,
    iterations), on C1-like draws and on the C4 chain."""
    from oracle import fvoracle as O
    import workloads as W
    Q.qh_far_low_fast_check.restype = ctypes.c_int64
    if seed == 3:
        flag, S, K, t, r, q, sig = W.chain_draws(100_000, seed=seed)
    else:
        import bench
        flag, S, K, t, r, sig, _ = bench.cpu_sample_c4(100_000)
    px = O.rows_price("black", flag, S, K, t, r, 0.0, sig)["price"]
    cols = [np.ascontiguousarray(a) for a in (flag, S, K, t, r, px)]
    nf, nb = ctypes.c_int64(0), ctypes.c_int64(0)
    bad = Q.qh_far_low_fast_check(*[_p(c) for c in cols], ctypes.c_int64(len(flag)),
                                  ctypes.byref(nf), ctypes.byref(nb))
    assert nf.value > 30_000 and bad == 0
    assert nb.value < nf.value // 100, (nb.value, nf.value)


@pytest.mark.parametrize("case", ["c1", "c4", "c5", "bsm"])
def test_straight_line_classify_matches_careful(Q, case):
    """fv_fast.h's first pass (normalize_quote, bounds, first anchor, far-low
    test): every row it does not flag reproduces the careful pass exactly
    (classification, outputs of finished rows, the state handed on)."""
    import workloads as W
    from oracle import fvoracle as O
    Q.qh_classify_fast_check.restype = ctypes.c_int64
    model, q = 0, None
    if case == "c1":
        flag, S, K, t, r, q, sig = W.chain_draws(100_000, seed=11)
        q = np.zeros_like(S)
        px = O.rows_price("black", flag, S, K, t, r, 0.0, sig)["price"]
    elif case == "bsm":
        flag, S, K, t, r, q, sig = W.chain_draws(100_000, seed=12)
        model = 2
        px = O.rows_price("bsm", flag, S, K, t, r, q, sig)["price"]
    elif case == "c4":
        import bench
        flag, S, K, t, r, sig, _ = bench.cpu_sample_c4(100_000)
        q = np.zeros_like(S)
        px = O.rows_price("black", flag, S, K, t, r, 0.0, sig)["price"]
    else:
        flag, S, K, t, r, sig, kind, side = W.c5_params(100_000, seed=5)
        q = np.zeros_like(S)
        px0 = O.rows_price("black", flag, S, K, t, r, 0.0, sig)["price"]
        px = W.c5_prices(flag, S, K, t, r, kind, side, px0)
    cols = [np.ascontiguousarray(a) for a in (flag, S, K, t, r, q, px)]
    nb = ctypes.c_int64(0)
    bad = Q.qh_classify_fast_check(ctypes.c_int(model), *[_p(c) for c in cols], ctypes.c_int64(len(flag)),
                                   ctypes.byref(nb))
    assert bad == 0
    assert nb.value < len(flag) // 20, nb.value


@pytest.mark.parametrize("model", [0, 1, 2])
def test_straight_line_price_greeks_match_careful(Q, model):
    """fv_fast.h's price and fused price+Greeks rows: every row they do not
    flag is bit-identical to the careful rows (all six outputs + status)."""
    import workloads as W
    Q.qh_price_greeks_fast_check.restype = ctypes.c_int64
    flag, S, K, t, r, q, sig = W.chain_draws(100_000, seed=30 + model)
    if model != 2:
        q = np.zeros_like(q)

    def check(cols):
        cols = [np.ascontiguousarray(a) for a in cols]
        nb = ctypes.c_int64(0)
        bad = Q.qh_price_greeks_fast_check(ctypes.c_int(model), *[_p(c) for c in cols],
                                           ctypes.c_int64(len(cols[0])), ctypes.byref(nb))
        return bad, nb.value

    bad, nb = check((flag, S, K, t, r, q, sig))
    assert bad == 0 and nb < len(flag) // 100, (bad, nb)
    # wings: deep ITM/OTM, tiny and long maturities, tiny vols (many of these
    # leave the straight-line domains and go to the careful rows)
    m = len(flag) // 3
    K[:m] = S[:m] * np.exp(np.linspace(-8, 8, m))
    t[m:2 * m] = 10.0 ** np.linspace(-8, 1.5, m)
    sig[2 * m:3 * m] = 10.0 ** np.linspace(-7, 0.7, m)
    bad, nb = check((flag, S, K, t, r, q, sig))
    assert bad == 0, bad


@pytest.mark.parametrize("case", ["c2", "black", "c5"])
def test_straight_line_halley_matches_careful(Q, case):
    """fv_fast.h's Halley step (fx_hsm_pre / fx_halley_f): every quote it does
    not flag ends with the careful solver's status and sigma bits."""
    from oracle import fvoracle as O
    import workloads as W
    Q.qh_halley_fast_check.restype = ctypes.c_int64
    if case == "c5":
        flag, S, K, t, r, sig, kind, side = W.c5_params(20_000, seed=5)
        q = np.zeros_like(S)
        model = 0
        px = W.c5_prices(flag, S, K, t, r, kind, side, O.rows_price("black", flag, S, K, t, r, 0.0, sig)["price"])
    else:
        flag, S, K, t, r, q, sig = W.chain_draws(20_000, seed=40)
        model = 2 if case == "c2" else 0
        if model == 0:
            q = np.zeros_like(q)
        px = O.rows_price("bsm" if model else "black", flag, S, K, t, r, q, sig)["price"]
    cols = [np.ascontiguousarray(a) for a in (flag, S, K, t, r, q, px)]
    nb = ctypes.c_int64(0)
    bad = Q.qh_halley_fast_check(ctypes.c_int(model), *[_p(c) for c in cols], ctypes.c_int64(len(flag)),
                                 ctypes.byref(nb))
    assert bad == 0
    if case != "c5":
        assert nb.value < len(flag) // 100, nb.value


@pytest.mark.parametrize("case", ["c1", "wide"])
def test_straight_line_near_matches_careful(Q, case):
    """fv_fast.h's near-region solver (Hermite guess + Householder(3) on the
    middle objective, all three normalized_black branches): every quote it
    does not flag is bit-identical to the careful solver."""
    from oracle import fvoracle as O
    import workloads as W
    Q.qh_near_fast_check.restype = ctypes.c_int64
    flag, S, K, t, r, q, sig = W.chain_draws(100_000, seed=50)
    if case == "wide":                     # deep strikes, long/short maturities, high vols
        rng = np.random.default_rng(51)
        K = S * np.exp(rng.uniform(-4, 4, len(S)))
        t = 10.0 ** rng.uniform(-3, 1.3, len(S))
        sig = rng.uniform(0.05, 3.0, len(S))
    px = O.rows_price("black", flag, S, K, t, r, 0.0, sig)["price"]
    cols = [np.ascontiguousarray(a) for a in (flag, S, K, t, r, px)]
    nn, nb = ctypes.c_int64(0), ctypes.c_int64(0)
    bad = Q.qh_near_fast_check(*[_p(c) for c in cols], ctypes.c_int64(len(flag)), ctypes.byref(nn),
                               ctypes.byref(nb))
    assert nn.value > 10_000 and bad == 0, (nn.value, bad)
    assert nb.value < nn.value // 20, (nb.value, nn.value)


@pytest.mark.parametrize("case", ["c1", "wide"])
def test_straight_line_anchor_rest_matches_careful(Q, case):
    """fv_fast.h's second anchor stage (b_c, then b_hi): same region and
    anchor values as the careful stage on every unflagged quote (the central
    anchor's erfcx argument is 0 up to rounding: erfcx's y100 == 100 case)."""
    from oracle import fvoracle as O
    import workloads as W
    Q.qh_anchor_rest_fast_check.restype = ctypes.c_int64
    flag, S, K, t, r, q, sig = W.chain_draws(100_000, seed=60)
    if case == "wide":
        rng = np.random.default_rng(61)
        K = S * np.exp(rng.uniform(-4, 4, len(S)))
        t = 10.0 ** rng.uniform(-3, 1.3, len(S))
        sig = rng.uniform(0.05, 3.0, len(S))
    px = O.rows_price("black", flag, S, K, t, r, 0.0, sig)["price"]
    cols = [np.ascontiguousarray(a) for a in (flag, S, K, t, r, px)]
    ns, nb = ctypes.c_int64(0), ctypes.c_int64(0)
    bad = Q.qh_anchor_rest_fast_check(*[_p(c) for c in cols], ctypes.c_int64(len(flag)), ctypes.byref(ns),
                                      ctypes.byref(nb))
    assert ns.value > 10_000 and bad == 0, (ns.value, bad)
    assert nb.value < ns.value // 20, (nb.value, ns.value)


def test_unified_erfc_matches_glibc(Q):
    """fx_erfc_u2: the four fdlibm erfc ranges through one rational form give
    glibc's bits (fv_erfc_i) and fx_erfc's range flags, for every argument
    class: each range and its edges, |x| < 2^-56, x < -6, |x| >= 28, inf, nan."""
    Q.qh_erfc_u_check.restype = ctypes.c_int64
    rng = np.random.default_rng(11)
    edges = np.array([0.0, -0.0, 2.0**-60, 2.0**-56, 0.25, 0.84375, 1.25, 1 / 0.35, 6.0, 28.0,
                      np.inf, np.nan, 1e-300, 5e-324])
    edges = np.concatenate([edges, np.nextafter(edges, np.inf), np.nextafter(edges, -np.inf)])
    x = np.concatenate([edges, -edges,
                        rng.uniform(-30, 30, 200_000),
                        rng.uniform(-1.5, 1.5, 200_000),
                        rng.standard_normal(200_000) * 4,
                        np.exp(rng.uniform(-40, 4, 100_000)) * rng.choice([-1, 1], 100_000)])
    x = np.ascontiguousarray(x[rng.permutation(len(x))])
    nb = ctypes.c_int64(0)
    assert Q.qh_erfc_u_check(_p(x), ctypes.c_int64(len(x)), ctypes.byref(nb)) == 0
    # flags are fx_erfc's (checked above): |x| beyond ~26.5 (exp underflow) and nan / inf
    assert nb.value < 3 * len(x) // 8


@pytest.mark.parametrize("case", ["c2", "wide", "c5"])
def test_halley_fp32_sign_matches_careful(Q, case):
    """fx_halley_sign (the bracket pass's fp32 sign of f(10), margin 1e-4 disc
    (F + K)) never decides a sign the careful f disagrees with; checked at
    sigma = 10 and at values where f is small (near the solution)."""
    from oracle import fvoracle as O
    import workloads as W
    Q.qh_halley_sign_check.restype = ctypes.c_int64
    rng = np.random.default_rng(21)
    if case == "c5":
        flag, S, K, t, r, sig, kind, side = W.c5_params(30_000, seed=5)
        q = np.zeros_like(S)
        model = 0
        px = W.c5_prices(flag, S, K, t, r, kind, side, O.rows_price("black", flag, S, K, t, r, 0.0, sig)["price"])
    else:
        flag, S, K, t, r, q, sig = W.chain_draws(30_000, seed=41)
        model = 2
        if case == "wide":
            t = 10.0 ** rng.uniform(-6, 2.5, len(t))
            K = S * np.exp(rng.uniform(-8, 8, len(K)))
            sig = 10.0 ** rng.uniform(-3, 0.9, len(sig))
        px = O.rows_price("bsm", flag, S, K, t, r, q, sig)["price"]
    sigmas = np.array([10.0, 20.0, 40.0, 80.0, 100.0, 5.0, 2.0, 1.0, 0.5, 0.2, 0.1, 0.05])
    cols = [np.ascontiguousarray(a) for a in (flag.astype(np.int8), S, K, t, r, q, px)]
    und = ctypes.c_int64(0)
    bad = Q.qh_halley_sign_check(ctypes.c_int(model), *[_p(c) for c in cols], ctypes.c_int64(len(flag)),
                                 _p(sigmas), ctypes.c_int(len(sigmas)), ctypes.byref(und))
    assert bad == 0
    assert und.value < len(flag) * len(sigmas) // 4
