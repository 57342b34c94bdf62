"""Pin the CPU oracle (oracle/fvoracle.cpp) to the live reference's outputs
committed under tests/golden/ (made by tests/golden/gen_golden.py).  Every
comparison is bit-exact: IV values + NaN masks, status codes, LBR regions,
prices, Greeks, point values, per-row exceptions, BatchError texts."""
import glob
import json
import os

import numpy as np
import pytest

from _helpers import assert_bits, load
from conftest import GOLDEN

IV_FIXTURES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "lbr_*.npz"))
                     + glob.glob(os.path.join(GOLDEN, "halley_c*.npz")))


@pytest.mark.parametrize("name", IV_FIXTURES)
def test_iv_fixture_bit_exact(oracle, name):
    g = load(os.path.join(GOLDEN, name))
    model, method = str(g["model"]), str(g["method"])
    res = oracle.rows_iv(model, method, g["flag"], g["underlying"], g["strike"], g["t"],
                         g["r"], g["q"], g["price"])
    assert not res["exc"].any()
    ctx = {k: g[k] for k in ("flag", "underlying", "strike", "t", "r", "price")}
    assert_bits(res["status_code"], g["status"], f"{name} status", ctx)
    assert_bits(res["iv"], g["iv"], f"{name} iv", ctx)
    if "region" in g:
        assert_bits(res["region"], g["region"], f"{name} region", ctx)


def test_halley_grid_bit_exact(oracle):
    g = load(os.path.join(GOLDEN, "halley_grid.npz"))
    for m in ("black", "bs", "bsm"):
        res = oracle.rows_iv(m, "halley", g[f"{m}_flag"], g[f"{m}_underlying"], g[f"{m}_strike"],
                             g[f"{m}_t"], g[f"{m}_r"], g[f"{m}_q"], g[f"{m}_price"])
        assert_bits(res["status_code"], g[f"{m}_status"], f"halley grid {m} status")
        assert_bits(res["iv"], g[f"{m}_iv"], f"halley grid {m} iv")


@pytest.mark.parametrize("model", ["bsm", "bs", "black"])
def test_price_greeks_bit_exact(oracle, model):
    g = load(os.path.join(GOLDEN, "price_greeks.npz"))
    q = g["q"] if model == "bsm" else np.zeros_like(g["q"])
    args = (g["flag"], g["underlying"], g["strike"], g["t"], g["r"], q, g["sigma"])
    p = oracle.rows_price(model, *args)
    assert_bits(p["price"], g[f"{model}_price"], f"{model} price")
    gk = oracle.rows_greeks(model, *args)
    assert_bits(gk["status_code"], g[f"{model}_status"], f"{model} greeks status")
    for name in ("delta", "gamma", "theta", "rho", "vega"):
        assert_bits(gk[name], g[f"{model}_{name}"], f"{model} {name}")


def test_point_values_bit_exact(oracle):
    g = load(os.path.join(GOLDEN, "nb_points.npz"))
    nb = np.array([oracle.normalized_black(x, s)[0] for x, s in zip(g["nb_x"], g["nb_s"])])
    assert_bits(nb, g["nb"], "normalized_black", {"x": g["nb_x"], "s": g["nb_s"]})
    L = oracle.lib()
    assert_bits([L.orc_norm_cdf(float(v)) for v in g["cdf_x"]], g["cdf"], "norm_cdf")
    assert_bits([L.orc_inv_norm_cdf(float(v)) for v in g["icdf_p"]], g["icdf"], "inv_norm_cdf")


def test_normalized_black_branches_covered(oracle):
    g = load(os.path.join(GOLDEN, "nb_points.npz"))
    branches = {oracle.normalized_black(x, s)[1] for x, s in zip(g["nb_x"], g["nb_s"])}
    assert branches == {0, 1, 2, 3}


def _outcome_from_rows(oracle, res, i, keys):
    if res["exc"][i]:
        e = oracle.exception_for(res["exc"][i], res["exc_val"][i], bool(res["exc_np"][i]))
        name = "DomainError" if isinstance(e, oracle.OracleDomainError) else type(e).__name__
        return {"exc": name, "msg": str(e)}
    return {k: res[k][i] for k in keys}


def _same(a, b):
    if isinstance(a, float) or isinstance(b, float):
        a, b = float(a), float(b)
        return (np.isnan(a) and np.isnan(b)) or np.float64(a).view(np.int64) == np.float64(b).view(np.int64)
    return a == b


def test_exception_rows(oracle):
    """Per-row outcomes of fuzzed extreme rows: the same value, or the same
    exception type and message, as the reference."""
    cases = json.load(open(os.path.join(GOLDEN, "exceptions.json")))
    by_model = {}
    for c in cases:
        by_model.setdefault(c["in"]["model"], []).append(c)
    n_checked = 0
    for model, cs in by_model.items():
        col = {k: np.array([c["in"][k] for c in cs]) for k in
               ("flag", "underlying", "strike", "t", "r", "q", "sigma", "price")}
        flag = col["flag"].astype(np.int8)
        args = (flag, col["underlying"], col["strike"], col["t"], col["r"], col["q"])
        res = {
            "price": oracle.rows_price(model, *args, col["sigma"]),
            "greeks": oracle.rows_greeks(model, *args, col["sigma"]),
            "lbr": oracle.rows_iv(model, "lbr", *args, col["price"]),
            "halley": oracle.rows_iv(model, "halley", *args, col["price"]),
        }
        status_names = list(oracle.IV_STATUS)
        for i, c in enumerate(cs):
            for key in ("price", "greeks", "lbr", "halley"):
                if key not in c:
                    continue
                want = c[key]
                r = res[key]
                if r["exc"][i]:
                    e = oracle.exception_for(r["exc"][i], r["exc_val"][i], bool(r["exc_np"][i]))
                    name = "DomainError" if isinstance(e, oracle.OracleDomainError) else type(e).__name__
                    got = {"exc": name, "msg": str(e)}
                elif key == "price":
                    got = {"price": r["price"][i]}
                elif key == "greeks":
                    got = {g: r[g][i] for g in ("delta", "gamma", "theta", "rho", "vega")}
                else:
                    got = {"iv": r["iv"][i], "status": status_names[r["status_code"][i]]}
                assert set(got) == set(want), (key, c["in"], got, want)
                for k in want:
                    assert _same(got[k], want[k]), (key, c["in"], got, want)
                n_checked += 1
    assert n_checked > 5000


def test_validation_errors(oracle):
    cases = json.load(open(os.path.join(GOLDEN, "validation.json")))
    for c in cases:
        kw = dict(c["kwargs"])
        fn = getattr(oracle, c["fn"])
        try:
            fn(c["model"], **kw)
            got = {"ok": True}
        except oracle.OracleBatchError as e:
            got = {"kind": e.kind, "index": e.index, "detail": e.detail, "msg": str(e)}
        assert got == c["out"], (c, got)


@pytest.mark.parametrize("which,exc", [(0, ValueError), (1, OverflowError)])
def test_first_exception_row_wins_oracle(oracle, which, exc):
    from test_gpu_parity import first_exception_batch
    n, F, K, t, r, px = first_exception_batch(which)
    with pytest.raises(exc, match="math (domain|range) error"):
        oracle.batch_iv("black", "lbr", ["c"] * n, F, K, t, r, price=px)
