"""The paper-name façade (paper_2604_27210_b200.fast_vollib): backend
resolution, output containers, argument order and the py_vollib patches --
host logic only (the compute is stood in for by the CPU oracle, test
infrastructure).  tests/test_gpu_parity.py runs the same entry points on the
device against the oracle."""
import json
import sys
import types

import numpy as np
import pytest

from paper_2604_27210_b200 import fast_vollib as FV
from paper_2604_27210_b200.batch import ChainTable


@pytest.fixture
def oracle_engine(monkeypatch):
    """Route the façade's batch calls through the CPU oracle (no GPU here)."""
    from oracle import fvoracle as O
    from paper_2604_27210_b200.batch import _assemble
    from paper_2604_27210_b200.models import as_model
    O.lib()
    names = {"black": "black", "bs": "bs", "bsm": "bsm"}
    calls = []

    def price(model, flag, und, K, t, r, q=0.0, sigma=None):
        m = as_model(model)
        n, tb = _assemble(m, flag, und, K, t, r, q, sigma=sigma)
        calls.append(("price", m.value))
        out = O.rows_price(names[m.value], tb["flag"], tb["underlying"], tb["strike"], tb["t"], tb["r"],
                           tb["q"], tb["sigma"])["price"]
        return ChainTable(dict(tb, price=out))

    def iv(model, method, flag, und, K, t, r, price=None, q=0.0):
        m = as_model(model)
        n, tb = _assemble(m, flag, und, K, t, r, q, price=price)
        calls.append(("iv", m.value, method))
        res = O.rows_iv(names[m.value], method, tb["flag"], tb["underlying"], tb["strike"], tb["t"], tb["r"],
                        tb["q"], tb["price"])
        st = np.array(["converged", "fell_back_to_bisection", "below_intrinsic", "above_upper_bound",
                       "max_iterations"], dtype=object)[res["status_code"]]
        return ChainTable(dict(tb, iv=res["iv"], status=st))

    def greeks(model, flag, und, K, t, r, q=0.0, sigma=None):
        m = as_model(model)
        n, tb = _assemble(m, flag, und, K, t, r, q, sigma=sigma)
        calls.append(("greeks", m.value))
        g = O.rows_greeks(names[m.value], tb["flag"], tb["underlying"], tb["strike"], tb["t"], tb["r"],
                          tb["q"], tb["sigma"])
        return ChainTable(dict(tb, **{k: g[k] for k in FV.GREEKS}))

    monkeypatch.setattr(FV, "_engine", lambda backend: FV.resolve_backend(backend))
    monkeypatch.setattr(FV, "batch_price", price)
    monkeypatch.setattr(FV, "batch_iv", iv)
    monkeypatch.setattr(FV, "batch_greeks", greeks)
    monkeypatch.setattr(FV.jackel, "batch_iv", iv)
    return calls


def test_backend_resolution(monkeypatch):
    FV.set_backend(None)
    monkeypatch.delenv(FV.ENV_BACKEND, raising=False)
    assert FV.get_backend() == "b200"
    monkeypatch.setenv(FV.ENV_BACKEND, "jax")
    with pytest.raises(FV.BackendUnavailable):
        FV.get_backend()
    FV.set_backend("cuda")                      # set_backend beats the environment
    assert FV.get_backend() == "b200"
    with pytest.raises(FV.BackendUnavailable):
        FV.resolve_backend("numpy")             # keyword beats both
    with pytest.raises(ValueError):
        FV.set_backend("tpu")
    FV.set_backend(None)


def test_no_cpu_fallback():
    from paper_2604_27210_b200._native import NativeUnavailable
    import paper_2604_27210_b200._native as N
    try:
        have_gpu = N.load().fv_device_count() > 0
    except NativeUnavailable:
        have_gpu = False
    if have_gpu:
        pytest.skip("a GPU is visible")
    with pytest.raises(NativeUnavailable):
        FV.fast_black("c", 100.0, 100.0, 1.0, 0.01, 0.2)


def test_paper_listing_round_trip(oracle_engine):
    """price three quotes, then invert them (the SPEC's
    acceptance example: IV recovers 0.2)."""
    flags = np.array(["c", "c", "p"])
    K = np.array([95, 100, 105])
    prices = FV.fast_black_scholes(flag=flags, S=100.0, K=K, t=0.25, r=0.05, sigma=0.20, return_as="numpy")
    assert prices.shape == (3,)
    iv = FV.fast_implied_volatility(price=prices, S=100.0, K=K, t=0.25, r=0.05, flag=flags, return_as="numpy")
    assert np.allclose(iv, 0.2, atol=1e-8)
    assert ("iv", "bs", "halley") in oracle_engine


def test_return_as_containers(oracle_engine):
    pd = pytest.importorskip("pandas")
    args = ("c", 100.0, np.array([90.0, 100.0, 110.0]), 0.5, 0.01, 0.25)
    df = FV.fast_black(*args)
    assert isinstance(df, pd.DataFrame) and list(df.columns) == ["Price"] and len(df) == 3
    s = FV.fast_black(*args, return_as="series")
    assert isinstance(s, pd.Series) and s.name == "Price"
    a = FV.fast_black(*args, return_as="numpy")
    assert isinstance(a, np.ndarray) and np.array_equal(a, df["Price"].to_numpy())
    d = FV.fast_black(*args, return_as="dict")
    assert list(d) == ["Price"]
    j = json.loads(FV.fast_black(*args, return_as="json"))
    assert j["Price"] == [float(x) for x in a]
    g = FV.get_all_greeks("p", 100.0, 95.0, 1.0, 0.02, 0.3, return_as="dataframe")
    assert list(g.columns) == ["delta", "gamma", "theta", "rho", "vega"]
    assert np.array_equal(FV.vectorized_vega("p", 100.0, 95.0, 1.0, 0.02, 0.3, return_as="numpy"),
                          g["vega"].to_numpy())
    a32 = FV.fast_black(*args, return_as="numpy", dtype=np.float32)
    assert a32.dtype == np.float32
    with pytest.raises(ValueError):
        FV.fast_black(*args, return_as="xml")


def test_models_and_argument_order(oracle_engine):
    from oracle import fvoracle as O
    flag = np.array(["c", "p"])
    F, K, t, r, sig = 100.0, np.array([95.0, 105.0]), 0.7, 0.03, 0.22
    px = FV.fast_black(flag, F, K, t, r, sig, return_as="numpy")
    # py_vollib order for Black-76 IV: (price, F, K, r, t, flag)
    iv = FV.fast_implied_volatility_black(px, F, K, r, t, flag, return_as="numpy")
    want = O.rows_iv("black", "halley", np.array([1, -1], np.int8), np.full(2, F), K, np.full(2, t),
                     np.full(2, r), 0.0, px)["iv"]
    assert np.array_equal(iv, want)
    # q given -> BSM (py_vollib_vectorized convention)
    FV.fast_implied_volatility(px, 100.0, K, t, r, flag, q=0.01, return_as="numpy")
    assert oracle_engine[-1] == ("iv", "bsm", "halley")
    lbr = FV.jackel.jackel_iv_black(px, F, K, t, r, flag)
    assert oracle_engine[-1] == ("iv", "black", "lbr") and lbr.shape == (2,)


def test_on_error(oracle_engine):
    px = np.array([1e-9, 5.0])                      # first row below intrinsic for a deep ITM call
    with pytest.warns(RuntimeWarning):
        FV.fast_implied_volatility(px, 100.0, np.array([50.0, 100.0]), 1.0, 0.0, "c", return_as="numpy")
    with pytest.raises(ValueError):
        FV.fast_implied_volatility(px, 100.0, np.array([50.0, 100.0]), 1.0, 0.0, "c", return_as="numpy",
                                   on_error="raise")
    out = FV.fast_implied_volatility(px, 100.0, np.array([50.0, 100.0]), 1.0, 0.0, "c", return_as="numpy",
                                     on_error="ignore")
    assert np.isnan(out[0]) and np.isfinite(out[1])


def _fake_py_vollib(monkeypatch):
    names = ["py_vollib", "py_vollib.black", "py_vollib.black_scholes", "py_vollib.black_scholes_merton",
             "py_vollib.black.implied_volatility", "py_vollib.black_scholes.implied_volatility",
             "py_vollib.black_scholes_merton.implied_volatility", "py_vollib.black.greeks",
             "py_vollib.black.greeks.analytical", "py_vollib.black_scholes.greeks",
             "py_vollib.black_scholes.greeks.analytical", "py_vollib.black_scholes_merton.greeks",
             "py_vollib.black_scholes_merton.greeks.analytical"]
    mods = {}
    for n in names:
        m = types.ModuleType(n)
        mods[n] = m
        monkeypatch.setitem(sys.modules, n, m)
    mods["py_vollib.black_scholes"].black_scholes = "upstream"
    return mods


def test_patch_py_vollib(monkeypatch, oracle_engine):
    mods = _fake_py_vollib(monkeypatch)
    undo = FV.patch_py_vollib()
    bs = mods["py_vollib.black_scholes"].black_scholes
    p = bs("c", 100.0, 100.0, 0.5, 0.01, 0.2)
    assert isinstance(p, float) and p > 0
    iv = mods["py_vollib.black_scholes.implied_volatility"].implied_volatility(p, 100.0, 100.0, 0.5, 0.01, "c")
    assert abs(iv - 0.2) < 1e-10
    d = mods["py_vollib.black_scholes_merton.greeks.analytical"].delta("p", 100.0, 90.0, 1.0, 0.01, 0.3, 0.02)
    assert -1.0 < d < 0.0
    undo()
    assert mods["py_vollib.black_scholes"].black_scholes == "upstream"
    assert not hasattr(mods["py_vollib.black"], "black")


def test_patch_py_vollib_vectorized(monkeypatch):
    m = types.ModuleType("py_vollib_vectorized")
    m.vectorized_black = "upstream"
    monkeypatch.setitem(sys.modules, "py_vollib_vectorized", m)
    undo = FV.patch_py_vollib_vectorized()
    assert m.vectorized_black is FV.fast_black and m.get_all_greeks is FV.get_all_greeks
    undo()
    assert m.vectorized_black == "upstream" and not hasattr(m, "get_all_greeks")


def test_patch_missing_upstream():
    if "py_vollib" in sys.modules or "py_vollib_vectorized" in sys.modules:
        pytest.skip("upstream present")
    with pytest.raises(ImportError):
        FV.patch_py_vollib()
    with pytest.raises(ImportError):
        FV.patch_py_vollib_vectorized()
