"""Wide-domain fuzz: every entry point on the device against the CPU oracle,
bit for bit, far outside the benchmark distributions -- forwards and strikes
over 12 decades, maturities from 1e-8 to 100 years, rates of +-50 %, vols
from 1e-6 to 30, t = 0 and sigma = 0 edges, prices from deep below intrinsic
to above the cap.  This is where the straight-line routines' range flags and
the careful replays (fv_fast.h) earn their keep: every row must come out as
the reference computes it.

Rows on which the reference raises a Python exception are removed first (a
batch with one raises as a whole: tests/test_gpu_parity.py's exception tests
and the golden exception fixture cover them); every other row is compared --
values and NaN masks, statuses, LBR regions.
"""
import numpy as np
import pytest

from _helpers import assert_bits

pytestmark = pytest.mark.gpu

MODELS = {"black": 0, "bs": 1, "bsm": 2}


@pytest.fixture(scope="module")
def env():
    import torch
    from oracle import fvoracle as O
    from paper_2604_27210_b200 import _native
    lib = _native.lib_for_compute()
    dev = torch.device("cuda", 0)
    lib.fv_set_stream(torch.cuda.current_stream(dev).cuda_stream)
    return lib, dev, O


def wide_draws(n, seed, model):
    """60 % 'wide but solvable' rows (vols 1 % - 300 %, maturities 1e-4 - 30 y,
    log-moneyness ~ N(0, 0.6)), 40 % extreme rows (12 decades of forward,
    |log-moneyness| up to 12, t down to 1e-8 and 0, sigma down to 1e-6 and 0);
    forwards over 12 decades throughout."""
    rng = np.random.default_rng(seed)
    ext = rng.random(n) < 0.4
    flag = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
    un = 10.0 ** rng.uniform(-6, 6, n)
    lnk = np.where(ext & (rng.random(n) < 0.5), rng.uniform(-12, 12, n), rng.normal(0, 0.6, n))
    K = un * np.exp(lnk)
    t = np.where(ext, np.where(rng.random(n) < 0.05, 0.0, 10.0 ** rng.uniform(-8, 2, n)),
                 10.0 ** rng.uniform(-4, 1.5, n))
    r = np.where(rng.random(n) < 0.2, 0.0, np.where(ext, rng.uniform(-0.5, 0.5, n), rng.uniform(-0.05, 0.1, n)))
    q = np.where(ext, rng.uniform(-0.2, 0.5, n), rng.uniform(0.0, 0.06, n)) if model == "bsm" else np.zeros(n)
    sig = np.where(ext, np.where(rng.random(n) < 0.05, 0.0, 10.0 ** rng.uniform(-6, 1.5, n)),
                   10.0 ** rng.uniform(-2, 0.5, n))
    return flag, un, K, t, r, q, sig


def _keep(res):
    return np.asarray(res["exc"]) == 0


def _dev(dev, arrays):
    import torch
    return [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in arrays]


def _price_greeks_dev(lib, dev, model, cols):
    import torch
    from paper_2604_27210_b200 import _native
    n = cols[0].numel()
    outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(6)]
    st = torch.empty(n, dtype=torch.int8, device=dev)
    ep, eg = _native.fv_error(), _native.fv_error()
    rc = lib.fv_price_greeks(model, *[_native.col(c) for c in cols], n, *[o.data_ptr() for o in outs],
                             st.data_ptr(), ep, eg)
    assert rc == 0, (ep.message, eg.message)
    return [o.cpu().numpy() for o in outs], st.cpu().numpy()


def _iv_dev(lib, dev, model, method, cols):
    import torch
    from paper_2604_27210_b200 import _native
    n = cols[0].numel()
    iv = torch.empty(n, dtype=torch.float64, device=dev)
    st = torch.empty(n, dtype=torch.int8, device=dev)
    reg = torch.empty(n, dtype=torch.int8, device=dev)
    err = _native.fv_error()
    rc = lib.fv_batch_iv(model, method, *[_native.col(c) for c in cols], n, iv.data_ptr(), st.data_ptr(),
                         reg.data_ptr(), err)
    assert rc == 0, err.message
    return iv.cpu().numpy(), st.cpu().numpy(), reg.cpu().numpy()


@pytest.mark.parametrize("model", list(MODELS))
def test_fuzz_price_greeks(env, model):
    lib, dev, O = env
    flag, un, K, t, r, q, sig = wide_draws(2_000_000, 101 + MODELS[model], model)
    p = O.rows_price(model, flag, un, K, t, r, q, sig)
    g = O.rows_greeks(model, flag, un, K, t, r, q, sig)
    keep = _keep(p) & _keep(g)
    cols = [c[keep] for c in (flag, un, K, t, r, q, sig)]
    outs, st = _price_greeks_dev(lib, dev, MODELS[model], _dev(dev, cols))
    ctx = dict(zip(("flag", "un", "K", "t", "r", "q", "sigma"), cols))
    assert_bits(outs[0], p["price"][keep], f"{model} price", ctx)
    for j, name in enumerate(("delta", "gamma", "theta", "rho", "vega"), start=1):
        assert_bits(outs[j], g[name][keep], f"{model} {name}", ctx)
    assert (st == g["status_code"][keep]).all(), f"{model} greeks status"
    assert keep.mean() > 0.9


@pytest.mark.parametrize("method", ["lbr", "halley"])
@pytest.mark.parametrize("model", list(MODELS))
def test_fuzz_iv(env, model, method):
    lib, dev, O = env
    rows = 2_000_000 if method == "lbr" else 600_000
    flag, un, K, t, r, q, sig = wide_draws(rows, 211 + 7 * MODELS[model] + (method == "lbr"), model)
    rng = np.random.default_rng(5 + MODELS[model])
    p = O.rows_price(model, flag, un, K, t, r, q, sig)
    keep = _keep(p)
    flag, un, K, t, r, q, sig = [c[keep] for c in (flag, un, K, t, r, q, sig)]
    px = p["price"][keep]
    # quotes: the model price, perturbed prices, and prices below intrinsic /
    # above the cap / zero / tiny
    kind = rng.integers(0, 6, px.size)
    pert = px * (1.0 + rng.normal(0, 1e-3, px.size))
    cap = np.where(flag > 0, un, K) * 1.5
    px = np.select([kind == 0, kind == 1, kind == 2, kind == 3, kind == 4],
                   [px, pert, px * 1e-6, cap, px * rng.uniform(0, 1, px.size)], default=px)
    want = O.rows_iv(model, method, flag, un, K, t, r, q, px)
    ok = _keep(want)
    cols = [c[ok] for c in (flag, un, K, t, r, q, px)]
    iv, st, reg = _iv_dev(lib, dev, MODELS[model], 1 if method == "lbr" else 0, _dev(dev, cols))
    ctx = dict(zip(("flag", "un", "K", "t", "r", "q", "price"), cols))
    assert (st == want["status_code"][ok]).all(), \
        f"{model} {method} status: {int((st != want['status_code'][ok]).sum())} rows differ"
    assert_bits(iv, want["iv"][ok], f"{model} {method} iv", ctx)
    if method == "lbr":
        assert (reg == want["region"][ok]).all(), f"{model} lbr region"
    assert ok.mean() > 0.8
