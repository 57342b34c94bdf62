"""Parity on EVERY row at every BASELINE size:
the device-resident C-ABI call on the full workload, compared bit for bit with
the CPU oracle run on all host cores over the same rows -- IV values and NaN
masks, statuses, prices and all five Greeks, and no row where the reference
would have raised.

  C1  jackel_iv_black (LBR), 1M synthetic_chain(seed 0) Black-76 quotes
  C2  Halley BSM with dividend yield, 10M quotes
  C3  fused price + Greeks, 10M quotes, for BSM, BS and Black-76
  C4  LBR on the whole 100M-quote chain
  C5  the 10M-row wing-stress set, LBR and Halley
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def env():
    import torch
    import bench
    from paper_2604_27210_b200 import _native
    lib = _native.lib_for_compute()
    dev = torch.device("cuda", 0)
    lib.fv_set_stream(torch.cuda.current_stream(dev).cuda_stream)
    return lib, dev, bench


def _run(lib, bench, model, method, cols, n, want_greeks=False):
    """One device-resident call; returns the outputs as numpy."""
    import torch
    from paper_2604_27210_b200 import _native
    dev = cols["strike"].device
    if want_greeks:
        outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(6)]
        st = torch.empty(n, dtype=torch.int8, device=dev)
        ep, eg = _native.fv_error(), _native.fv_error()
        rc = lib.fv_price_greeks(model, *bench.native_cols(cols, "sigma"), n, *[o.data_ptr() for o in outs],
                                 st.data_ptr(), ep, eg)
        assert rc == 0, (ep.message, eg.message)
        names = ("price", "delta", "gamma", "theta", "rho", "vega")
        got = {k: o.cpu().numpy() for k, o in zip(names, outs)}
        got["status"] = st.cpu().numpy()
        return got
    iv = torch.empty(n, dtype=torch.float64, device=dev)
    st = torch.empty(n, dtype=torch.int8, device=dev)
    err = _native.fv_error()
    rc = lib.fv_batch_iv(model, method, *bench.native_cols(cols, "price"), n, iv.data_ptr(), st.data_ptr(),
                         None, err)
    assert rc == 0, err.message
    return {"iv": iv.cpu().numpy(), "status": st.cpu().numpy()}


def _oracle(bench, workload, cols, model_name=None, method_name=None):
    from oracle import fvoracle as O
    O.lib()
    O.set_threads(THREADS)
    h = {k: v.cpu().numpy() for k, v in cols.items()}
    a = [h[k] for k in ("flag", "underlying", "strike", "t", "r", "q")]
    if method_name is None:
        p = O.rows_price(model_name, *a, h["sigma"])
        g = O.rows_greeks(model_name, *a, h["sigma"])
        return {"price": p["price"], "delta": g["delta"], "gamma": g["gamma"], "theta": g["theta"],
                "rho": g["rho"], "vega": g["vega"], "status": g["status_code"],
                "exc": p["exc"].astype(np.int32) + g["exc"]}
    w = O.rows_iv(model_name, method_name, *a, h["price"])
    return {"iv": w["iv"], "status": w["status_code"], "exc": w["exc"].astype(np.int32)}


def _check(bench, got, want, what):
    bad = bench.parity_count(got, want)
    n = len(next(iter(got.values())))
    print(f"{what}: {n} rows checked, {bad} mismatches")
    assert bad == 0, f"{what}: {bad} of {n} rows differ from the oracle"
    return n


def test_c1_bench_config_every_row(env):
    """C1 exactly as bench.py runs it: synthetic_chain(1_000_000, seed=0) on
    Black-76 (q ignored), LBR."""
    lib, dev, bench = env
    cols = bench.draws_device("c1", 1_000_000, 0, dev)
    cols.pop("kind"), cols.pop("side")
    n = cols["flag"].numel()
    cols["price"] = bench.price_on_device(lib, 0, cols, n)
    got = _run(lib, bench, 0, 1, cols, n)
    assert _check(bench, got, _oracle(bench, "c1", cols, "black", "lbr"), "C1 1M LBR") == 1_000_000


def test_c2_every_row(env):
    lib, dev, bench = env
    cols = bench.draws_device("c2", 10_000_000, 0, dev)
    cols.pop("kind"), cols.pop("side")
    n = cols["flag"].numel()
    cols["price"] = bench.price_on_device(lib, 2, cols, n)
    got = _run(lib, bench, 2, 0, cols, n)
    assert _check(bench, got, _oracle(bench, "c2", cols, "bsm", "halley"), "C2 10M Halley") == n
    counts = np.bincount(got["status"].astype(np.int64), minlength=5).tolist()
    assert counts == [9558752, 376255, 64993, 0, 0], counts     # SURVEY 8(a) H1's mix


@pytest.mark.parametrize("model_name,code", [("bsm", 2), ("bs", 1), ("black", 0)])
def test_c3_every_row(env, model_name, code):
    """C3's 10M draws through the fused price + Greeks kernel, per model
    (q = 0 for the models that take no dividend)."""
    import torch
    lib, dev, bench = env
    cols = bench.draws_device("c3", 10_000_000, 0, dev)
    cols.pop("kind"), cols.pop("side")
    if code != 2:
        cols["q"] = torch.zeros(1, dtype=torch.float64, device=dev)
    n = cols["flag"].numel()
    got = _run(lib, bench, code, -1, cols, n, want_greeks=True)
    want = _oracle(bench, "c3", cols, model_name, None)
    assert _check(bench, got, want, f"C3 10M price+Greeks {model_name}") == n


@pytest.mark.parametrize("method_name,code", [("lbr", 1), ("halley", 0)])
def test_c5_every_row(env, method_name, code):
    """The wing-stress set at its BASELINE size (10M draws; rows that would
    only raise Python exceptions are dropped by the generator)."""
    import torch
    import workloads as W
    lib, dev, bench = env
    cols = bench.draws_device("c5", 10_000_000, 0, dev)
    kind, side = cols.pop("kind"), cols.pop("side")
    n = cols["flag"].numel()
    px = bench.price_on_device(lib, 0, cols, n).cpu().numpy()
    h = {k: cols[k].cpu().numpy() for k in ("flag", "underlying", "strike", "t", "r")}
    cols["price"] = torch.from_numpy(W.c5_prices(h["flag"], h["underlying"], h["strike"], h["t"], h["r"],
                                                 kind, side, px)).to(dev)
    got = _run(lib, bench, 0, code, cols, n)
    want = _oracle(bench, "c5", cols, "black", method_name)
    assert _check(bench, got, want, f"C5 {n} {method_name}") == n
    st = np.bincount(got["status"].astype(np.int64), minlength=5)
    assert st[2] > 0.3 * n and st[3] > 0.1 * n, st.tolist()     # below / above bound rows present


def test_c4_100m_every_row(env):
    """The whole 100M-quote C4 chain in one device-resident call, every row
    against the oracle on all host cores (~100 M LBR solves on the CPU)."""
    import workloads as W
    lib, dev, bench = env
    n = W.C4_ROWS
    cols = bench.c4_device(n, 0, dev)
    cols["price"] = bench.price_on_device(lib, 0, cols, n)
    got = _run(lib, bench, 0, 1, cols, n)
    cols.pop("sigma")
    want = _oracle(bench, "c4", cols, "black", "lbr")
    assert _check(bench, got, want, "C4 100M LBR") == W.C4_ROWS
    counts = np.bincount(got["status"].astype(np.int64), minlength=5).tolist()
    assert counts == [92467604, 0, 7532396, 0, 0], counts


def test_multi_round_calls_bit_identical(env):
    """Device calls split into several LBR classify/solve rounds and Halley
    chunks (fv_set_round_rows forces rounds of 2^16 / 2^15 rows on a 300k-row
    batch) are bit-identical to the single-round calls: the round loop of
    launch_iv (queue offsets, sub_args, per-round counters) is exercised."""
    lib, dev, bench = env
    cols = bench.draws_device("c2", 300_000, 9, dev)
    cols.pop("kind"), cols.pop("side")
    n = cols["flag"].numel()
    cols["price"] = bench.price_on_device(lib, 2, cols, n)
    one = {m: _run(lib, bench, 2, m, cols, n) for m in (0, 1)}
    assert lib.fv_set_round_rows(1 << 16, 1 << 15) == 0
    try:
        many = {m: _run(lib, bench, 2, m, cols, n) for m in (0, 1)}
    finally:
        assert lib.fv_set_round_rows(0, 0) == 0
    for m in (0, 1):
        for k in ("iv", "status"):
            assert np.array_equal(one[m][k].view(np.uint8), many[m][k].view(np.uint8)), (m, k)
    want = _oracle(bench, "c2", cols, "bsm", "halley")
    _check(bench, many[0], want, "multi-round Halley")
    assert lib.fv_set_round_rows(1 << 27, 1 << 27) != 0          # Halley chunks are int32-indexed
