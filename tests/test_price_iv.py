"""Price -> IV round trip (fv_price_iv / batch.price_iv) and
the bench-harness mirror (paper_2604_27210_b200/bench.py).

The round trip must equal the reference's two calls in sequence --
batch_price(model, ..., sigma) then batch_iv(model, method, ..., price=<that
column>) -- bit for bit, with the same exception: batch_price's errors first,
then the method check, then batch_iv's.  Pinned by tests/golden/bench_chain.npz
(the reference's synthetic_chain + batch_iv + run_bench, gen_bench.py), by the
oracle on seeded workloads, and against our own batch_price -> batch_iv (each
pinned to the reference by test_gpu_parity.py) on the fuzzed exception rows."""
import io
import json
import os
import contextlib

import numpy as np
import pytest

from _helpers import assert_bits, load
from conftest import GOLDEN

IV_NAMES = np.array(["converged", "fell_back_to_bisection", "below_intrinsic",
                     "above_upper_bound", "max_iterations"], dtype=object)


def test_bench_draws_match_reference_generator():
    """bench._draws restates synthetic_chain's generator calls (bench.py:21-28)."""
    from paper_2604_27210_b200 import bench
    g = load(os.path.join(GOLDEN, "bench_chain.npz"))
    flag, S, K, t, r, q, sigma = bench._draws(int(g["rows"]), int(g["seed"]))
    assert (np.where(flag == "c", 1, -1) == g["flag"]).all()
    for name, got in (("S", S), ("K", K), ("t", t), ("r", r), ("q", q), ("sigma", sigma)):
        assert_bits(got, g[name], name)


def test_price_iv_declared_and_bound():
    from paper_2604_27210_b200 import _native
    lib = _native.load()
    assert lib.fv_price_iv.restype is not None
    import paper_2604_27210_b200 as fv
    assert callable(fv.price_iv) and callable(fv.bench.run_roundtrip)


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def fv():
    import paper_2604_27210_b200 as fv
    from paper_2604_27210_b200 import _native
    _native.lib_for_compute()
    return fv


@pytest.fixture(scope="module")
def oracle_mod():
    from oracle import fvoracle
    fvoracle.lib()
    return fvoracle


def _price_iv_native(model, method, cols, device, region=True):
    """fv_price_iv with host or device pointers: (rc, ep, ei, price, iv, status, region)."""
    from paper_2604_27210_b200 import _native
    lib = _native.lib_for_compute()
    n = len(cols[0])
    cols = [np.ascontiguousarray(cols[0], np.int8)] + [np.ascontiguousarray(c, np.float64)
                                                       for c in cols[1:]]
    ep, ei = _native.fv_error(), _native.fv_error()
    if device:
        import torch
        dcols = [torch.from_numpy(c).cuda() for c in cols]
        px = torch.empty(n, dtype=torch.float64, device="cuda")
        iv = torch.empty(n, dtype=torch.float64, device="cuda")
        st = torch.empty(n, dtype=torch.int8, device="cuda")
        reg = torch.empty(n, dtype=torch.int8, device="cuda")
        rc = lib.fv_price_iv(model, method, *[_native.col(c) for c in dcols], n, px.data_ptr(),
                             iv.data_ptr(), st.data_ptr(), reg.data_ptr() if region else None, ep, ei)
        return (rc, ep, ei, px.cpu().numpy(), iv.cpu().numpy(), st.cpu().numpy(),
                reg.cpu().numpy() if region else None)
    px = np.empty(n)
    iv = np.empty(n)
    st = np.empty(n, np.int8)
    reg = np.empty(n, np.int8)
    rc = lib.fv_price_iv(model, method, *[_native.col(c) for c in cols], n, px.ctypes.data,
                         iv.ctypes.data, st.ctypes.data, reg.ctypes.data if region else None, ep, ei)
    return rc, ep, ei, px, iv, st, (reg if region else None)


@pytest.mark.gpu
@pytest.mark.parametrize("device", [True, False])
@pytest.mark.parametrize("model,mname,method,mcode", [
    (2, "bsm", "halley", 0), (2, "bsm", "lbr", 1), (0, "black", "lbr", 1), (0, "black", "halley", 0),
    (1, "bs", "lbr", 1)])
def test_round_trip_vs_oracle(fv, oracle_mod, device, model, mname, method, mcode):
    import workloads as W
    flag, S, K, t, r, q, sig = W.chain_draws(150_001, seed=21 + model)
    if model != 2:
        q = np.zeros_like(S)
    want_p = oracle_mod.rows_price(mname, flag, S, K, t, r, q, sig)
    assert not want_p["exc"].any()
    want = oracle_mod.rows_iv(mname, method, flag, S, K, t, r, q, want_p["price"])
    rc, ep, ei, px, iv, st, reg = _price_iv_native(model, mcode, (flag, S, K, t, r, q, sig), device)
    assert rc == 0, (ep.message, ei.message)
    assert_bits(px, want_p["price"], "price")
    assert_bits(st, want["status_code"], "status")
    assert_bits(iv, want["iv"], "iv")
    if method == "lbr":
        assert_bits(reg, want["region"], "region")


@pytest.mark.gpu
def test_round_trip_host_chunks_and_broadcast(fv):
    """Host pipeline over many chunks (chunk rows not a multiple of anything)
    with broadcast r / q / sigma columns equals the device-resident call."""
    from paper_2604_27210_b200 import _native
    import workloads as W
    lib = _native.load()
    n = 300_001
    flag, S, K, t, r, q, sig = W.chain_draws(n, seed=5)
    cols = (flag, S, K, t, np.array([0.02]), np.array([0.01]), np.array([0.35]))
    lib.fv_set_chunk_rows(65_537)
    try:
        a = _price_iv_native(2, 1, cols, False)
    finally:
        lib.fv_set_chunk_rows(1 << 22)
    full = (flag, S, K, t, np.full(n, 0.02), np.full(n, 0.01), np.full(n, 0.35))
    b = _price_iv_native(2, 1, full, True)
    assert a[0] == 0 and b[0] == 0, (a[1].message, a[2].message, b[1].message)
    for j, what in ((3, "price"), (4, "iv"), (5, "status"), (6, "region")):
        assert_bits(a[j], b[j], what + " host vs device")


@pytest.mark.gpu
def test_python_round_trip_equals_two_calls(fv):
    import workloads as W
    flag, S, K, t, r, q, sig = W.chain_draws(70_000, seed=9)
    fl = W.flag_chars(flag)
    for method in ("halley", "lbr"):
        tb = fv.price_iv("bsm", method, fl, S, K, t, r, q, sigma=sig)
        p = fv.batch_price("bsm", fl, S, K, t, r, q, sigma=sig)["price"]
        ref = fv.batch_iv("bsm", method, fl, S, K, t, r, price=p, q=q)
        assert list(tb.columns) == ["flag", "underlying", "strike", "t", "r", "q", "sigma",
                                    "price", "iv", "status"]
        assert_bits(tb["price"], p, "price")
        assert_bits(tb["iv"], ref["iv"], method + " iv")
        assert (tb["status"] == ref["status"]).all()
        assert tb["status"].dtype == object


def _outcome(fn):
    try:
        tb = fn()
        return {"price": tb["price"][0], "iv": tb["iv"][0], "status": str(tb["status"][0])}
    except Exception as e:  # noqa: BLE001
        return {"exc": type(e).__name__, "msg": str(e)}


@pytest.mark.gpu
def test_round_trip_exceptions_match_two_calls(fv):
    """Every fuzzed extreme row of exceptions.json: the fused call raises what
    batch_price -> batch_iv raises (price errors first), else the same bits."""
    cases = json.load(open(os.path.join(GOLDEN, "exceptions.json")))
    kinds = {"price_exc": 0, "iv_exc": 0, "ok": 0}
    for c in cases:
        a = c["in"]
        m = a["model"]
        base = ([("c" if a["flag"] > 0 else "p")], [a["underlying"]], [a["strike"]], [a["t"]],
                [a["r"]])
        for method in ("lbr", "halley"):
            got = _outcome(lambda: fv.price_iv(m, method, *base, [a["q"]], sigma=[a["sigma"]]))

            def two():
                p = fv.batch_price(m, *base, [a["q"]], sigma=[a["sigma"]])["price"]
                tb = fv.batch_iv(m, method, *base, price=p, q=[a["q"]])
                tb.columns["price"] = p
                return tb
            try:
                fv.batch_price(m, *base, [a["q"]], sigma=[a["sigma"]])
                price_ok = True
            except Exception:  # noqa: BLE001
                price_ok = False
            want = _outcome(two)
            kinds["ok" if "exc" not in want else ("iv_exc" if price_ok else "price_exc")] += 1
            if "exc" in want:
                assert got == want, (method, a, got, want)
            else:
                assert "exc" not in got, (method, a, got, want)
                assert got["status"] == want["status"], (method, a, got, want)
                assert np.float64(got["iv"]).tobytes() == np.float64(want["iv"]).tobytes() or (
                    np.isnan(got["iv"]) and np.isnan(want["iv"])), (method, a, got, want)
                assert np.float64(got["price"]).tobytes() == np.float64(want["price"]).tobytes()
    assert min(kinds.values()) > 50, kinds


@pytest.mark.gpu
def test_round_trip_error_order_in_a_batch(fv):
    """Several failing rows in one batch: a price-stage exception at a later
    row beats an IV-stage exception at an earlier one; validation beats both;
    a bad method is reported only once the prices succeeded."""
    n = 6000
    F = np.full(n, 100.0)
    K = np.full(n, 100.0)
    t = np.full(n, 1.0)
    r = np.zeros(n)
    sig = np.full(n, 0.2)
    fl = ["c"] * n
    # IV stage raises at row 1000: a price above the LBR upper bound cannot come
    # from the pricer, so use a row the LBR solver rejects with an exception --
    # take one from the fuzzed set
    cases = json.load(open(os.path.join(GOLDEN, "exceptions.json")))
    iv_row = None
    for c in cases:
        a = c["in"]
        if a["model"] != "black":
            continue
        try:
            p = fv.batch_price("black", ["c" if a["flag"] > 0 else "p"], [a["underlying"]],
                               [a["strike"]], [a["t"]], [a["r"]], sigma=[a["sigma"]])["price"]
        except Exception:  # noqa: BLE001
            continue
        try:
            fv.batch_iv("black", "lbr", ["c" if a["flag"] > 0 else "p"], [a["underlying"]],
                        [a["strike"]], [a["t"]], [a["r"]], price=p)
        except Exception as e:  # noqa: BLE001
            iv_row = (a, type(e), str(e))
            break
    assert iv_row is not None
    a, iv_exc, iv_msg = iv_row
    fl[1000] = "c" if a["flag"] > 0 else "p"
    F[1000], K[1000], t[1000], r[1000], sig[1000] = (a["underlying"], a["strike"], a["t"], a["r"],
                                                     a["sigma"])
    with pytest.raises(iv_exc) as e1:
        fv.price_iv("black", "lbr", fl, F, K, t, r, sigma=sig)
    assert str(e1.value) == iv_msg
    r2 = r.copy()
    r2[3000] = -1000.0               # exp(-r t) overflows in the pricer: OverflowError
    with pytest.raises(OverflowError, match="math range error"):
        fv.price_iv("black", "lbr", fl, F, K, t, r2, sigma=sig)
    with pytest.raises(OverflowError, match="math range error"):
        fv.price_iv("black", "nope", fl, F, K, t, r2, sigma=sig)
    sig2 = sig.copy()
    sig2[5000] = -0.1
    with pytest.raises(fv.BatchError) as e3:
        fv.price_iv("black", "lbr", fl, F, K, t, r2, sigma=sig2)
    assert (e3.value.kind, e3.value.index) == ("DomainError", 5000)
    with pytest.raises(fv.BatchError, match="unknown IV method"):
        fv.price_iv("black", "nope", fl, F, K, t, r, sigma=sig)


@pytest.mark.gpu
def test_round_trip_sharded_over_devices(fv):
    """Two host shards on device 0: same bits, and the merged error is the
    price stage's when it failed in either shard."""
    from paper_2604_27210_b200 import _native
    import workloads as W
    n = 2_400_000
    flag, S, K, t, r, q, sig = W.chain_draws(n, seed=31)
    fl = W.flag_chars(flag)
    one = fv.price_iv("bsm", "lbr", fl, S, K, t, r, q, sigma=sig)
    _native.set_devices((0, 0))
    try:
        two = fv.price_iv("bsm", "lbr", fl, S, K, t, r, q, sigma=sig)
        r2 = r.copy()
        r2[2_000_000] = -1e4          # price stage overflow in the second shard
        with pytest.raises(OverflowError, match="math range error"):
            fv.price_iv("bsm", "lbr", fl, S, K, t, r2, q, sigma=sig)
    finally:
        _native.set_devices(())
    for c in ("price", "iv"):
        assert np.array_equal(one[c].view(np.int64), two[c].view(np.int64)), c
    assert (one["status"] == two["status"]).all()


@pytest.mark.gpu
def test_bench_mirror_matches_reference(fv, tmp_path):
    """synthetic_chain prices, batch_iv results and run_bench's report equal the
    reference's (tests/golden/bench_chain.npz); run_roundtrip agrees."""
    from paper_2604_27210_b200 import bench
    g = load(os.path.join(GOLDEN, "bench_chain.npz"))
    rows, seed = int(g["rows"]), int(g["seed"])
    flag, S, K, t, r, q, sigma, price = bench.synthetic_chain(rows, seed)
    assert_bits(price, g["price"], "synthetic_chain price")
    for method in ("halley", "lbr"):
        tb = fv.price_iv("bsm", method, flag, S, K, t, r, q, sigma=sigma)
        assert_bits(tb["price"], g["price"], "round-trip price")
        assert_bits(tb["iv"], g[f"{method}_iv"], f"{method} iv")
        assert (tb["status"] == IV_NAMES[g[f"{method}_status"]]).all()
        for runner in (bench.run_bench, bench.run_roundtrip):
            out = tmp_path / f"{method}.csv"
            assert runner(rows, method, str(out), None, seed) == 0
            head, line = out.read_text().strip().splitlines()
            cells = line.split(",")
            assert head == str(g[f"{method}_report_head"])
            assert [cells[0], cells[1], cells[4]] == list(g[f"{method}_report_cells"])
            assert float(cells[3]) > 0
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            bench.run_bench(rows, method, None, None, seed)
        assert buf.getvalue().splitlines()[0] == str(g[f"{method}_report_head"])


@pytest.mark.gpu
def test_round_trip_edge_shapes(fv):
    """Empty and one-row batches, broadcast-only inputs, a dividend on a
    non-BSM model (batch_price's DomainError), a missing sigma."""
    empty = fv.price_iv("bsm", "lbr", [], [], [], [], [], [], sigma=[])
    assert empty["iv"].shape == (0,) and empty["status"].shape == (0,)
    one = fv.price_iv("black", "halley", ["p"], [100.0], [90.0], [0.5], [0.01], sigma=[0.3])
    p = fv.batch_price("black", ["p"], [100.0], [90.0], [0.5], [0.01], sigma=[0.3])["price"]
    ref = fv.batch_iv("black", "halley", ["p"], [100.0], [90.0], [0.5], [0.01], price=p)
    assert one["price"].tobytes() == p.tobytes() and one["iv"].tobytes() == ref["iv"].tobytes()
    n = 5
    bc = fv.price_iv("bsm", "lbr", ["c"] * n, 100.0, np.linspace(80, 120, n), 1.0, 0.02, 0.01,
                     sigma=0.25)
    p = fv.batch_price("bsm", ["c"] * n, 100.0, np.linspace(80, 120, n), 1.0, 0.02, 0.01, sigma=0.25)["price"]
    ref = fv.batch_iv("bsm", "lbr", ["c"] * n, 100.0, np.linspace(80, 120, n), 1.0, 0.02, price=p, q=0.01)
    assert bc["iv"].tobytes() == ref["iv"].tobytes()
    with pytest.raises(fv.BatchError) as e:
        fv.price_iv("bs", "lbr", ["c"] * n, 100.0, np.linspace(80, 120, n), 1.0, 0.02, 0.01, sigma=0.25)
    with pytest.raises(fv.BatchError) as e2:
        fv.batch_price("bs", ["c"] * n, 100.0, np.linspace(80, 120, n), 1.0, 0.02, 0.01, sigma=0.25)
    assert str(e.value) == str(e2.value)
    with pytest.raises(fv.BatchError, match="batch_price requires sigma"):
        fv.price_iv("bsm", "lbr", ["c"], [100.0], [100.0], [1.0], [0.0])


@pytest.mark.gpu
@pytest.mark.parametrize("method,mcode", [("halley", 0), ("lbr", 1)])
def test_round_trip_full_10m(fv, oracle_mod, method, mcode):
    """BASELINE size for the round trip (the bench workload rt): the whole
    10M-row C2 draw set priced and inverted in one device-resident
    fv_price_iv call equals batch_price then batch_iv on every row (price, iv,
    status bits); a strided 1-in-100 sample is bit-compared with the oracle;
    the host-pointer call is bit-identical to the device-resident one."""
    import sys
    import torch
    from conftest import REPO
    if REPO not in sys.path:
        sys.path.insert(0, REPO)
    import bench
    from paper_2604_27210_b200 import _native
    lib = _native.lib_for_compute()
    dev = torch.device("cuda", 0)
    n = 10_000_000
    cols = bench.draws_device("c2", n, 0, dev)
    ncols = bench.native_cols(cols, "sigma")
    px = torch.empty(n, dtype=torch.float64, device=dev)
    iv = torch.empty(n, dtype=torch.float64, device=dev)
    st = torch.empty(n, dtype=torch.int8, device=dev)
    ep, ei = _native.fv_error(), _native.fv_error()
    assert lib.fv_price_iv(2, mcode, *ncols, n, px.data_ptr(), iv.data_ptr(), st.data_ptr(), None,
                           ep, ei) == 0, (ep.message, ei.message)
    px2 = bench.price_on_device(lib, 2, cols, n)
    cols2 = dict(cols, price=px2)
    iv2 = torch.empty(n, dtype=torch.float64, device=dev)
    st2 = torch.empty(n, dtype=torch.int8, device=dev)
    err = _native.fv_error()
    assert lib.fv_batch_iv(2, mcode, *bench.native_cols(cols2, "price"), n, iv2.data_ptr(), st2.data_ptr(),
                           None, err) == 0, err.message
    torch.cuda.synchronize()
    assert torch.equal(px.view(torch.int64), px2.view(torch.int64))
    assert torch.equal(iv.view(torch.int64), iv2.view(torch.int64))
    assert torch.equal(st, st2)
    idx = torch.arange(0, n, 100, device=dev)
    samp = {k: cols[k][idx].cpu().numpy() for k in ("flag", "underlying", "strike", "t", "r", "q", "sigma")}
    wp = oracle_mod.rows_price("bsm", samp["flag"], samp["underlying"], samp["strike"], samp["t"], samp["r"],
                               samp["q"], samp["sigma"])
    assert_bits(px[idx].cpu().numpy(), wp["price"], "rt-10M sample price")
    want = oracle_mod.rows_iv("bsm", method, samp["flag"], samp["underlying"], samp["strike"], samp["t"],
                              samp["r"], samp["q"], wp["price"])
    assert_bits(st[idx].cpu().numpy(), want["status_code"], "rt-10M sample status")
    assert_bits(iv[idx].cpu().numpy(), want["iv"], "rt-10M sample iv")
    hcols = {k: (v.cpu().pin_memory() if v.numel() > 1 else v.cpu()) for k, v in cols.items() if torch.is_tensor(v)}
    hpx = torch.empty(n, dtype=torch.float64).pin_memory()
    hiv = torch.empty(n, dtype=torch.float64).pin_memory()
    hst = torch.empty(n, dtype=torch.int8).pin_memory()
    assert lib.fv_price_iv(2, mcode, *bench.native_cols(hcols, "sigma"), n, hpx.data_ptr(), hiv.data_ptr(),
                           hst.data_ptr(), None, ep, ei) == 0, (ep.message, ei.message)
    assert torch.equal(hpx.view(torch.int64), px.cpu().view(torch.int64))
    assert torch.equal(hiv.view(torch.int64), iv.cpu().view(torch.int64))
    assert torch.equal(hst, st.cpu())


@pytest.mark.gpu
def test_price_iv_sharded_single_rank(fv):
    """distributed.price_iv_sharded without a process group (one rank) equals
    price_iv; a price-stage exception comes back as stage 0's outcome."""
    import torch
    from paper_2604_27210_b200 import distributed as D
    import workloads as W
    flag, S, K, t, r, q, sig = W.chain_draws(50_001, seed=23)
    ref = fv.price_iv("bsm", "halley", W.flag_chars(flag), S, K, t, r, q, sigma=sig)
    cols = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in
            dict(flag=flag, underlying=S, strike=K, t=t, r=r, q=q, sigma=sig).items()}
    out, outcome = D.price_iv_sharded("bsm", "halley", cols, len(flag))
    assert outcome is None
    assert_bits(out["price"].cpu().numpy(), ref["price"], "sharded price")
    assert_bits(out["iv"].cpu().numpy(), ref["iv"], "sharded iv")
    r2 = r.copy()
    r2[777] = -1e4                   # exp(-r t) overflows in the pricer
    cols["r"] = torch.from_numpy(r2).cuda()
    out, outcome = D.price_iv_sharded("bsm", "halley", cols, len(flag))
    assert outcome == (0, ("exc", 1, 777)), outcome
