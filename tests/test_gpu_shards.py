"""One logical batch over several device-resident shards from one process
(fv_run_shards: one host thread per shard, each on its shard's device and
stream) and the gather to one device (fv_gather: NVLink peer copies).  On the
1-GPU pool every shard sits on device 0 -- the host threads, per-shard
dispatch and the outcome merge are the same code a multi-GPU box runs.
Bit-identical to the single call; errors are the single call's, at GLOBAL
rows."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import torch
    import bench
    from paper_2604_27210_b200 import _native
    lib = _native.lib_for_compute()
    dev = torch.device("cuda", 0)
    lib.fv_set_stream(torch.cuda.current_stream(dev).cuda_stream)
    cols = bench.draws_device("c2", 300_000, 11, dev)
    cols.pop("kind"), cols.pop("side")
    n = cols["flag"].numel()
    cols["price"] = bench.price_on_device(lib, 2, cols, n)
    return lib, dev, bench, cols, n


def _split(cols, bounds):
    """Shards as separate device allocations (clones), in row order."""
    out = []
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        out.append({k: (v[lo:hi].clone() if v.numel() > 1 else v.clone()) for k, v in cols.items()})
    return out


def _single_iv(lib, bench, cols, n, method):
    import torch
    from paper_2604_27210_b200 import _native
    iv = torch.empty(n, dtype=torch.float64, device=cols["strike"].device)
    st = torch.empty(n, dtype=torch.int8, device=cols["strike"].device)
    err = _native.fv_error()
    rc = lib.fv_batch_iv(2, method, *bench.native_cols(cols, "price"), n, iv.data_ptr(), st.data_ptr(), None, err)
    return rc, err, iv, st


@pytest.mark.parametrize("method", ["lbr", "halley"])
def test_device_shards_bit_identical_and_gathered(setup, method):
    import torch
    from paper_2604_27210_b200 import _native
    from paper_2604_27210_b200 import distributed as D
    lib, dev, bench, cols, n = setup
    rc, err, iv, st = _single_iv(lib, bench, cols, n, 1 if method == "lbr" else 0)
    assert rc == 0, err.message
    shards = _split(cols, [0, 70_001, 150_000, n])
    outs, rc2, e1, e2 = D.run_device_shards(_native.FV_KIND_IV, "bsm", method, shards)
    assert rc2 == 0, e1.message
    full_iv = D.gather_device([o["iv"] for o in outs], dev)
    full_st = D.gather_device([o["status"] for o in outs], dev)
    assert torch.equal(full_iv.view(torch.int64), iv.view(torch.int64))
    assert torch.equal(full_st, st)


def test_device_shards_price_greeks(setup):
    import torch
    from paper_2604_27210_b200 import _native
    from paper_2604_27210_b200 import distributed as D
    lib, dev, bench, cols, n = setup
    outs1 = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(6)]
    st1 = torch.empty(n, dtype=torch.int8, device=dev)
    ep, eg = _native.fv_error(), _native.fv_error()
    assert lib.fv_price_greeks(2, *bench.native_cols(cols, "sigma"), n, *[o.data_ptr() for o in outs1],
                               st1.data_ptr(), ep, eg) == 0
    shards = _split(cols, [0, 123_457, n])
    outs, rc, e1, e2 = D.run_device_shards(_native.FV_KIND_PRICE_GREEKS, "bsm", None, shards)
    assert rc == 0
    for j, name in enumerate(("price", "delta", "gamma", "theta", "rho", "vega")):
        g = D.gather_device([o[name] for o in outs], dev)
        assert torch.equal(g.view(torch.int64), outs1[j].view(torch.int64)), name


def test_device_shards_errors_at_global_rows(setup):
    """A non-finite price in the LAST shard and a negative t (a later check in
    the reference's order) in the first: the NonFiniteInput row wins, at its
    global index, exactly as the single call reports it."""
    import torch
    from paper_2604_27210_b200 import _native
    from paper_2604_27210_b200 import distributed as D
    lib, dev, bench, cols, n = setup
    bad = {k: v.clone() for k, v in cols.items()}
    bad["price"][250_000] = float("nan")
    bad["t"][10] = -1.0
    rc, err, _, _ = _single_iv(lib, bench, bad, n, 1)
    assert rc == _native.FV_ERR_BATCH and err.index == 250_000
    single = err.message
    outs, rc2, e1, e2 = D.run_device_shards(_native.FV_KIND_IV, "bsm", "lbr", _split(bad, [0, 100_000, n]))
    assert rc2 == _native.FV_ERR_BATCH and e1.index == 250_000, e1.message
    assert e1.message == single
    cr, er, ec = _native.last_outcome(lib)
    assert cr[6] == 250_000 and cr[9] == 10                    # merged check rows (non-finite price, t < 0), global


def test_gather_uneven_sources(setup):
    """fv_gather of sources of uneven size (one empty) in order."""
    import torch
    from paper_2604_27210_b200 import distributed as D
    lib, dev, bench, cols, n = setup
    parts = [torch.arange(k, dtype=torch.float64, device=dev) + 1000 * i for i, k in enumerate((5, 0, 17, 1))]
    g = D.gather_device(parts, dev)
    assert torch.equal(g, torch.cat(parts))


@pytest.mark.parametrize("case", ["neg_underlying", "nan_r", "dividend_black", "bad_flag", "neg_t_and_nan_k"])
def test_device_broadcast_column_checks_match_host(setup, case):
    """Device calls check broadcast (stride-0) columns in the kernels instead
    of reading them back to the host: the reported BatchError (check, row 0,
    message) is the host call's, also when a row-wise column fails a LATER
    check at an earlier row."""
    import torch
    from paper_2604_27210_b200 import _native
    lib, dev, bench, cols, n = setup
    m = 2000
    h = {k: (v[:m].cpu().numpy().copy() if v.numel() > 1 else v.cpu().numpy().copy()) for k, v in cols.items()}
    model = 2
    if case == "neg_underlying":
        h["underlying"] = np.array([-1.0])
    elif case == "nan_r":
        h["r"] = np.array([np.nan])
    elif case == "dividend_black":
        model = 0
        h["q"] = np.array([0.01])
    elif case == "bad_flag":
        h["flag"] = np.array([3], np.int8)
    else:
        h["t"] = np.array([-0.5])
        h["strike"][7] = np.nan
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in h.items()}
    res = []
    for src in (h, d):
        for method in (1, 0):
            iv = (torch.empty(m, dtype=torch.float64, device=dev) if src is d else np.empty(m))
            st = (torch.empty(m, dtype=torch.int8, device=dev) if src is d else np.empty(m, np.int8))
            err = _native.fv_error()
            rc = lib.fv_batch_iv(model, method, *bench.native_cols(src, "price"), m, _native.ptr(iv),
                                 _native.ptr(st), None, err)
            res.append((rc, err.kind, err.index, err.message))
    assert all(r == res[0] for r in res), res
    assert res[0][0] == _native.FV_ERR_BATCH
    if case == "neg_t_and_nan_k":
        assert res[0][2] == 7                    # NonFinite strike (earlier check) at row 7 beats t < 0 at row 0
    else:
        assert res[0][2] == 0
