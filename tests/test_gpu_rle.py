"""Run-length transport of piecewise-constant host columns (fv_kernels.cu
find_runs_batch / k_expand_runs): a host-buffer call whose chunk holds a
column as a few runs of one value ships the runs and rebuilds the column in
HBM.  The
results, statuses and error records must be bit-identical to the
device-resident call on the same columns (and so to the oracle, which the
device path is pinned to), whatever the runs look like: boundaries on chunk
edges, -0.0 next to 0.0, NaN payloads, a run per 64 rows exactly at the
budget, and columns that fall back to plain copies."""
import os
import sys

import numpy as np
import pytest

from _helpers import assert_bits

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2604_27210_b200 import _native
    return _native.lib_for_compute()


def _runs(rng, n, mean_len, values):
    """A column of runs: lengths ~ geometric(mean_len), values cycling over `values`."""
    out = np.empty(n)
    i = 0
    k = 0
    while i < n:
        ln = int(rng.geometric(1.0 / mean_len))
        out[i:i + ln] = values[k % len(values)]
        i += ln
        k += 1
    return out


def _call(lib, kind, cols, n, host, pinned=False):
    import torch
    from paper_2604_27210_b200 import _native
    if host:
        hc = [torch.from_numpy(np.ascontiguousarray(c)) for c in cols]
        if pinned:
            hc = [c.pin_memory() for c in hc]
        outs = [torch.empty(n, dtype=torch.float64) for _ in range(6)]
        st = torch.empty(n, dtype=torch.int8)
        if pinned:
            outs = [o.pin_memory() for o in outs]
            st = st.pin_memory()
    else:
        hc = [torch.from_numpy(np.ascontiguousarray(c)).cuda() for c in cols]
        outs = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(6)]
        st = torch.empty(n, dtype=torch.int8, device="cuda")
    fc = [_native.col(c) for c in hc]
    e1, e2 = _native.fv_error(), _native.fv_error()
    if kind == "lbr":
        rc = lib.fv_batch_iv(0, 1, *fc, n, outs[0].data_ptr(), st.data_ptr(), None, e1)
        res = [outs[0]]
    else:
        rc = lib.fv_price_greeks(2, *fc, n, *[o.data_ptr() for o in outs], st.data_ptr(), e1, e2)
        res = outs
    torch.cuda.synchronize()
    h2d = lib.fv_last_h2d_bytes()
    got = [r.cpu().numpy().copy() for r in res] + [st.cpu().numpy().copy()]
    return rc, (e1.code, e1.kind, e1.index, e1.message), got, h2d


def _chain(n, seed, t_run=5_000):
    """C4-shaped rows: flag in two runs, t in runs of t_run, the strike ladder
    (t_run distinct strikes) repeated for every maturity (shipped whole)."""
    rng = np.random.default_rng(seed)
    flag = np.where(np.arange(n) < n // 2, 1, -1).astype(np.int8)
    t = np.repeat(np.linspace(0.02, 2.0, n // t_run + 1), t_run)[:n]
    ladder = 100.0 * np.exp(rng.uniform(-0.4, 0.4, t_run))
    K = ladder[np.arange(n) % t_run]
    return flag, t, K, rng


def test_chain_runs_shipped_and_bit_identical(lib, oracle):
    n = 1_000_000
    flag, t, K, rng = _chain(n, 1)
    F = np.full(1, 100.0)
    r = np.full(1, 0.03)
    q = np.zeros(1)
    sig = rng.uniform(0.05, 0.9, n)
    px = oracle.rows_price("black", flag, np.full(n, 100.0), K, t, np.full(n, 0.03), np.zeros(n), sig)["price"]
    cols = [flag, F, K, t, r, q, px]
    want = _call(lib, "lbr", cols, n, host=False)
    for pinned in (True, False):
        got = _call(lib, "lbr", cols, n, host=True, pinned=pinned)
        assert got[0] == want[0] == 0
        for a, b in zip(got[2], want[2]):
            assert_bits(a, b, "host (runs) vs device, pinned=%s" % pinned)
        assert got[3] < n * 16 + 64 * 1024, got[3]               # t and flag as runs: K and price whole
    o = oracle.rows_iv("black", "lbr", flag, np.full(n, 100.0), K, t, np.full(n, 0.03), np.zeros(n), px)
    assert_bits(want[2][0], o["iv"], "device vs oracle")


@pytest.mark.parametrize("chunk", [1 << 16, 98_304, 1 << 22])
def test_run_edges_signed_zero_nan(lib, chunk):
    """Runs straddling chunk edges, -0.0 next to 0.0 (r), NaN payloads in the
    sigma column (a NonFiniteInput error at the first NaN row): host and device
    calls agree on every output bit and on the error record."""
    n = 600_001
    rng = np.random.default_rng(7)
    flag = np.where(_runs(rng, n, 3000, [1.0, -1.0]) > 0, 1, -1).astype(np.int8)
    S = _runs(rng, n, 700, [100.0, 101.5, 99.25])
    K = 100.0 * np.exp(rng.uniform(-0.3, 0.3, n))
    t = _runs(rng, n, 4000, [0.25, 0.5, 1.0, 2.0])
    r = _runs(rng, n, 900, [0.0, -0.0, 0.01])
    q = np.zeros(n)
    sig = _runs(rng, n, 200, [0.2, 0.3, 0.45])
    cols = [flag, S, K, t, r, q, sig]
    want = _call(lib, "pg", cols, n, host=False)
    lib.fv_set_chunk_rows(chunk)
    try:
        got = _call(lib, "pg", cols, n, host=True)
        assert got[0] == want[0] and got[1] == want[1]
        for a, b in zip(got[2], want[2]):
            assert_bits(a, b, "price+greeks host (runs) vs device")
        assert got[3] < n * (1 + 6 * 8)
        # a NaN with a payload in a run: the error row and message must not move
        sig2 = sig.copy()
        nan = np.frombuffer(np.uint64(0x7ff8000000000123).tobytes(), np.float64)[0]
        sig2[400_000:400_500] = nan
        cols2 = [flag, S, K, t, r, q, sig2]
        w2 = _call(lib, "pg", cols2, n, host=False)
        g2 = _call(lib, "pg", cols2, n, host=True)
        assert w2[0] != 0 and g2[0] == w2[0] and g2[1] == w2[1], (g2[1], w2[1])
    finally:
        lib.fv_set_chunk_rows(1 << 22)


def test_budget_edge_and_fallback(lib):
    """Three chunks of 2^18 rows (budget 4096 runs each): a t column with
    exactly 4096 runs per chunk goes as runs; one more run in the middle chunk
    sends that chunk's t whole; both calls are bit-identical to the device."""
    chunk = 1 << 18
    n = 3 * chunk
    budget = chunk // 64
    rng = np.random.default_rng(3)
    flag = np.ones(n, np.int8)
    K = 100.0 * np.exp(rng.uniform(-0.3, 0.3, n))
    sig = np.full(n, 0.3)
    r = np.full(1, 0.02)
    q = np.zeros(1)
    S = np.full(1, 100.0)
    lib.fv_set_chunk_rows(chunk)
    try:
        for extra in (0, 1):
            t = np.empty(n)
            v = 0.1
            for c in range(3):
                runs = budget + (extra if c == 1 else 0)
                edges = np.sort(rng.choice(np.arange(1, chunk), runs - 1, replace=False)) + c * chunk
                for lo, hi in zip(np.r_[c * chunk, edges], np.r_[edges, (c + 1) * chunk]):
                    t[lo:hi] = v
                    v += 0.0001
            cols = [flag, S, K, t, r, q, sig]
            want = _call(lib, "pg", cols, n, host=False)
            got = _call(lib, "pg", cols, n, host=True)
            assert got[0] == want[0] == 0
            for a, b in zip(got[2], want[2]):
                assert_bits(a, b, "t runs per chunk = budget + %d" % extra)
            runs_bytes = 3 * (12 * budget + 64)              # t as runs in every chunk, sigma and flag 1 run
            if extra == 0:
                assert 8 * n < got[3] < 8 * n + runs_bytes + 1024, got[3]
            else:
                assert got[3] >= 8 * n + 8 * chunk, got[3]   # the middle chunk's t went whole
    finally:
        lib.fv_set_chunk_rows(1 << 22)


def test_random_columns_fall_back(lib):
    """Columns of distinct values ship whole: the byte count is the plain one."""
    n = 500_000
    rng = np.random.default_rng(5)
    flag = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
    cols = [flag, rng.uniform(90, 110, n), rng.uniform(80, 120, n), rng.uniform(0.1, 2, n),
            rng.uniform(0, 0.05, n), rng.uniform(0, 0.02, n), rng.uniform(0.1, 0.6, n)]
    want = _call(lib, "pg", cols, n, host=False)
    got = _call(lib, "pg", cols, n, host=True)
    for a, b in zip(got[2], want[2]):
        assert_bits(a, b, "random columns")
    assert got[3] >= n * (1 + 6 * 8)


def test_concurrent_host_calls_with_runs(lib):
    """Host calls from several threads at once (the C ABI releases the GIL via
    ctypes): run scans share the copy pool and its reused buffers, so every
    thread's result must still match its own device-resident call."""
    import threading
    n = 400_000
    results = {}

    def work(k):
        flag, t, K, rng = _chain(n, 100 + k, t_run=4_000 + 1_000 * k)
        S, r, q = np.full(1, 100.0), np.full(n, 0.01 * k), np.zeros(1)
        sig = np.repeat(rng.uniform(0.1, 0.5, n // 8_000 + 1), 8_000)[:n]
        cols = [flag, S, K, t, r, q, sig]
        want = _call(lib, "pg", cols, n, host=False)
        got = [_call(lib, "pg", cols, n, host=True) for _ in range(3)]
        results[k] = (want, got)

    threads = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert len(results) == 4
    for k, (want, got) in results.items():
        for g in got:
            assert g[0] == want[0] == 0
            for a, b in zip(g[2], want[2]):
                assert_bits(a, b, "thread %d" % k)


def test_outcome_block_rearmed_between_calls(lib):
    """The call's outcome block is read back and re-armed in place by the last
    kernel of each call (k_publish_status): a call that fails validation, or
    raises mid-batch, must not leak its failing rows into the next call's
    outcome -- alternate failing and clean calls on device and host pointers."""
    from paper_2604_27210_b200 import _native
    n = 50_000
    rng = np.random.default_rng(9)
    flag = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
    S, r, q = np.full(n, 100.0), np.full(n, 0.01), np.zeros(n)
    K = 100.0 * np.exp(rng.uniform(-0.3, 0.3, n))
    t = rng.uniform(0.1, 2.0, n)
    sig = rng.uniform(0.1, 0.6, n)
    bad_sig = sig.copy()
    bad_sig[31_337] = -1.0                                  # DomainError: negative sigma at row 31337
    clean = [flag, S, K, t, r, q, sig]
    broken = [flag, S, K, t, r, q, bad_sig]
    want = _call(lib, "pg", clean, n, host=False)
    assert want[0] == 0
    for host in (False, True, False, True):
        b = _call(lib, "pg", broken, n, host=host)
        assert b[0] == _native.FV_ERR_BATCH and b[1][2] == 31_337, b[1]
        g = _call(lib, "pg", clean, n, host=host)
        assert g[0] == 0 and g[1][0] == 0, g[1]
        for a, w in zip(g[2], want[2]):
            assert_bits(a, w, "clean call after a failing one (host=%s)" % host)
