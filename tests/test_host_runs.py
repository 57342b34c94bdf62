"""The host side of the run-length transport (fv_host_find_runs: the scan a
host-buffer call runs on its copy threads before shipping a chunk's column as
runs), on CPU against a numpy restatement: bit-pattern equality (-0.0 is not
0.0, NaN payloads are values), runs across the scan's part boundaries, the
exact budget (at most rows/64 runs goes, one more gives up), flag columns."""
import ctypes

import numpy as np
import pytest


@pytest.fixture(scope="module")
def lib():
    from paper_2604_27210_b200 import _native
    try:
        return _native.load()
    except _native.NativeUnavailable as exc:
        pytest.skip(str(exc))


def _want(col):
    bits = col.view(np.uint64) if col.dtype == np.float64 else col.view(np.uint8)
    starts = np.r_[0, np.flatnonzero(bits[1:] != bits[:-1]) + 1]
    return starts.astype(np.int32), bits[starts]


def _runs(lib, col, budget):
    n = col.size
    starts = np.full(budget + 2, -7, np.int32)
    vals = np.zeros(budget + 1, np.uint64 if col.dtype == np.float64 else np.uint8)
    nr = ctypes.c_int64()
    assert lib.fv_host_find_runs(col.ctypes.data, col.dtype.itemsize, n, budget, starts.ctypes.data,
                                 vals.ctypes.data, ctypes.byref(nr)) == 0
    if nr.value < 0:
        return None
    assert starts[nr.value] == n
    return starts[:nr.value], vals[:nr.value]


@pytest.mark.parametrize("n", [1, 7, 8, 9, 65_535, 65_536, 100_003, 1_000_000])
def test_runs_match_numpy(lib, n):
    rng = np.random.default_rng(n)
    vals = np.array([0.0, -0.0, 1.5, np.inf, -np.inf,
                     np.frombuffer(np.uint64(0x7ff8000000000001).tobytes(), np.float64)[0],
                     np.frombuffer(np.uint64(0x7ff8000000000002).tobytes(), np.float64)[0]])
    lens = rng.geometric(1.0 / 500, size=n // 10 + 2)
    col = np.repeat(vals[rng.integers(0, vals.size, lens.size)], lens)[:n]
    col = np.resize(col, n) if col.size < n else col
    want = _want(col)
    got = _runs(lib, col, max(1, want[0].size))                 # budget exactly the true count
    assert got is not None
    np.testing.assert_array_equal(got[0], want[0])
    np.testing.assert_array_equal(got[1], want[1])
    if want[0].size > 1:
        assert _runs(lib, col, want[0].size - 1) is None          # one short of it: gives up


def test_run_boundaries_on_part_edges(lib):
    """Runs that start exactly at, just before and just after the scan's part
    boundaries (parts of n/k rows, k = n >> 15 capped by the pool)."""
    n = 1 << 20
    col = np.zeros(n)
    v = 1.0
    for edge in range(1 << 15, n, 1 << 15):
        for e in (edge - 1, edge, edge + 1):
            col[e:] = v
            v += 1.0
    want = _want(col)
    got = _runs(lib, col, want[0].size)
    np.testing.assert_array_equal(got[0], want[0])
    np.testing.assert_array_equal(got[1], want[1])


def test_flags_and_distinct_values(lib):
    n = 300_000
    fl = np.where(np.arange(n) < 123_457, 1, -1).astype(np.int8)
    got = _runs(lib, fl, n // 64)
    np.testing.assert_array_equal(got[0], [0, 123_457])
    np.testing.assert_array_equal(got[1].view(np.int8), [1, -1])
    rnd = np.random.default_rng(1).uniform(size=n)
    assert _runs(lib, rnd, n // 64) is None
