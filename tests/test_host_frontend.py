"""The batch front end's host loops (csrc/fv_host.cpp):
threaded flag parsing and status object columns must give exactly the
reference's results (batch.py:78-88 parse_flags, :217/:259 status arrays)."""
import importlib
import sys

import numpy as np
import pytest


@pytest.fixture(scope="module")
def H():
    from paper_2604_27210_b200 import _build
    _build.build_host()
    return importlib.import_module("paper_2604_27210_b200._fvhost")


def _ref_flags(flags):
    out = np.empty(len(flags), dtype=np.int8)
    for i, f in enumerate(flags):
        if f in ("c", "C"):
            out[i] = 1
        elif f in ("p", "P"):
            out[i] = -1
        else:
            return i, None
    return -1, out


@pytest.mark.parametrize("n", [1, 5, 70_000, 3_000_001])
def test_parse_flags_matches_reference_loop(H, n):
    rng = np.random.default_rng(n)
    fl = rng.choice(np.array(["c", "C", "p", "P"]), n)
    out, bad = H.parse_flags_u(fl)
    assert bad == -1
    np.testing.assert_array_equal(out, np.where(np.char.lower(fl) == "c", 1, -1).astype(np.int8))
    if n <= 70_000:
        assert _ref_flags(list(fl))[1].tolist() == out.tolist()


@pytest.mark.parametrize("badval", ["x", "cc", "", "c ", " p", "ć", "q"])
def test_parse_flags_first_bad_index(H, badval):
    n = 2_500_000
    fl = np.full(n, "p", dtype="U2")
    rng = np.random.default_rng(7)
    idx = np.sort(rng.choice(n, 5, replace=False))
    fl[idx] = badval
    out, bad = H.parse_flags_u(fl)
    assert bad == idx[0]
    # the package entry raises BadFlag at that row with the reference message
    from paper_2604_27210_b200.batch import BatchError, parse_flags
    with pytest.raises(BatchError) as ei:
        parse_flags(fl)
    assert ei.value.index == idx[0]
    assert str(ei.value) == f"BadFlag at row {idx[0]}: option flag must be 'c' or 'p', got {fl[idx[0]]!r}"


def test_status_objects_match_take(H):
    from paper_2604_27210_b200.solver import GREEK_STATUS_NAMES, IV_STATUS_NAMES
    rng = np.random.default_rng(3)
    for names in (IV_STATUS_NAMES, GREEK_STATUS_NAMES):
        for n in (0, 1, 100_000, 4_000_000):
            codes = rng.integers(0, len(names), n).astype(np.int8)
            got = H.status_objects(tuple(names), codes)
            want = np.array(names, dtype=object)[codes]
            assert got.dtype == object and got.shape == (n,)
            assert (got == want).all()
            if n:
                assert all(got[i] is names[codes[i]] for i in rng.integers(0, n, 100))


def test_status_objects_reference_counts(H):
    names = tuple("state_%d_%s" % (i, "z" * i) for i in range(3))   # not interned: mortal
    before = [sys.getrefcount(x) for x in names]
    codes = np.array([0, 1, 1, 2, 2, 2] * 200_000, dtype=np.int8)
    arr = H.status_objects(names, codes)
    after = [sys.getrefcount(x) for x in names]
    assert [a - b for a, b in zip(after, before)] == [200_000, 400_000, 600_000]
    del arr
    assert [sys.getrefcount(x) for x in names] == before


def test_status_objects_rejects_bad_codes(H):
    names = ("a_%d" % 1, "b_%d" % 2)
    before = [sys.getrefcount(x) for x in names]
    codes = np.zeros(3_000_000, dtype=np.int8)
    codes[2_000_000] = 5
    with pytest.raises(ValueError, match="row 2000000"):
        H.status_objects(names, codes)
    assert [sys.getrefcount(x) for x in names] == before


def test_repr_doubles_is_python_repr(H):
    """Shortest round-trip digits + CPython's 'r' layout, on random bit
    patterns (every exponent, subnormals, nan/inf) and typical values."""
    rng = np.random.default_rng(5)
    x = np.concatenate([
        rng.integers(0, 2**64, 300_000, dtype=np.uint64).view(np.float64),
        rng.standard_normal(100_000) * 10.0 ** rng.integers(-30, 30, 100_000),
        np.round(rng.uniform(0, 500, 50_000), 4),
        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e16, 1e15, 9999999999999998.0, 1e-4, 1e-5,
                  5e-324, 1.7976931348623157e308, 2.2250738585072014e-308, 1e22, 1e23, 0.1, 100.0]),
    ])
    assert H.repr_doubles(x) == [repr(float(v)) for v in x]


def _python_csv(table):
    from paper_2604_27210_b200 import batch as B
    saved, B._fvhost = B._fvhost, None
    try:
        return B.format_output(table, "csv")
    finally:
        B._fvhost = saved


def test_format_csv_matches_python_rules(H):
    from paper_2604_27210_b200 import batch as B
    from paper_2604_27210_b200.solver import IV_STATUS_NAMES
    rng = np.random.default_rng(9)
    n = 50_000
    iv = rng.uniform(0.05, 2.0, n)
    iv[rng.integers(0, n, 500)] = np.nan
    cols = {
        "flag": np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8),
        "underlying": np.broadcast_to(np.float64(100.0), (n,)),       # stride-0 broadcast column
        "strike": 100 * np.exp(rng.uniform(-0.6, 0.6, n)),
        "t": rng.uniform(1e-9, 30, n),
        "r": np.full(n, -0.0),
        "price": rng.integers(0, 2**64, n, dtype=np.uint64).view(np.float64),
        "iv": iv,
        "status": np.array(IV_STATUS_NAMES, dtype=object)[rng.integers(0, 5, n)],
    }
    t = B.ChainTable(cols)
    fast = B.format_output(t, "csv")
    assert fast == _python_csv(t)
    assert fast.startswith("flag,underlying,strike,t,r,price,iv,status\n")


def test_format_csv_falls_back_outside_fast_path(H):
    from paper_2604_27210_b200 import batch as B
    n = 2000
    odd = np.empty(n, dtype=object)
    odd[:] = [1.5, "x", 3] * (n // 3) + [2.0] * (n % 3)   # mixed objects: Python rules per cell
    t = B.ChainTable({"a": np.arange(n, dtype=np.float32), "b": odd, "c": np.zeros(n, dtype=bool)})
    assert H.format_csv(("a", "b", "c"), (t["a"], t["b"], t["c"])) is None
    assert B.format_output(t, "csv") == _python_csv(t)


@pytest.mark.parametrize("fmt", ["csv", "json", "plain"])
@pytest.mark.parametrize("fast", [True, False])
def test_format_output_reference_golden(fmt, fast):
    """format_output against the reference's own text (tests/golden/gen_format.py)."""
    import json
    import os
    from paper_2604_27210_b200 import batch as B
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "format_output.json")))
    cols = {}
    for k, v in g["columns"].items():
        if k == "flag":
            cols[k] = np.array(v, dtype=np.int8)
        elif k == "status":
            cols[k] = np.array(v, dtype=object)
        else:
            cols[k] = np.array([float.fromhex(x) for x in v])
    saved = B._fvhost
    if not fast:
        B._fvhost = None
    else:
        B._CSV_MIN_ROWS, saved_min = 1, B._CSV_MIN_ROWS
    try:
        text = B.format_output(B.ChainTable(cols), fmt)
    finally:
        B._fvhost = saved
        if fast:
            B._CSV_MIN_ROWS = saved_min
    assert text == g[fmt]


def test_format_json_matches_python_rules(H):
    from paper_2604_27210_b200 import batch as B
    from paper_2604_27210_b200.solver import GREEK_STATUS_NAMES
    rng = np.random.default_rng(19)
    n = 120_000
    v = rng.integers(0, 2**64, n, dtype=np.uint64).view(np.float64)
    cols = {"flag": np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8),
            "strike": 100 * np.exp(rng.uniform(-0.6, 0.6, n)), "vega": v,
            "status": np.array(GREEK_STATUS_NAMES, dtype=object)[rng.integers(0, 2, n)]}
    t = B.ChainTable(cols)
    fast = B.format_output(t, "json")
    saved, B._fvhost = B._fvhost, None
    try:
        slow = B.format_output(t, "json")
    finally:
        B._fvhost = saved
    assert fast == slow
    # outside the fast path: float32, a non-flag integer column, strings needing escapes
    for extra in ({"x": np.ones(n, np.float32)}, {"x": np.arange(n)},
                  {"x": np.array(['a"b', "ok"] * (n // 2), dtype=object)}):
        c2 = dict(cols, **extra)
        assert H.format_json(tuple('"%s"' % k for k in c2), tuple(c2.values()), 0) is None
