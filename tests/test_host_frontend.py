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
