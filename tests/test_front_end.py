"""The drop-in front end (paper_2604_27210_b200.batch) reproduces the
reference's pre-kernel semantics on CPU: flag parsing (vectorised, same
BadFlag row/repr), broadcasting / ShapeMismatch, method and missing-column
errors -- checked against the reference's own outputs in
tests/golden/validation.json.  Errors found inside the fused GPU pass
(NonFiniteInput, DomainError) are covered by tests/test_gpu_parity.py."""
import json
import os

import numpy as np
import pytest

import paper_2604_27210_b200 as fv
from paper_2604_27210_b200 import batch as B
from conftest import GOLDEN

PRE_DEVICE = ("BadFlag", "ShapeMismatch")


def _cases():
    return json.load(open(os.path.join(GOLDEN, "validation.json")))


def test_pre_device_validation_matches_reference():
    n = 0
    for c in _cases():
        out = c["out"]
        pre = out.get("kind") in PRE_DEVICE or "requires" in out.get("detail", "") \
            or "unknown IV method" in out.get("detail", "")
        if not pre:
            continue
        kw = dict(c["kwargs"])
        try:
            getattr(fv, c["fn"])(c["model"], **kw)
            got = {"ok": True}
        except fv.BatchError as e:
            got = {"kind": e.kind, "index": e.index, "detail": e.detail, "msg": str(e)}
        except Exception as e:  # the missing-column cases validate first (device)
            got = {"exc": type(e).__name__}
        if got.get("exc") == "NativeUnavailable":
            continue
        assert got == out, (c, got)
        n += 1
    assert n > 20


@pytest.mark.parametrize("flags,want", [
    (["c", "C", "p", "P"], [1, 1, -1, -1]),
    (np.array(["p", "c"]), [-1, 1]),
    ("C", [1]),
    ([], []),
])
def test_parse_flags_values(flags, want):
    assert B.parse_flags(flags).tolist() == want


@pytest.mark.parametrize("flags,idx,rep", [
    (["c", "x"], 1, "'x'"),
    (np.array(["c", "p", "q"]), 2, "np.str_('q')"),
    (["c", 1], 1, "1"),
    (["c", None], 1, "None"),
    (np.array([b"c"]), 0, "np.bytes_(b'c')"),
    (["cc"], 0, "'cc'"),
])
def test_parse_flags_errors_match_reference_repr(flags, idx, rep):
    with pytest.raises(fv.BatchError) as ei:
        B.parse_flags(flags)
    assert ei.value.kind == "BadFlag" and ei.value.index == idx
    assert ei.value.detail == f"option flag must be 'c' or 'p', got {rep}"


def test_broadcast_rules():
    assert B.broadcast([1, 5, 1]) == 5
    assert B.broadcast([1, 0, 1]) == 0
    with pytest.raises(fv.BatchError) as ei:
        B.broadcast([3, 4])
    assert ei.value.kind == "ShapeMismatch" and ei.value.index == 0


def test_broadcast_columns_stay_stride0():
    n, table = B._assemble(fv.Model.BLACK76, ["c"] * 4, 100.0, [90.0, 95.0, 100.0, 105.0], 1.0, 0.0,
                           price=[12.0, 8.0, 5.0, 3.0])
    assert n == 4 and table["underlying"].strides[0] == 0
    keep, cols = B._columns(table, "price")
    assert cols[1].stride == 0 and cols[2].stride == 1


def test_worker_count_env(monkeypatch):
    monkeypatch.setenv("FASTVOL_THREADS", "0")
    with pytest.raises(fv.BatchError, match="FASTVOL_THREADS must be a positive integer"):
        B.worker_count()
    monkeypatch.setenv("FASTVOL_THREADS", "abc")
    with pytest.raises(fv.BatchError):
        B.worker_count()
    monkeypatch.setenv("FASTVOL_THREADS", "3")
    assert B.worker_count() == 3


def test_format_output_matches_reference_text():
    t = B.ChainTable({"flag": np.array([1, -1], np.int8), "iv": np.array([0.2, np.nan]),
                      "status": np.array(["converged", "below_intrinsic"], dtype=object)})
    assert B.format_output(t, "csv") == "flag,iv,status\nc,0.2,converged\np,nan,below_intrinsic\n"
    assert json.loads(B.format_output(t, "json")) == {"flag": ["c", "p"], "iv": [0.2, None],
                                                       "status": ["converged", "below_intrinsic"]}
