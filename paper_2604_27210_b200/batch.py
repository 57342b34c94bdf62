"""Drop-in replacement for the reference batch engine, fastvol/batch.py.

Same entry points, signatures, broadcasting, 'c'/'p' flag parsing, ChainTable
results, status strings, BatchError kinds/indices/messages and Python
exceptions as /root/reference/pkg/src/fastvol/batch.py:33-334.  What changes
is underneath: the reference's per-row Python ``fill`` loops run under
``_run_chunked`` (batch.py:166-178); here each batch is ONE call into the
C ABI (include/fastvol_b200.h), which validates and computes on the B200 in a
single fused pass.  There is no CPU fallback.
"""

import json
import math
import os
from dataclasses import dataclass
from typing import Dict, Sequence, Union

import numpy as np

from . import _native
from .errors import DomainError
from .models import Model, as_model
from .solver import GREEK_STATUS_NAMES, IV_STATUS_NAMES

ENV_THREADS = "FASTVOL_THREADS"
MIN_CHUNK = 1024
INPUT_COLUMNS = ("flag", "underlying", "strike", "t", "r", "q", "sigma", "price")
GREEK_COLUMNS = ("delta", "gamma", "theta", "rho", "vega")

_IV_STATUS = np.array(IV_STATUS_NAMES, dtype=object)
_GREEK_STATUS = np.array(GREEK_STATUS_NAMES, dtype=object)

try:                        # csrc/fv_host.cpp: threaded flag parsing / status columns
    from . import _fvhost
except ImportError:         # not built: the numpy forms below (same results)
    _fvhost = None
_HOST_MIN_ROWS = 1 << 16
_CSV_MIN_ROWS = 1024


def _status_column(table: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """``table[codes]`` as a fresh object array (batch.py:217, :259)."""
    if _fvhost is not None and codes.shape[0] >= _HOST_MIN_ROWS:
        return _fvhost.status_objects(tuple(table), codes)
    return table[codes]
_CHECK_KIND = ["BadFlag"] + ["NonFiniteInput"] * 6 + ["DomainError"] * 5
_CHECK_COLUMN = ["flag", "underlying", "strike", "t", "r", "q", None,
                 "underlying", "strike", "t", "sigma", "q"]


class BatchError(Exception):
    """Pre-kernel batch rejection; ``index`` is the first offending row
    (batch.py:33-40)."""

    def __init__(self, kind: str, index: int, detail: str):
        self.kind = kind
        self.index = index
        self.detail = detail
        super().__init__(f"{kind} at row {index}: {detail}")


@dataclass
class ChainTable:
    """Columnar batch of contracts (batch.py:43-62)."""

    columns: Dict[str, np.ndarray]

    def __post_init__(self):
        lengths = {c.shape[0] for c in self.columns.values()}
        if len(lengths) > 1:
            raise BatchError("ShapeMismatch", 0, f"column lengths differ: {sorted(lengths)}")

    @property
    def length(self) -> int:
        for col in self.columns.values():
            return col.shape[0]
        return 0

    def __getitem__(self, name: str) -> np.ndarray:
        return self.columns[name]


# ---------------------------------------------------------------------------
# front end (batch.py:65-148 semantics; validation runs fused on the device)
# ---------------------------------------------------------------------------
def broadcast(lengths: Sequence[int]) -> int:
    """Common batch length under scalar-extends-to-N rules (batch.py:65-75)."""
    n = max(lengths, default=1)
    if 0 in lengths:
        n = 0
    for i, length in enumerate(lengths):
        if length not in (1, n):
            raise BatchError("ShapeMismatch", i, f"length {length} incompatible with batch size {n}")
    return n


def _flag_error(i, f):
    return BatchError("BadFlag", i, f"option flag must be 'c' or 'p', got {f!r}")


def parse_flags(flags: Union[str, Sequence[str]]) -> np.ndarray:
    """Case-insensitive 'c'/'p' -> int8 +1/-1 (batch.py:78-88), vectorised for
    string arrays; the first bad element raises BadFlag with its repr."""
    if isinstance(flags, str):
        flags = [flags]
    arr = flags if isinstance(flags, np.ndarray) else None
    if arr is None:
        try:
            arr = np.asarray(flags)
        except (ValueError, TypeError):
            arr = None
    if arr is not None and arr.ndim == 1 and arr.dtype.kind in "US":
        if arr.dtype.kind == "S":              # bytes never compare equal to 'c'
            if len(arr):
                raise _flag_error(0, flags[0])
            return np.empty(0, dtype=np.int8)
        # UCS-4 code points: an element equals 'c' exactly when its first code
        # point is 'c' and any padding code points are 0.  x | 0x20 folds the
        # case of exactly c/C and p/P (integer compares, ~10x faster than
        # numpy string compares at 1e7 rows)
        n = arr.shape[0]
        if n == 0:
            return np.empty(0, dtype=np.int8)
        if _fvhost is not None and n >= _HOST_MIN_ROWS:
            out, bad = _fvhost.parse_flags_u(np.ascontiguousarray(arr))
            if bad >= 0:
                raise _flag_error(bad, flags[bad])
            return out
        cp = np.ascontiguousarray(arr).view(np.uint32).reshape(n, arr.dtype.itemsize // 4)
        low = cp[:, 0] | np.uint32(0x20)
        is_c = low == 0x63
        ok = is_c | (low == 0x70)
        if cp.shape[1] > 1:
            ok &= (cp[:, 1:] == 0).all(axis=1)
        if not ok.all():
            i = int(np.flatnonzero(~ok)[0])
            raise _flag_error(i, flags[i])
        out = is_c.view(np.int8) * np.int8(2)
        out -= np.int8(1)
        return out
    out = np.empty(len(flags), dtype=np.int8)
    for i, f in enumerate(flags):
        if f == "c" or f == "C":
            out[i] = 1
        elif f == "p" or f == "P":
            out[i] = -1
        else:
            raise _flag_error(i, f)
    return out


def _as_column(values, n: int, name: str) -> np.ndarray:
    arr = np.atleast_1d(np.asarray(values, dtype=np.float64))
    if arr.ndim != 1:
        raise BatchError("ShapeMismatch", 0, f"column {name} is not 1-D")
    if arr.shape[0] == 1 and n != 1:
        arr = np.broadcast_to(arr, (n,))
    if arr.shape[0] != n:
        raise BatchError("ShapeMismatch", 0, f"column {name} has length {arr.shape[0]}, expected {n}")
    return arr


def validate(table: Dict[str, np.ndarray]) -> None:
    """Host-side restatement of batch.py:104-124 (public helper; the batch
    entry points run the same checks fused into the GPU pass instead)."""
    for name, col in table.items():
        if col.dtype.kind != "f":
            continue
        bad = np.flatnonzero(~np.isfinite(col))
        if bad.size:
            raise BatchError("NonFiniteInput", int(bad[0]), f"column {name} is not finite")
    for name in ("underlying", "strike"):
        if name in table:
            bad = np.flatnonzero(~(table[name] > 0.0))
            if bad.size:
                raise BatchError("DomainError", int(bad[0]), f"column {name} must be positive")
    for name in ("t", "sigma"):
        if name in table:
            bad = np.flatnonzero(table[name] < 0.0)
            if bad.size:
                raise BatchError("DomainError", int(bad[0]), f"column {name} must be >= 0")


def _assemble(model: Model, flag, underlying, strike, t, r, q=0.0, sigma=None, price=None):
    """batch.py:127-148 up to (not including) validate: flags, lengths,
    columns.  Returns (n, table)."""
    theta = parse_flags(flag)
    raw = {"underlying": underlying, "strike": strike, "t": t, "r": r, "q": q}
    if sigma is not None:
        raw["sigma"] = sigma
    if price is not None:
        raw["price"] = price
    lengths = [theta.shape[0]] + [np.atleast_1d(np.asarray(v, dtype=np.float64)).shape[0]
                                  for v in raw.values()]
    n = broadcast(lengths)
    table = {"flag": theta if theta.shape[0] == n else np.broadcast_to(theta, (n,))}
    for name, values in raw.items():
        table[name] = _as_column(values, n, name)
    return n, table


def worker_count() -> int:
    """FASTVOL_THREADS validation kept for parity (batch.py:151-163); the GPU
    path does not use host worker threads."""
    env = os.environ.get(ENV_THREADS)
    if env is not None:
        try:
            w = int(env)
        except ValueError as exc:
            raise BatchError("DomainError", 0, f"{ENV_THREADS} must be a positive integer") from exc
        if w < 1:
            raise BatchError("DomainError", 0, f"{ENV_THREADS} must be a positive integer")
        return w
    return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# native dispatch
# ---------------------------------------------------------------------------
def _native_col(a):
    """A 1-D column for the C ABI: broadcast views become stride-0 columns
    (never materialised), other views are made contiguous."""
    if a.ndim == 1 and a.shape[0] > 1 and a.strides[0] == 0:
        return a, _native.fv_col(a.ctypes.data, 0)
    if a.ndim == 1 and a.shape[0] == 1:
        return a, _native.fv_col(a.ctypes.data, 0)
    c = np.ascontiguousarray(a)
    return c, _native.fv_col(c.ctypes.data, 1)


def _columns(table, last):
    keep, cols = [], []
    for name in ("flag", "underlying", "strike", "t", "r", "q", last):
        arr = table[name]
        if name == "flag":
            arr = np.asarray(arr, dtype=np.int8)
        a, c = _native_col(arr)
        keep.append(a)
        cols.append(c)
    return keep, cols


def _value_repr(err):
    return repr(np.float64(err.value)) if err.value_is_numpy else repr(float(err.value))


def _raise_for(err, table, last_name):
    """Turn an fv_error into the exception the reference raises."""
    if err.code == _native.FV_ERR_BATCH:
        kind = _CHECK_KIND[err.kind]
        col = _CHECK_COLUMN[err.kind] or last_name
        if err.kind == 0:
            raise BatchError("BadFlag", int(err.index), "option flag must be 'c' or 'p'")
        if kind == "NonFiniteInput":
            detail = f"column {col} is not finite"
        elif err.kind in (7, 8):
            detail = f"column {col} must be positive"
        elif err.kind in (9, 10):
            detail = f"column {col} must be >= 0"
        else:
            raise BatchError("DomainError", int(err.index),
                             f"model {table['__model__']} does not accept a dividend yield")
        raise BatchError(kind, int(err.index), detail)
    if err.code == _native.FV_ERR_PYEXC:
        k = err.kind
        if k == 1:
            raise OverflowError("math range error")
        if k == 2:
            raise ValueError("math domain error")
        if k == 3:
            raise ZeroDivisionError("float division by zero")
        if k == 4:
            raise OverflowError(34, "Numerical result out of range")
        if k == 5:
            raise DomainError("F and K must be positive")
        if k == 6:
            raise DomainError(f"atm_inverse requires beta in (0, 1), got {_value_repr(err)}")
        if k == 7:
            raise DomainError(f"inv_norm_cdf requires p in (0, 1), got {_value_repr(err)}")
        if k == 8:
            raise DomainError(f"normalized_black requires x <= 0, got {_value_repr(err)}")
        if k == 9:
            raise DomainError(f"normalized_black requires s > 0, got {_value_repr(err)}")
        if k == 10:
            raise DomainError(f"objective_branch requires s > 0, got {_value_repr(err)}")
    raise RuntimeError("fastvol_b200: " + err.message.decode(errors="replace"))


def _ok_or_raise(rc, err, table, model, last):
    """Reference order: validation BatchError (_assemble), then the
    FASTVOL_THREADS check (_run_chunked -> worker_count), then the first
    raising row's exception (fill)."""
    if rc == _native.FV_ERR_BATCH:
        table = dict(table)
        table["__model__"] = model.value
        _raise_for(err, table, last)
    worker_count()
    if rc != _native.FV_OK:
        _raise_for(err, table, last)


# ---------------------------------------------------------------------------
# public batch API (batch.py:181-280)
# ---------------------------------------------------------------------------
def batch_price(model, flag, underlying, strike, t, r, q=0.0, sigma=None) -> ChainTable:
    """Price every row; returns the input columns plus ``price``."""
    model = as_model(model)
    n, table = _assemble(model, flag, underlying, strike, t, r, q, sigma=sigma)
    if "sigma" not in table:
        validate_order_then(table, model, need="sigma")
        raise BatchError("DomainError", 0, "batch_price requires sigma")
    out = np.empty(n, dtype=np.float64)
    if n:
        lib = _native.lib_for_compute()
        keep, cols = _columns(table, "sigma")
        err = _native.fv_error()
        rc = lib.fv_batch_price(model.code, *cols, n, out.ctypes.data, err)
        _ok_or_raise(rc, err, table, model, "sigma")
    cols_out = dict(table)
    cols_out["price"] = out
    return ChainTable(cols_out)


def batch_iv(model, method: str, flag, underlying, strike, t, r, price=None, q=0.0) -> ChainTable:
    """Invert the price column row by row (Halley or LBR); failed rows carry
    NaN plus an in-band status string."""
    if method not in ("halley", "lbr"):
        raise BatchError("DomainError", 0, f"unknown IV method {method!r}")
    model = as_model(model)
    n, table = _assemble(model, flag, underlying, strike, t, r, q, price=price)
    if "price" not in table:
        validate_order_then(table, model, need="price")
        raise BatchError("DomainError", 0, "batch_iv requires price")
    iv = np.empty(n, dtype=np.float64)
    codes = np.empty(n, dtype=np.int8)
    if n:
        lib = _native.lib_for_compute()
        keep, cols = _columns(table, "price")
        err = _native.fv_error()
        rc = lib.fv_batch_iv(model.code, 1 if method == "lbr" else 0, *cols, n, iv.ctypes.data,
                             codes.ctypes.data, None, err)
        _ok_or_raise(rc, err, table, model, "price")
    cols_out = dict(table)
    cols_out["iv"] = iv
    cols_out["status"] = _status_column(_IV_STATUS, codes)
    return ChainTable(cols_out)


def price_iv(model, method: str, flag, underlying, strike, t, r, q=0.0, sigma=None) -> ChainTable:
    """Price -> IV round trip in one C-ABI call (``fv_price_iv``; SURVEY 8(f)
    rank 3): the reference's ``batch_price(model, ..., sigma=sigma)`` followed
    by ``batch_iv(model, method, ..., price=<that price column>, q=q)``, as its
    bench harness runs them (bench.py:19-40).  Returns the input columns
    (sigma included), then ``price``, ``iv`` and ``status``; values, statuses
    and the exception raised are those of the two reference calls in sequence
    (batch_price's errors first, then the method check, then batch_iv's)."""
    model = as_model(model)
    if method not in ("halley", "lbr"):
        batch_price(model, flag, underlying, strike, t, r, q, sigma=sigma)
        raise BatchError("DomainError", 0, f"unknown IV method {method!r}")
    n, table = _assemble(model, flag, underlying, strike, t, r, q, sigma=sigma)
    if "sigma" not in table:
        validate_order_then(table, model, need="sigma")
        raise BatchError("DomainError", 0, "batch_price requires sigma")
    price = np.empty(n, dtype=np.float64)
    iv = np.empty(n, dtype=np.float64)
    codes = np.empty(n, dtype=np.int8)
    if n:
        lib = _native.lib_for_compute()
        keep, cols = _columns(table, "sigma")
        ep, ei = _native.fv_error(), _native.fv_error()
        rc = lib.fv_price_iv(model.code, 1 if method == "lbr" else 0, *cols, n, price.ctypes.data,
                             iv.ctypes.data, codes.ctypes.data, None, ep, ei)
        if rc in (_native.FV_ERR_CUDA, _native.FV_ERR_ARG):
            _raise_for(ep, table, "sigma")
        _ok_or_raise(ep.code, ep, table, model, "sigma")          # batch_price
        iv_table = dict(table)
        iv_table["price"] = price
        _ok_or_raise(ei.code, ei, iv_table, model, "price")       # batch_iv
    cols_out = dict(table)
    cols_out["price"] = price
    cols_out["iv"] = iv
    cols_out["status"] = _status_column(_IV_STATUS, codes)
    return ChainTable(cols_out)


def batch_greeks(model, flag, underlying, strike, t, r, q=0.0, sigma=None) -> ChainTable:
    """All five Greeks per row; zero-vol / zero-time rows carry NaNs plus a
    ``step_function_edge`` status."""
    model = as_model(model)
    n, table = _assemble(model, flag, underlying, strike, t, r, q, sigma=sigma)
    if "sigma" not in table:
        validate_order_then(table, model, need="sigma")
        raise BatchError("DomainError", 0, "batch_greeks requires sigma")
    outs = {name: np.empty(n, dtype=np.float64) for name in GREEK_COLUMNS}
    codes = np.empty(n, dtype=np.int8)
    if n:
        lib = _native.lib_for_compute()
        keep, cols = _columns(table, "sigma")
        err = _native.fv_error()
        rc = lib.fv_batch_greeks(model.code, *cols, n, *[outs[g].ctypes.data for g in GREEK_COLUMNS],
                                 codes.ctypes.data, err)
        _ok_or_raise(rc, err, table, model, "sigma")
    cols_out = dict(table)
    cols_out.update(outs)
    cols_out["status"] = _status_column(_GREEK_STATUS, codes)
    return ChainTable(cols_out)


def validate_order_then(table, model, need):
    """A batch without its sigma/price column still runs the reference's
    validate() and dividend check first (batch.py:145-147 precede the
    'requires sigma/price' error)."""
    validate(table)
    if model is not Model.BLACK_SCHOLES_MERTON and np.any(table["q"] != 0.0):
        idx = int(np.flatnonzero(table["q"] != 0.0)[0])
        raise BatchError("DomainError", idx, f"model {model.value} does not accept a dividend yield")


# ---------------------------------------------------------------------------
# serialization (batch.py:287-334), unchanged semantics
# ---------------------------------------------------------------------------
def _cell_text(value) -> str:
    if isinstance(value, (float, np.floating)):
        return repr(float(value))
    if isinstance(value, (np.int8, np.integer, int)):
        return "c" if int(value) > 0 else "p"
    return str(value)


def _plain_text(value) -> str:
    if isinstance(value, (float, np.floating)):
        return f"{float(value):.8g}"
    if isinstance(value, (np.int8, np.integer, int)):
        return "c" if int(value) > 0 else "p"
    return str(value)


def _csv(table: ChainTable, names) -> str:
    if _fvhost is not None and table.length >= _CSV_MIN_ROWS:
        # threaded shortest-round-trip formatting (csrc/fv_host.cpp); None when
        # a column is outside its float64 / integer / str-object cases
        text = _fvhost.format_csv(tuple(names), tuple(np.asarray(table[c]) for c in names))
        if text is not None:
            return text
    cols = [table[c] for c in names]
    rows = (",".join(_cell_text(col[i]) for col in cols) for i in range(table.length))
    return "\n".join([",".join(names), *rows]) + "\n"


def _json(table: ChainTable, names) -> str:
    if _fvhost is not None and table.length >= _CSV_MIN_ROWS:
        text = _fvhost.format_json(tuple(json.dumps(n) for n in names),
                                   tuple(np.asarray(table[c]) for c in names),
                                   names.index("flag") if "flag" in names else -1)
        if text is not None:
            return text
    obj = {}
    for name in names:
        col = table[name]
        if col.dtype.kind == "f":
            obj[name] = [float(v) if math.isfinite(v) else None for v in col]
        elif name == "flag":
            obj[name] = ["p" if v <= 0 else "c" for v in col]
        else:
            obj[name] = [str(v) for v in col]
    return json.dumps(obj)


def _plain(table: ChainTable, names) -> str:
    grid = [list(names)] + [[_plain_text(table[c][i]) for c in names] for i in range(table.length)]
    widths = [max(len(row[j]) for row in grid) for j in range(len(names))]
    return "".join("  ".join(cell.ljust(w) for cell, w in zip(row, widths)) + "\n" for row in grid)


_FORMATS = {"csv": _csv, "json": _json, "plain": _plain}


def format_output(table: ChainTable, fmt: str = "csv") -> str:
    """Serialize a table to csv, json, or a plain aligned listing
    (batch.py:294-326)."""
    if fmt not in _FORMATS:
        raise BatchError("DomainError", 0, f"unknown output format {fmt!r}")
    return _FORMATS[fmt](table, list(table.columns))
