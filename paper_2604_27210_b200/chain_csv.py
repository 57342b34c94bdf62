"""Option-chain CSV input (the reference's `vol chain` reader,
fastvol/cli.py:140-173 ``_read_chain`` + ``_numeric``), the data format on the
input side of the batch path.

``read_chain(path)`` returns the columns by header name and
``numeric(cols, name)`` the float64 column, with the reference's checks and
``DataError`` messages.  Files in the common subset (no quoting, '\\n' line
ends, ASCII, one-character flags) are split and parsed by the host extension
(csrc/fv_host.cpp ``parse_chain_csv``: std::from_chars, correctly rounded
like ``float()``) on several threads; cells outside its strict decimal form
go through ``float()`` itself, and every other file through the ``csv``
module -- the same values and the same first error either way.
"""
import csv
from typing import Dict

import numpy as np

from . import batch as _batch

CHAIN_COLUMNS = ("flag", "S", "F", "K", "t", "r", "q", "sigma", "price")   # cli.py:21


class DataError(Exception):
    """A chain file the reader rejects (cli.py:24)."""


class ChainColumns(dict):
    """Columns by header name.  On the fast path the numeric columns are
    float64 arrays whose cells outside the strict decimal form are still
    pending (``numeric`` applies ``float()`` to them in row order)."""

    def __init__(self, *args, **kw):
        super().__init__(*args, **kw)
        self.pending = {}          # name -> [(row, column index)]
        self.raw = b""
        self._lines = None

    def cell(self, row: int, col: int) -> str:
        if self._lines is None:
            self._lines = self.raw.split(b"\n")
        return self._lines[row + 1].split(b",")[col].decode("ascii")


def _read_csv_module(path):
    try:
        with open(path, newline="") as fh:
            reader = csv.reader(fh)
            try:
                header = next(reader)
            except StopIteration:
                raise DataError(f"{path}: empty file (header required)")
            rows = list(reader)
    except OSError as exc:
        raise DataError(f"cannot read {path}: {exc}")
    return header, rows


def _check_header(path, header):
    for name in header:
        if name not in CHAIN_COLUMNS:
            raise DataError(f"{path}: unknown column {name!r}")
    if "S" in header and "F" in header:
        raise DataError(f"{path}: columns S and F are mutually exclusive")


def _read_slow(path) -> ChainColumns:
    header, rows = _read_csv_module(path)
    _check_header(path, header)
    cols = ChainColumns((name, []) for name in header)
    for i, row in enumerate(rows):
        if len(row) != len(header):
            raise DataError(f"{path}: row {i} has {len(row)} cells, expected {len(header)}")
        for name, cell in zip(header, row):
            cols[name].append(cell)
    return cols


def read_chain(path: str) -> ChainColumns:
    """Columns of a chain CSV by header name (cli.py:140-163): numpy arrays on
    the fast path (float64; 'flag' as a 'U1' array), else lists of cells."""
    if _batch._fvhost is None:
        return _read_slow(path)
    try:
        with open(path, "rb") as fh:
            data = fh.read()
    except OSError as exc:
        raise DataError(f"cannot read {path}: {exc}")
    fast = _batch._fvhost.parse_chain_csv(data)
    if fast is None:
        return _read_slow(path)
    header, arrays, bad = fast
    _check_header(path, header)
    if len(set(header)) != len(header):      # repeated names share one list in the reference
        return _read_slow(path)
    cols = ChainColumns(zip(header, arrays))
    cols.raw = data
    for row, j in bad:
        cols.pending.setdefault(header[j], []).append((row, j))
    return cols


def numeric(cols: ChainColumns, name: str) -> np.ndarray:
    """The float64 column ``name`` (cli.py:166-173): the first cell that is
    not a number raises ``DataError`` with the reference's message."""
    col = cols[name]
    if isinstance(col, np.ndarray):
        pend = getattr(cols, "pending", {}).get(name)
        if not pend:
            return col
        col = col.copy()
        for row, j in sorted(pend):
            cell = cols.cell(row, j)
            try:
                col[row] = float(cell)
            except ValueError:
                raise DataError(f"row {row}, column {name}: not a number: {cell!r}")
        return col
    out = np.empty(len(col), dtype=np.float64)
    for i, cell in enumerate(col):
        try:
            out[i] = float(cell)
        except ValueError:
            raise DataError(f"row {i}, column {name}: not a number: {cell!r}")
    return out
