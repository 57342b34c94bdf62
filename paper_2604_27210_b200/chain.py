"""Option-chain processing: the data path of the reference's ``vol chain``
subcommand (fastvol/cli.py:176-280 ``_chain``) on the B200 batch path.

``run_chain(input, model, compute, method, fmt)`` reads the chain CSV
(``chain_csv.read_chain`` / ``numeric``), runs the requested stages on the
GPU in the reference's order -- price, then iv, then greeks -- and returns the
text ``format_output`` renders for the assembled table (input columns in
header order, then the computed ones).  Column checks, the header-only shape,
``DataError`` messages and the error raised first are the reference's; a
``BatchError`` from a stage surfaces as ``DataError(str(exc))`` as in
cli.py:263-264.  Argument parsing and exit codes stay with the CLI (out of
scope): a caller maps ``DataError`` to exit code 1.

When both price and iv are requested, the two stages run as one
``price_iv`` call (the price column is produced and inverted on the device
without a host round trip); its values and its first error are those of
``batch_price`` followed by ``batch_iv`` (tests/test_price_iv.py).
"""
from typing import Optional

import numpy as np

from . import batch as B
from .batch import BatchError, ChainTable, format_output
from .chain_csv import DataError, numeric, read_chain
from .models import Model

__all__ = ["run_chain", "DataError"]


def _flag_codes(flag) -> np.ndarray:
    """cli.py:268: 1 for 'c' / 'C', -1 for anything else (the cells passed
    parse_flags already, so that means 'p' / 'P')."""
    f = np.asarray(flag)
    return np.where((f == "c") | (f == "C"), 1, -1).astype(np.int8)


def run_chain(input: str, model: str, compute: str = "price", method: str = "halley",
              fmt: str = "csv", output: Optional[str] = None) -> str:
    """cli.py:176-280 on the GPU: returns the output text (and writes it to
    ``output`` when given, as ``_emit`` does)."""
    mdl = Model.parse(model)
    items = [c.strip() for c in compute.split(",") if c.strip()]
    for c in items:
        if c not in ("price", "iv", "greeks"):
            raise DataError(f"unknown --compute item {c!r}")
    cols = read_chain(input)
    n = len(next(iter(cols.values()))) if cols else 0

    if "flag" not in cols:
        raise DataError("missing required column: flag")
    need_under = "F" if mdl is Model.BLACK76 else "S"
    if need_under not in cols:
        raise DataError(f"missing required column: {need_under}")
    for name in ("K", "t", "r"):
        if name not in cols:
            raise DataError(f"missing required column: {name}")
    if "q" in cols and mdl is not Model.BLACK_SCHOLES_MERTON:
        raise DataError(f"model {model} does not accept a q column")

    flag = cols["flag"] if n else []
    under = numeric(cols, need_under)
    strike = numeric(cols, "K")
    t = numeric(cols, "t")
    r = numeric(cols, "r")
    q = numeric(cols, "q") if "q" in cols else np.zeros(n)
    sigma = numeric(cols, "sigma") if "sigma" in cols else None
    price = numeric(cols, "price") if "price" in cols else None

    if n == 0:                                   # cli.py:202-216: header-only input
        out_names = list(cols)
        extra = []
        for c in items:
            if c == "price" and "price" not in cols:
                extra.append("price")
            if c == "iv":
                extra.extend(["iv", "status"])
            if c == "greeks":
                extra.extend(list(B.GREEK_COLUMNS))
        text = ",".join(out_names + extra) + "\n"
        if fmt == "json":
            text = format_output(ChainTable({name: np.empty(0) for name in out_names + extra}), "json")
        return _emit(text, output)

    try:
        result = {}
        base = dict(flag=flag, underlying=under, strike=strike, t=t, r=r, q=q)
        if "price" in items:
            if sigma is None:
                raise DataError("--compute price requires a sigma column")
            if "iv" in items:                    # price then iv, one device call
                table = B.price_iv(mdl, method, sigma=sigma, **base)
                price = table["price"]
                result["price"] = table["price"]
                result["iv"] = table["iv"]
                result["status"] = table["status"]
            else:
                table = B.batch_price(mdl, sigma=sigma, **base)
                price = table["price"]
                result["price"] = table["price"]
        if "iv" in items and "iv" not in result:
            if price is None:
                raise DataError("--compute iv requires a price column (or --compute price,iv)")
            table = B.batch_iv(mdl, method, price=price, **base)
            result["iv"] = table["iv"]
            result["status"] = table["status"]
        if "greeks" in items:
            if sigma is None:
                raise DataError("--compute greeks requires a sigma column")
            table = B.batch_greeks(mdl, sigma=sigma, **base)
            for name in B.GREEK_COLUMNS:
                result[name] = table[name]
            if "iv" not in items:
                result["status"] = table["status"]
    except BatchError as exc:
        if exc.kind == "BadFlag" and isinstance(flag, np.ndarray):
            # the reference's reader hands batch_* a list of str (cli.py:160-163),
            # so its message shows the cell's str repr, not numpy's np.str_(...)
            exc = B._flag_error(exc.index, str(flag[exc.index]))
        raise DataError(str(exc))

    out = {}
    parsed = {"flag": _flag_codes(flag), need_under: under, "K": strike, "t": t, "r": r}
    for name in cols:                            # cli.py:269-278
        if name == "q":
            out["q"] = q
        elif name == "sigma":
            out["sigma"] = sigma
        elif name == "price" and "price" not in result:
            out["price"] = price
        elif name in parsed:
            out[name] = parsed[name]
    for name, col in result.items():
        out[name] = col
    return _emit(format_output(ChainTable(out), fmt), output)


def _emit(text: str, output: Optional[str]) -> str:
    """cli.py:95-100: the text to ``output`` (an ASCII str is written as its
    bytes by the host extension, GIL released -- the same file contents as
    the text-mode write, without its encode copy)."""
    if output:
        if B._fvhost is None or B._fvhost.write_text(output, text) is None:
            with open(output, "w") as fh:
                fh.write(text)
    return text
