"""Chain CSV input (paper_2604_27210_b200/chain_csv.py; the reference's
cli.py:140-173 ``_read_chain`` / ``_numeric``): the threaded fast path gives
the reference reader's values bit for bit and the same first error."""
import csv

import numpy as np
import pytest

from paper_2604_27210_b200 import _build, batch as B, chain_csv as C


@pytest.fixture(scope="module", autouse=True)
def host_ext():
    _build.build_host()
    import importlib
    B._fvhost = importlib.import_module("paper_2604_27210_b200._fvhost")


class RefError(Exception):
    pass


def ref_read(path):
    """cli.py:140-163, restated (csv module)."""
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        try:
            header = next(reader)
        except StopIteration:
            raise RefError(f"{path}: empty file (header required)")
        rows = list(reader)
    for name in header:
        if name not in C.CHAIN_COLUMNS:
            raise RefError(f"{path}: unknown column {name!r}")
    if "S" in header and "F" in header:
        raise RefError(f"{path}: columns S and F are mutually exclusive")
    cols = {name: [] for name in header}
    for i, row in enumerate(rows):
        if len(row) != len(header):
            raise RefError(f"{path}: row {i} has {len(row)} cells, expected {len(header)}")
        for name, cell in zip(header, row):
            cols[name].append(cell)
    return cols


def ref_numeric(cols, name):
    """cli.py:166-173, restated."""
    out = np.empty(len(cols[name]), dtype=np.float64)
    for i, cell in enumerate(cols[name]):
        try:
            out[i] = float(cell)
        except ValueError:
            raise RefError(f"row {i}, column {name}: not a number: {cell!r}")
    return out


def outcome(reader, numeric, path, names):
    try:
        cols = reader(path)
        res = {}
        for n in names:
            if n in cols:
                res[n] = numeric(cols, n).view(np.int64).tolist()
        if "flag" in cols:
            res["flag"] = [str(x) for x in cols["flag"]]
        return ("ok", res)
    except (RefError, C.DataError) as e:
        return ("err", str(e))


def check(path, names=("F", "S", "K", "t", "r", "q", "sigma", "price")):
    assert outcome(C.read_chain, C.numeric, path, names) == outcome(ref_read, ref_numeric, path, names)


def write(tmp_path, text, name="chain.csv"):
    p = tmp_path / name
    p.write_bytes(text.encode())
    return str(p)


def test_large_clean_chain(tmp_path):
    rng = np.random.default_rng(3)
    n = 200_000
    K = 100 * np.exp(rng.uniform(-0.6, 0.6, n))
    t = rng.uniform(1e-4, 3, n)
    px = rng.integers(0, 2**64, n, dtype=np.uint64).view(np.float64)
    fl = rng.choice(["c", "p", "C", "P"], n)
    fmt = [repr, lambda v: "%.6g" % v, lambda v: "%.3e" % v, lambda v: "%.17f" % v]
    lines = ["flag,F,K,t,r,price"]
    for i in range(n):
        f = fmt[i % 4]
        lines.append(f"{fl[i]},100,{f(K[i])},{f(t[i])},0.03,{repr(float(px[i]))}")
    path = write(tmp_path, "\n".join(lines) + "\n")
    fast = B._fvhost.parse_chain_csv(open(path, "rb").read())
    assert fast is not None
    check(path)


@pytest.mark.parametrize("cell", ["nan", "-nan", "inf", "-inf", "Infinity", "1e400", "-1e-400", "5e-324",
                                  " 1.5", "2.5 ", "+2", "1_000.5", "0x1p3", ".5", "5.", "-.5e-3", "1e5",
                                  "abc", "", "1.5.2", "--1", "1e", "e5", "nan(12)"])
def test_special_cells(tmp_path, cell):
    body = "\n".join(f"c,100,{100 + i},0.5,0.03,{cell if i == 700 else 1.25}" for i in range(1500))
    check(write(tmp_path, "flag,F,K,t,r,price\n" + body + "\n"))


@pytest.mark.parametrize("text", [
    "",                                                    # empty file
    "flag,F,K,t,r\n",                                      # header only
    "flag,F,K,t,r",                                        # header only, no newline
    "flag,F,K,t,r\nc,100,100,0.5,0.03",                    # no final newline
    "flag,F,K,t,r\nc,100,100,0.5\n",                       # ragged row
    "flag,F,K,t,r\nc,100,100,0.5,0.03\n\nc,100,100,0.5,0.03\n",   # empty line
    "flag,F,K,t,x\nc,100,100,0.5,0.03\n",                  # unknown column
    "flag,S,F,K,t,r\nc,100,100,100,0.5,0.03\n",            # S and F
    "flag,F,K,t,r\r\nc,100,100,0.5,0.03\r\n",              # CRLF
    "flag,F,K,t,r\n\"c\",100,\"1,5\",0.5,0.03\n",          # quoted cells
    "flag,F,K,t,r\ncall,100,100,0.5,0.03\n",               # long flag text
    "flag,F,F,t,r\nc,100,101,0.5,0.03\n",                  # repeated column name
])
def test_edge_files(tmp_path, text):
    check(write(tmp_path, text))


def test_first_error_is_reference_row_order(tmp_path):
    rows = [f"c,100,{100 + i},0.5,0.03" for i in range(5000)]
    rows[4000] = "c,100,bad1,0.5,0.03"
    rows[300] = "c,100,+1e2,0.5,oops"
    rows[2000] = "c,100,bad0,0.5,0.03"
    check(write(tmp_path, "flag,F,K,t,r\n" + "\n".join(rows) + "\n"))
