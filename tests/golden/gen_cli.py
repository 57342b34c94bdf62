#!/usr/bin/env python3
"""Golden fixture for the chain data path (paper_2604_27210_b200/chain.py)
from the REAL reference CLI (fastvol 0.1.0, /root/reference/pkg/src/fastvol/
cli.py ``main(["chain", ...])``, imported read-only).  Run in the build
container; the output is committed.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_cli.py

cli_chain.json.gz: for each case the input CSV text, the chain arguments, and
the reference's exit code, output text (--output file) and stderr line.  The
cases follow the reference's own CLI acceptance test
(pkg/tests/test_acceptance.py:255-322: a bs chain priced, inverted and
Greeked, then re-inverted from its own prices, a bad flag -> exit 1) and add
the other models, both methods, json output, q / sigma / price pass-through
columns, header-only files, the reader's slow path (CRLF line ends, quoted
cells) and each DataError the data path raises.
"""
import contextlib
import csv
import gzip
import io
import json
import math
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from fastvol.cli import main as cli_main  # noqa: E402


def _csv_text(header, rows, crlf=False):
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\r\n" if crlf else "\n")
    w.writerow(header)
    for row in rows:
        w.writerow(row)
    return buf.getvalue()


def acceptance_rows(n, seed=77):
    """test_acceptance.py:255-275's chain generator (bs model, sigma column)."""
    rng = np.random.default_rng(seed)
    rows = []
    for _ in range(n):
        t = float(rng.uniform(0.1, 2.0))
        sig = float(rng.uniform(0.1, 0.8))
        x = float(rng.uniform(-1.0, 1.0)) * min(2.0 * sig * math.sqrt(t), 0.4)
        rows.append(["c" if rng.random() < 0.5 else "p", "100.0", repr(float(100.0 * math.exp(-x))), repr(t),
                     repr(float(rng.uniform(-0.01, 0.05))), repr(sig)])
    return rows


def wide_rows(n, seed, under="F", with_q=False, with_price=False):
    """Wider draws: deep wings, short maturities, a few t = 0 / sigma = 0
    rows (Greeks' step-function edge) and upper-case flags."""
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        flag = "cpCP"[int(rng.integers(0, 4))]
        u = 100.0
        k = float(100.0 * math.exp(rng.uniform(-2.5, 2.5)))
        t = float(rng.choice([0.0, 1.0 / 365.0, rng.uniform(0.01, 3.0)], p=[0.02, 0.08, 0.9]))
        r = float(rng.uniform(-0.01, 0.06))
        sig = float(rng.choice([0.0, rng.uniform(0.05, 1.5)], p=[0.02, 0.98]))
        row = [flag, repr(u), repr(k), repr(t), repr(r)]
        if with_q:
            row.append(repr(float(rng.uniform(0.0, 0.04))))
        row.append(repr(sig))
        if with_price:
            row.append(repr(float(rng.uniform(0.0, 60.0))))
        rows.append(row)
    return rows


def run_ref(text, model, compute, method="halley", fmt="csv", name="chain.csv"):
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, name)
        with open(src, "w", newline="") as fh:
            fh.write(text)
        out = os.path.join(d, "out.txt")
        err = io.StringIO()
        so = io.StringIO()
        argv = ["chain", "--input", src, "--model", model, "--compute", compute, "--method", method,
                "--format", fmt, "--output", out]
        with contextlib.redirect_stderr(err), contextlib.redirect_stdout(so):
            rc = cli_main(argv)
        body = open(out).read() if os.path.exists(out) else ""
        return rc, body, err.getvalue().replace(src, "<input>")


def main():
    cases = []

    def add(name, text, model, compute, method="halley", fmt="csv"):
        rc, out, err = run_ref(text, model, compute, method, fmt)
        cases.append(dict(name=name, input=text, model=model, compute=compute, method=method, fmt=fmt,
                          rc=rc, out=out, err=err))
        print(f"{name:24s} rc={rc} out={len(out)}B err={err.strip()[:70]!r}")
        return out

    acc = acceptance_rows(1500)
    hdr = ["flag", "S", "K", "t", "r", "sigma"]
    priced = add("bs_price_iv_greeks", _csv_text(hdr, acc), "bs", "price,iv,greeks")
    # re-invert from the reference's own price column (test_acceptance.py:296-312)
    got = list(csv.DictReader(io.StringIO(priced)))
    requote = [[a[0], a[1], a[2], a[3], a[4], g["price"]] for a, g in zip(acc, got)]
    add("bs_reinvert", _csv_text(["flag", "S", "K", "t", "r", "price"], requote), "bs", "iv")
    add("bs_reinvert_lbr", _csv_text(["flag", "S", "K", "t", "r", "price"], requote), "bs", "iv", "lbr")

    w76 = wide_rows(800, 11, with_price=True)
    add("black_lbr_iv_greeks_json", _csv_text(["flag", "F", "K", "t", "r", "sigma", "price"], w76), "black",
        "iv,greeks", "lbr", "json")
    add("black_price_iv_halley", _csv_text(["flag", "F", "K", "t", "r", "sigma", "price"], w76), "black",
        "price,iv", "halley")
    wq = wide_rows(800, 12, with_q=True)
    add("bsm_greeks_q", _csv_text(["flag", "S", "K", "t", "r", "q", "sigma"], wq), "bsm", "greeks")
    add("bsm_price_json", _csv_text(["flag", "S", "K", "t", "r", "q", "sigma"], wq), "bsm", "price", fmt="json")
    # column order: the input header order is kept, computed columns follow
    perm = [[r[3], r[0], r[5], r[2], r[1], r[4]] for r in acc[:300]]
    add("bs_permuted_header", _csv_text(["t", "flag", "sigma", "K", "S", "r"], perm), "bs", "price,greeks")
    # the reader's slow path: CRLF line ends, quoted cells
    add("bs_crlf", _csv_text(hdr, acc[:300], crlf=True), "bs", "price")
    quoted = '"flag","S","K","t","r","sigma"\n' + "".join(
        f'"{a[0]}",{a[1]},"{a[2]}",{a[3]},{a[4]},{a[5]}\n' for a in acc[:200])
    add("bs_quoted", quoted, "bs", "price,iv")
    # header-only files
    add("header_only_csv", "flag,S,K,t,r,sigma\n", "bs", "price,iv,greeks")
    add("header_only_json", "flag,F,K,t,r,price\n", "black", "iv", fmt="json")
    # data errors (exit code 1, "error: ..." on stderr)
    bad = _csv_text(hdr, acc[:50])
    add("err_bad_flag", bad + "x,100,100,1,0,0.2\n", "bs", "price")
    add("err_not_a_number", bad + "c,100,abc,1,0,0.2\n", "bs", "price")
    add("err_negative_sigma", bad + "c,100,100,1,0,-0.2\n", "bs", "price")
    add("err_missing_column", "flag,S,K,t,sigma\nc,100,100,1,0.2\n", "bs", "price")
    add("err_q_not_accepted", "flag,S,K,t,r,q,sigma\nc,100,100,1,0,0.01,0.2\n", "bs", "price")
    add("err_price_needs_sigma", "flag,S,K,t,r\nc,100,100,1,0\n", "bs", "price")
    add("err_iv_needs_price", "flag,S,K,t,r,sigma\nc,100,100,1,0,0.2\n", "bs", "iv")
    add("err_unknown_compute", "flag,S,K,t,r,sigma\nc,100,100,1,0,0.2\n", "bs", "price,vega")
    add("err_ragged_row", "flag,S,K,t,r,sigma\nc,100,100,1,0,0.2\nc,100,100\n", "bs", "price")
    add("err_unknown_column", "flag,S,K,t,r,sigma,zz\nc,100,100,1,0,0.2,1\n", "bs", "price")
    add("err_S_and_F", "flag,S,F,K,t,r,sigma\nc,100,100,100,1,0,0.2\n", "bs", "price")
    add("err_empty_file", "", "bs", "price")
    add("err_nonfinite_price", "flag,F,K,t,r,price\nc,100,100,1,0,8\np,100,100,1,0,nan\n", "black", "iv", "lbr")
    path = os.path.join(HERE, "cli_chain.json.gz")
    with gzip.open(path, "wt") as fh:
        json.dump({"source": "fastvol 0.1.0 cli.main (reference)", "cases": cases}, fh)
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
