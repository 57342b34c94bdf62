"""Drop-in for the reference's throughput harness, fastvol/bench.py.

``synthetic_chain`` draws the same seeded BSM contracts as the reference
(bench.py:19-31: flag, K, t, r, q, sigma from ``numpy.random.default_rng(seed)``
in that order, S = 100) and prices them with ``batch_price``; ``run_bench``
times ``batch_iv`` on them and writes the same CSV report
(``rows,method,seconds,rows_per_sec,converged``, bench.py:34-54).  Both go
through the B200 path, so the reported rows/sec is the GPU's.

``run_roundtrip`` is the same workload as one fused price -> IV call
(``batch.price_iv`` -> ``fv_price_iv``): synthetic_chain's
pricing and run_bench's inversion without the price column leaving the
device in between.
"""

import sys
import time
from typing import Optional

import numpy as np

from .batch import batch_iv, batch_price, price_iv
from .models import Model


def _draws(rows: int, seed: int):
    """bench.py:21-28: (flag, S, K, t, r, q, sigma), same generator calls."""
    rng = np.random.default_rng(seed)
    flag = np.where(rng.random(rows) < 0.5, "c", "p")
    S = np.full(rows, 100.0)
    K = S * np.exp(rng.uniform(-0.6, 0.6, rows))
    t = rng.uniform(0.1, 2.0, rows)
    r = rng.uniform(-0.01, 0.05, rows)
    q = rng.uniform(0.0, 0.03, rows)
    sigma = rng.uniform(0.1, 0.8, rows)
    return flag, S, K, t, r, q, sigma


def synthetic_chain(rows: int, seed: int = 0):
    """Seeded random BSM contracts with known sigma, plus their prices
    (bench.py:19-31)."""
    flag, S, K, t, r, q, sigma = _draws(rows, seed)
    priced = batch_price(Model.BLACK_SCHOLES_MERTON, flag, S, K, t, r, q, sigma=sigma)
    return flag, S, K, t, r, q, sigma, priced["price"]


def _converged(status) -> int:
    return int(np.count_nonzero((status == "converged") | (status == "fell_back_to_bisection")))


def _report(rows, method, elapsed, ok, output, figure) -> int:
    rps = rows / elapsed if elapsed > 0 else float("inf")
    text = ("rows,method,seconds,rows_per_sec,converged\n"
            f"{rows},{method},{elapsed!r},{rps!r},{ok}\n")
    if output:
        with open(output, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    if figure:
        _write_figure(figure, rows, method, rps)
    return 0


def run_bench(rows: int, method: str = "halley", output: Optional[str] = None,
              figure: Optional[str] = None, seed: int = 0) -> int:
    """bench.py:34-54: invert a synthetic chain, report rows/sec."""
    flag, S, K, t, r, q, sigma, price = synthetic_chain(rows, seed)
    start = time.perf_counter()
    table = batch_iv(Model.BLACK_SCHOLES_MERTON, method, flag, S, K, t, r, price=price, q=q)
    elapsed = time.perf_counter() - start
    return _report(rows, method, elapsed, _converged(table["status"]), output, figure)


def run_roundtrip(rows: int, method: str = "halley", output: Optional[str] = None,
                  figure: Optional[str] = None, seed: int = 0) -> int:
    """The same chain priced and inverted in one fused call; the timed region
    covers both stages (same report format)."""
    flag, S, K, t, r, q, sigma = _draws(rows, seed)
    start = time.perf_counter()
    table = price_iv(Model.BLACK_SCHOLES_MERTON, method, flag, S, K, t, r, q, sigma=sigma)
    elapsed = time.perf_counter() - start
    return _report(rows, method, elapsed, _converged(table["status"]), output, figure)


def _write_figure(path: str, rows: int, method: str, rps: float) -> None:
    """The reference's matplotlib report figure (bench.py:57-69) is outside
    the hot path this package rebuilds: asking for one is an error here."""
    raise NotImplementedError("throughput figures are not part of the B200 path; omit --figure "
                              f"(requested {path!r} for {rows} rows, {method}, {rps:.3g} rows/s)")
