#!/usr/bin/env python3
"""Host-side cost of the run-length transport's scan (fv_host_find_runs, no
device needed) on C4-shaped 2.5M-row chunks: a maturity column (50 runs), a
strike ladder and a price column (both give up), a flag column (1 run).

    python tools/runs_bench.py
"""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_27210_b200 import _native  # noqa: E402


def main():
    lib = _native.load()
    nr = ctypes.c_int64()
    for n in (262_144, 2_500_000):
        cols = {"t": np.repeat(np.linspace(0.01, 5, n // 50000 + 1), 50000)[:n].copy(),
                "K": 100 * np.exp(np.linspace(-2, 2, 50000))[np.arange(n) % 50000],
                "price": np.random.default_rng(0).uniform(0, 10, n),
                "flag": np.ones(n, np.int8)}
        budget = n // 64
        starts = np.empty(budget + 2, np.int32)
        vals = np.empty(budget + 1, np.uint64)
        for name, col in cols.items():
            ts = []
            for _ in range(9):
                t0 = time.perf_counter()
                lib.fv_host_find_runs(col.ctypes.data, col.dtype.itemsize, n, budget, starts.ctypes.data,
                                      vals.ctypes.data, ctypes.byref(nr))
                ts.append(time.perf_counter() - t0)
            print("rows %8d %-6s runs %6d  min %7.1f us  median %7.1f us  (%.1f GB/s at min)"
                  % (n, name, nr.value, 1e6 * min(ts), 1e6 * float(np.median(ts)),
                     n * col.dtype.itemsize / min(ts) / 1e9))


if __name__ == "__main__":
    main()
