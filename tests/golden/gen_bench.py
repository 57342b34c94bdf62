#!/usr/bin/env python3
"""Golden fixture for the bench-harness mirror (paper_2604_27210_b200/bench.py)
and the fused price -> IV call, from the REAL reference (fastvol 0.1.0,
/root/reference/pkg/src/fastvol/bench.py, imported read-only).  Run in the
build container; the output is committed.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_bench.py

bench_chain.npz: synthetic_chain(2000, seed=0) -- inputs (flag as int8), the
reference's price column -- then batch_iv(BSM, method, ...) on it for both
methods (iv, status codes) and the converged count run_bench reports, plus
run_bench's report text with the timing cells blanked.
"""
import io
import os
import sys
import contextlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from fastvol import bench as RB  # noqa: E402
from fastvol.batch import batch_iv  # noqa: E402
from fastvol.models import Model  # noqa: E402

IV_CODES = {"converged": 0, "fell_back_to_bisection": 1, "below_intrinsic": 2,
            "above_upper_bound": 3, "max_iterations": 4}


def main():
    rows, seed = 2000, 0
    flag, S, K, t, r, q, sigma, price = RB.synthetic_chain(rows, seed)
    out = dict(flag=np.where(flag == "c", 1, -1).astype(np.int8), S=S, K=K, t=t, r=r, q=q,
               sigma=sigma, price=price, rows=np.int64(rows), seed=np.int64(seed))
    for method in ("halley", "lbr"):
        tb = batch_iv(Model.BLACK_SCHOLES_MERTON, method, list(flag), S, K, t, r, price=price, q=q)
        out[f"{method}_iv"] = tb["iv"]
        out[f"{method}_status"] = np.array([IV_CODES[s] for s in tb["status"]], np.int8)
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            assert RB.run_bench(rows, method, None, None, seed) == 0
        head, line = buf.getvalue().strip().splitlines()
        cells = line.split(",")
        out[f"{method}_report_head"] = np.array(head)
        out[f"{method}_report_cells"] = np.array([cells[0], cells[1], cells[4]])
    np.savez_compressed(os.path.join(HERE, "bench_chain.npz"), **out)
    print("bench_chain.npz:", {m: str(out[f"{m}_report_cells"]) for m in ("halley", "lbr")})


if __name__ == "__main__":
    main()
