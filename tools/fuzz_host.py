#!/usr/bin/env python3
"""Fuzz of the HOST-buffer call paths through the Python API (the drop-in
batch_* / price_iv): random batch sizes (1 row to a few million, odd sizes
across chunk boundaries), random broadcast patterns (any column a scalar or
a 1-element list), random models / methods / entry points, calls back to
back with different scalars -- every result checked against the oracle on the
same rows.  Prints a JSON summary (mismatching calls listed).

    python tools/fuzz_host.py [seconds] > fuzz_host.json
"""
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

from test_gpu_fuzz import wide_draws  # noqa: E402

MODELS = ("black", "bs", "bsm")


def same(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return bool(np.all((a.view(np.int64) == b.view(np.int64)) | (np.isnan(a) & np.isnan(b))))


def main():
    import paper_2604_27210_b200 as fv
    from oracle import fvoracle as O
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    rng = np.random.default_rng(12345)
    t0 = time.time()
    calls = rows = 0
    bad = []
    while time.time() - t0 < budget:
        model = MODELS[int(rng.integers(0, 3))]
        n = int(rng.choice([1, 2, 3, 31, 64, 1000, 65537, 262143, 262145, 1 << 20, 3_000_001]))
        flag, un, K, t, r, q, sig = wide_draws(n, int(rng.integers(0, 1 << 30)), model)
        p = O.rows_price(model, flag, un, K, t, r, q, sig)
        g = O.rows_greeks(model, flag, un, K, t, r, q, sig)
        keep = (p["exc"] == 0) & (g["exc"] == 0)
        if not keep.any():
            continue
        flag, un, K, t, r, q, sig = [c[keep] for c in (flag, un, K, t, r, q, sig)]
        n = flag.size
        cols = {"un": un, "K": K, "t": t, "r": r, "q": q, "sig": sig}
        # broadcast some columns: one value for every row (as a scalar or a 1-element list)
        for name in cols:
            if n > 1 and rng.random() < 0.3:
                v = float(cols[name][0])
                cols[name] = np.full(n, v)
        un, K, t, r, q, sig = (cols[k] for k in ("un", "K", "t", "r", "q", "sig"))
        fc = np.where(flag > 0, "c", "p")

        def arg(a):
            if n > 1 and np.all(a == a[0]) and rng.random() < 0.5:
                return float(a[0]) if rng.random() < 0.5 else [float(a[0])]
            return a
        kind = int(rng.integers(0, 4))
        try:
            if kind == 0:
                want = O.rows_price(model, flag, un, K, t, r, q, sig)
                if (want["exc"] != 0).any():
                    continue
                got = fv.batch_price(model, fc, arg(un), arg(K), arg(t), arg(r), arg(q), sigma=arg(sig))
                ok = same(got["price"], want["price"])
            elif kind == 1:
                want = O.rows_greeks(model, flag, un, K, t, r, q, sig)
                if (want["exc"] != 0).any():
                    continue
                got = fv.batch_greeks(model, fc, arg(un), arg(K), arg(t), arg(r), arg(q), sigma=arg(sig))
                ok = all(same(got[k], want[k]) for k in ("delta", "gamma", "theta", "rho", "vega"))
            else:
                method = "lbr" if kind == 2 else "halley"
                px = O.rows_price(model, flag, un, K, t, r, q, sig)["price"]
                if n > 1 and rng.random() < 0.2:
                    px = np.full(n, float(px[0]))
                want = O.rows_iv(model, method, flag, un, K, t, r, q, px)
                if (want["exc"] != 0).any():
                    continue
                got = fv.batch_iv(model, method, fc, arg(un), arg(K), arg(t), arg(r), price=arg(px), q=arg(q))
                codes = {"converged": 0, "fell_back_to_bisection": 1, "below_intrinsic": 2,
                         "above_upper_bound": 3, "max_iterations": 4}
                st = np.array([codes[s] for s in got["status"]], np.int8)
                ok = same(got["iv"], want["iv"]) and bool((st == want["status_code"]).all())
        except Exception as exc:  # noqa: BLE001
            ok = False
            got = repr(exc)
        calls += 1
        rows += n
        if not ok:
            bad.append({"model": model, "n": n, "kind": kind, "detail": str(got)[:200]})
    print(json.dumps({"seconds": round(time.time() - t0, 1), "calls": calls, "rows": rows,
                      "mismatching_calls": len(bad), "first": bad[:20]}, indent=1))


if __name__ == "__main__":
    main()
