#!/usr/bin/env python3
"""Back-to-back 1-row host calls whose broadcast scalars differ (batch_price
with a sigma, then batch_iv with a price): every batch_iv must see its own
price, not the previous call's sigma (the broadcast-scalar copy is ordered
on the pipeline's stream).  Prints the count of wrong results.

    FV_LIB=... python tools/stress_scalars.py [iterations]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import paper_2604_27210_b200 as fv  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    base = (["p"], [2.279255594198151e+122], [7.81815240030788e+117], [3.279971536884726e-05],
            [0.026461581327708927])
    good = fv.batch_iv("black", "lbr", *base, price=[-0.0], q=[0.0])
    want = (str(good["status"][0]), np.float64(good["iv"][0]).tobytes())
    bad = 0
    for i in range(n):
        fv.batch_price("black", *base, [0.0], sigma=[1.9518652727891157e-10 * (1 + (i % 7))])
        tb = fv.batch_iv("black", "lbr", *base, price=[-0.0], q=[0.0])
        got = (str(tb["status"][0]), np.float64(tb["iv"][0]).tobytes())
        if got != want:
            bad += 1
            if bad <= 3:
                print("WRONG", i, tb["status"][0], tb["iv"][0], flush=True)
    print("lib", os.environ.get("FV_LIB", "default"), "iterations", n, "wrong", bad, "expected", want[0])


if __name__ == "__main__":
    main()
