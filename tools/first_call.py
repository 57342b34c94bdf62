#!/usr/bin/env python3
"""Per-call wall time of repeated host-buffer calls (first-call costs:
workspace growth, pinned staging, lazy module loading)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_27210_b200 as fv                      # noqa: E402
from paper_2604_27210_b200 import bench as FB           # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
flag, S, K, t, r, q, sig, price = FB.synthetic_chain(n, 0)
for label, fn in (("batch_iv halley", lambda: fv.batch_iv("bsm", "halley", flag, S, K, t, r, price=price, q=q)),
                  ("batch_iv lbr", lambda: fv.batch_iv("bsm", "lbr", flag, S, K, t, r, price=price, q=q)),
                  ("price_iv halley", lambda: fv.price_iv("bsm", "halley", flag, S, K, t, r, q, sigma=sig)),
                  ("batch_price", lambda: fv.batch_price("bsm", flag, S, K, t, r, q, sigma=sig))):
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    print(label, " ".join("%.4f" % x for x in ts), flush=True)
