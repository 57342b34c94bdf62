#!/usr/bin/env python3
"""End-to-end `vol chain` data path on the B200 (chain.run_chain), by stage:
CSV read + parse, numeric columns, the device calls, output formatting and
the write.  Shows where the time of a CLI-sized job goes (SURVEY 8(f) rank 2:
the CSV formats either side of the path run on host threads).

    python tools/chain_e2e.py [rows] [compute] > chain_e2e.json
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def make_chain(path, n, seed=77):
    rng = np.random.default_rng(seed)
    t = rng.uniform(0.1, 2.0, n)
    sig = rng.uniform(0.1, 0.8, n)
    x = rng.uniform(-1.0, 1.0, n) * np.minimum(2.0 * sig * np.sqrt(t), 0.4)
    K = 100.0 * np.exp(-x)
    r = rng.uniform(-0.01, 0.05, n)
    fl = np.where(rng.random(n) < 0.5, "c", "p")
    with open(path, "w") as fh:
        fh.write("flag,S,K,t,r,sigma\n")
        fh.writelines(f"{a},100.0,{b!r},{c!r},{d!r},{e!r}\n" for a, b, c, d, e in
                      zip(fl, K.tolist(), t.tolist(), r.tolist(), sig.tolist()))


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    compute = sys.argv[2] if len(sys.argv) > 2 else "price,iv,greeks"
    from paper_2604_27210_b200 import batch as B, chain, chain_csv
    d = tempfile.mkdtemp()
    src = os.path.join(d, "chain.csv")
    make_chain(src, rows)
    out = os.path.join(d, "out.csv")
    chain.run_chain(src, "bs", compute, output=out)                 # warm-up (first-use allocations)
    stages = {}
    orig = {}

    def wrap(mod, name):
        f = getattr(mod, name)
        orig[(mod, name)] = f

        def g(*a, **k):
            t0 = time.perf_counter()
            try:
                return f(*a, **k)
            finally:
                stages[name] = stages.get(name, 0.0) + time.perf_counter() - t0
        setattr(mod, name, g)

    for mod, name in ((chain, "read_chain"), (chain, "numeric"), (B, "price_iv"), (B, "batch_price"),
                      (B, "batch_iv"), (B, "batch_greeks"), (chain, "format_output"), (chain, "_emit")):
        wrap(mod, name)
    reps = 3
    t0 = time.perf_counter()
    for _ in range(reps):
        chain.run_chain(src, "bs", compute, output=out)
    total = (time.perf_counter() - t0) / reps
    for (mod, name), f in orig.items():
        setattr(mod, name, f)
    res = {"rows": rows, "compute": compute, "threads": B.worker_count(), "input_bytes": os.path.getsize(src),
           "output_bytes": os.path.getsize(out), "seconds_per_call": total,
           "rows_per_sec": rows / total,
           "stages_s": {k: v / reps for k, v in stages.items()}}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
