#!/usr/bin/env python3
"""Weighted distinct FP64 operation count of the reference's Halley path
(solver.py:49-161, implied_vol_halley) per quote, split by the phase the
B200 kernels follow: bracket (:60-112: forward, discount, f(SIGMA_LO), f(hi),
f(guess) -> k_halley_bracket), halley (:115-144 -> k_halley_iter) and bisect
(:146-161 -> k_halley_bisect).  Same rules as tools/w_count.py (weights
add/sub/mul 1, div 8, sqrt 8, exp 15, log 20, erfc 45; an (op, operands)
pair is charged once per quote, to the phase that first computes it); the
phase is the solver.py line being executed (sys.settrace).  Runs a read-only
import of the reference (/root/reference) on a C2 sample; the result is
committed as profiles/w_phases_c2.json and read by bench.py.

    python tools/w_count_halley.py [rows] > profiles/w_phases_c2.json
"""
import json
import math
import os
import sys
import types

sys.dont_write_bytecode = True
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
import w_count as WC  # noqa: E402  (CF floats, note(), STATE)

STATE = WC.STATE


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
    import fastvol.distributions as D
    import fastvol.pricing as P
    import fastvol.solver as S
    from fastvol.models import Model
    mathns = types.SimpleNamespace(**{k: getattr(math, k) for k in dir(math) if not k.startswith("_")})
    mathns.exp = WC.counted("exp", math.exp)
    mathns.log = WC.counted("log", math.log)
    mathns.sqrt = WC.counted("sqrt", math.sqrt)
    mathns.erfc = WC.counted("erfc", math.erfc)
    for mod in (D, P, S):
        mod.math = mathns
    solver_file = S.__file__

    def tracer(frame, event, arg):
        if frame.f_code.co_filename != solver_file or frame.f_code.co_name != "implied_vol_halley":
            return tracer
        if event == "line":
            ln = frame.f_lineno
            STATE["phase"] = "bracket" if ln < 115 else ("halley" if ln < 146 else "bisect")
        return tracer

    from oracle import fvoracle as O
    import workloads as W
    O.lib()
    flag, Su, K, t, r, q, sig = W.chain_draws(rows, seed=0)
    px = O.rows_price("bsm", flag, Su, K, t, r, q, sig)["price"]
    phases = ("bracket", "halley", "bisect")
    tot = {p: 0.0 for p in phases}
    reach = {p: 0 for p in phases}
    totals = []
    sys.settrace(tracer)
    try:
        for i in range(rows):
            STATE["seen"] = set()
            STATE["w"] = {}
            STATE["phase"] = "bracket"
            S.implied_vol_halley(WC.CF(px[i]), int(flag[i]), Model.BLACK_SCHOLES_MERTON, WC.CF(Su[i]),
                                 WC.CF(K[i]), WC.CF(t[i]), WC.CF(r[i]), WC.CF(q[i]))
            w = STATE["w"]
            totals.append(sum(w.values()))
            for p in phases:
                if w.get(p, 0.0) > 0.0:
                    reach[p] += 1
                tot[p] += w.get(p, 0.0)
    finally:
        sys.settrace(None)
    out = {"workload": "c2", "rows": rows, "sample": f"chain_draws({rows}, seed=0) (the C2 generator), BSM Halley",
           "W_total_mean": float(np.mean(totals)),
           "phases": {p: {"W_per_quote": tot[p] / rows, "share_reaching": reach[p] / rows,
                          "W_per_reaching_quote": tot[p] / max(1, reach[p])} for p in phases}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
