#!/usr/bin/env python3
"""Repeat the golden exception cases (tests/golden/exceptions.json: fuzzed
extreme rows with the reference's outcomes) through batch_price -> batch_iv
and the fused price_iv, one-row host calls, and count rows whose iv / status
differ from the reference's -- a hunt for nondeterministic results.

    FV_LIB=... python tools/stress_exceptions.py [reps]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import paper_2604_27210_b200 as fv  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    cases = json.load(open("tests/golden/exceptions.json"))
    bad = 0
    total = 0
    shown = 0
    for rep in range(reps):
        for c in cases:
            a = c["in"]
            base = ([("c" if a["flag"] > 0 else "p")], [a["underlying"]], [a["strike"]], [a["t"]], [a["r"]])
            try:
                p = fv.batch_price(a["model"], *base, [a["q"]], sigma=[a["sigma"]])["price"]
            except Exception:  # noqa: BLE001
                continue
            for m in ("lbr", "halley"):
                want = c.get(m)
                outs = {}
                for path in ("golden", "two", "fused"):
                    try:
                        if path == "golden":
                            tb = fv.batch_iv(a["model"], m, *base, price=[a["price"]], q=[a["q"]])
                        elif path == "two":
                            tb = fv.batch_iv(a["model"], m, *base, price=p, q=[a["q"]])
                        else:
                            tb = fv.price_iv(a["model"], m, *base, [a["q"]], sigma=[a["sigma"]])
                        outs[path] = (str(tb["status"][0]), np.float64(tb["iv"][0]))
                    except Exception as e:  # noqa: BLE001
                        outs[path] = ("exc", type(e).__name__)
                checks = []
                if isinstance(want, dict) and "status" in want:
                    wiv = np.float64(float("nan") if want["iv"] is None else want["iv"])
                    checks.append(("golden", outs["golden"], (want["status"], wiv)))
                checks.append(("fused-vs-two", outs["fused"], outs["two"]))
                for name, got, exp in checks:
                    total += 1
                    same = got[0] == exp[0] and (
                        not isinstance(got[1], np.floating) or got[1].tobytes() == exp[1].tobytes()
                        or (np.isnan(got[1]) and np.isnan(exp[1])))
                    if not same:
                        bad += 1
                        if shown < 8:
                            shown += 1
                            print("MISMATCH", rep, m, name, got, "want", exp, a, flush=True)
    print(json.dumps({"lib": os.environ.get("FV_LIB", "default"), "reps": reps, "rows": total, "mismatches": bad}))


if __name__ == "__main__":
    main()
