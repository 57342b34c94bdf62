#!/usr/bin/env python3
"""Long wide-domain fuzz of every entry point against the oracle (the draws
of tests/test_gpu_fuzz.py, many seeds): prints one JSON summary and every
mismatching row (inputs included).  Device-resident C-ABI calls on cuda:0.

    python tools/fuzz_big.py [seconds] [rows_per_batch] > fuzz.json
"""
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

from test_gpu_fuzz import MODELS, _dev, _iv_dev, _keep, _price_greeks_dev, wide_draws  # noqa: E402


def bits_bad(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    same = (got.view(np.int64) == want.view(np.int64)) | (np.isnan(got) & np.isnan(want))
    return np.flatnonzero(~same)


def main():
    import torch
    from oracle import fvoracle as O
    from paper_2604_27210_b200 import _native
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 600.0
    rows = int(sys.argv[2]) if len(sys.argv) > 2 else 4_000_000
    lib = _native.lib_for_compute()
    dev = torch.device("cuda", 0)
    lib.fv_set_stream(torch.cuda.current_stream(dev).cuda_stream)
    t0 = time.time()
    checked = {}
    bad_rows = []
    seed = 10_000
    while time.time() - t0 < budget:
        for model in MODELS:
            seed += 1
            flag, un, K, t, r, q, sig = wide_draws(rows, seed, model)
            p = O.rows_price(model, flag, un, K, t, r, q, sig)
            g = O.rows_greeks(model, flag, un, K, t, r, q, sig)
            keep = _keep(p) & _keep(g)
            cols = [c[keep] for c in (flag, un, K, t, r, q, sig)]
            outs, st = _price_greeks_dev(lib, dev, MODELS[model], _dev(dev, cols))
            names = ("price", "delta", "gamma", "theta", "rho", "vega")
            for j, name in enumerate(names):
                want = p["price"][keep] if j == 0 else g[name][keep]
                for i in bits_bad(outs[j], want)[:5]:
                    bad_rows.append({"entry": f"{model} {name}", "seed": seed, "got": repr(outs[j][i]),
                                     "want": repr(want[i]), "inputs": [repr(float(c[i])) for c in cols]})
            checked[f"{model} price+greeks"] = checked.get(f"{model} price+greeks", 0) + int(keep.sum())
            rng = np.random.default_rng(seed)
            px = p["price"][keep]
            kind = rng.integers(0, 6, px.size)
            cap = np.where(cols[0] > 0, cols[1], cols[2]) * 1.5
            px = np.select([kind == 1, kind == 2, kind == 3, kind == 4],
                           [px * (1.0 + rng.normal(0, 1e-3, px.size)), px * 1e-6, cap,
                            px * rng.uniform(0, 1, px.size)], default=px)
            for method, mcode in (("lbr", 1), ("halley", 0)):
                n_m = px.size if method == "lbr" else min(px.size, rows // 4)
                c_m = [c[:n_m] for c in cols[:6]] + [px[:n_m]]
                want = O.rows_iv(model, method, *c_m)
                ok = _keep(want)
                c_ok = [c[ok] for c in c_m]
                iv, stv, reg = _iv_dev(lib, dev, MODELS[model], mcode, _dev(dev, c_ok))
                for i in bits_bad(iv, want["iv"][ok])[:5]:
                    bad_rows.append({"entry": f"{model} {method} iv", "seed": seed, "got": repr(iv[i]),
                                     "want": repr(want["iv"][ok][i]), "inputs": [repr(float(c[i])) for c in c_ok]})
                for i in np.flatnonzero(stv != want["status_code"][ok])[:5]:
                    bad_rows.append({"entry": f"{model} {method} status", "seed": seed, "got": int(stv[i]),
                                     "want": int(want["status_code"][ok][i]),
                                     "inputs": [repr(float(c[i])) for c in c_ok]})
                if method == "lbr":
                    for i in np.flatnonzero(reg != want["region"][ok])[:5]:
                        bad_rows.append({"entry": f"{model} lbr region", "seed": seed, "got": int(reg[i]),
                                         "want": int(want["region"][ok][i]),
                                         "inputs": [repr(float(c[i])) for c in c_ok]})
                checked[f"{model} {method}"] = checked.get(f"{model} {method}", 0) + int(ok.sum())
            if time.time() - t0 >= budget:
                break
    print(json.dumps({"seconds": time.time() - t0, "rows_checked": checked,
                      "total_rows": sum(checked.values()), "mismatches": len(bad_rows),
                      "first_mismatches": bad_rows[:50]}, indent=1))


if __name__ == "__main__":
    main()
