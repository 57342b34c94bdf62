#!/usr/bin/env python3
"""How much of k_halley_iter's cost is the erfc range mix?  Times the Halley
passes (fv_set_kernel_timing, serialised) on 10M-quote BSM batches whose
quotes keep both normal-CDF arguments in one erfc range group -- 'inner'
(near the money: |d1|, |d2| < 1.25 sqrt2 at every iterate, mostly) and
'tail' (deep wings) -- next to C2's draws, and divides by the number of
Halley-phase f evaluations (a float64 replay of solver.py:115-144 in numpy,
which follows the solver's path closely enough to count its trips).

    python tools/halley_classes.py [rows] > halley_classes.json
"""
import json
import os
import sys

import numpy as np
from scipy.special import erfc

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def draws(kind, n, seed=0):
    rng = np.random.default_rng(seed)
    flag = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
    S = np.full(n, 100.0)
    t = rng.uniform(0.1, 2.0, n)
    r = rng.uniform(-0.01, 0.05, n)
    q = rng.uniform(0.0, 0.03, n)
    sig = rng.uniform(0.1, 0.8, n)
    if kind == "c2":
        K = S * np.exp(rng.uniform(-0.6, 0.6, n))
    elif kind == "inner":
        s = sig * np.sqrt(t)
        K = S * np.exp((r - q) * t) * np.exp(rng.uniform(-0.15, 0.15, n) * s)
    else:                                              # tail: |x| ~ 3-5 s, OTM side
        s = sig * np.sqrt(t)
        x = rng.uniform(3.0, 5.0, n) * s
        K = S * np.exp((r - q) * t) * np.exp(np.where(flag > 0, x, -x))
    return flag, S, K, t, r, q, sig


def sim_trips(flag, S, K, t, r, q, sig):
    """Halley-phase f evaluations and their erfc range classes (float64 replay)."""
    F = S * np.exp((r - q) * t)
    sq = np.sqrt(t)
    lnFK = np.log(F / K)
    th = flag.astype(float)
    disc = np.exp(-r * t)

    def price(sg):
        s = sg * sq
        d1 = (lnFK + 0.5 * s * s) / s
        d2 = d1 - s
        raw = th * (F * 0.5 * erfc(-th * d1 / np.sqrt(2)) - K * 0.5 * erfc(-th * d2 / np.sqrt(2)))
        return disc * np.clip(raw, np.maximum(th * (F - K), 0), np.where(th > 0, F, K))

    def cls(sg):
        s = sg * sq
        d1 = (lnFK + 0.5 * s * s) / s
        d2 = d1 - s
        g1 = np.abs(d1) < 1.25 * np.sqrt(2)
        g2 = np.abs(d2) < 1.25 * np.sqrt(2)
        return np.where(g1 & g2, 0, np.where(~g1 & ~g2, 2, 1))

    target = price(sig)
    tol = np.minimum(1e-12 * np.maximum(1, disc * np.where(th > 0, F, K)),
                     1e-10 * (target - disc * np.maximum(th * (F - K), 0)))
    lo = np.full(len(S), 1e-9)
    hi = np.full(len(S), 10.0)
    sg = np.clip(np.sqrt(2 * np.pi / t) * target / S, 0.05, 2.0)
    fv = price(sg) - target
    hi = np.where(fv > 0, np.minimum(hi, sg), hi)
    lo = np.where(fv < 0, np.maximum(lo, sg), lo)
    active = np.abs(fv) > tol
    trips = 0
    counts = np.zeros(3)
    with np.errstate(all="ignore"):
        for _ in range(16):
            if not active.any():
                break
            s = sg * sq
            d1 = (lnFK + 0.5 * s * s) / s
            d2 = d1 - s
            vega = disc * F * np.exp(-0.5 * d1 * d1) / np.sqrt(2 * np.pi) * sq
            den = 2 * vega * vega - fv * vega * d1 * d2 / sg
            cand = sg - 2 * fv * vega / den
            ok = np.isfinite(cand) & (lo < cand) & (cand < hi) & (vega > 0)
            x = np.where(ok, cand, 0.5 * (lo + hi))
            fx = price(x) - target
            c = cls(x)
            counts += np.bincount(c[active], minlength=3)
            trips += int(active.sum())
            rej = ok & ~(np.abs(fx) < np.abs(fv))
            mid = 0.5 * (lo + hi)
            trips += int((rej & active).sum())
            x = np.where(rej, mid, x)
            fx = np.where(rej, price(mid) - target, fx)
            hi = np.where(active & (fx > 0), x, hi)
            lo = np.where(active & (fx < 0), x, lo)
            step = x - sg
            sg = np.where(active, x, sg)
            fv = np.where(active, fx, fv)
            active &= ~((np.abs(step) <= 1e-12 * np.maximum(1, sg)) | (np.abs(fv) <= tol))
    return trips, (counts / counts.sum()).round(4).tolist()


def main():
    import torch
    from paper_2604_27210_b200 import _native
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    dev = torch.device("cuda", 0)
    lib = _native.lib_for_compute()
    lib.fv_set_stream(torch.cuda.current_stream(dev).cuda_stream)
    out = {"rows": rows}
    for kind in ("c2", "inner", "tail"):
        flag, S, K, t, r, q, sig = draws(kind, rows)
        sub = slice(0, min(rows, 400_000))
        trips, mix = sim_trips(flag[sub], S[sub], K[sub], t[sub], r[sub], q[sub], sig[sub])
        trips_per_quote = trips / len(S[sub])
        cols = [torch.from_numpy(flag).to(dev)] + [torch.from_numpy(c).to(dev) for c in (S, K, t, r, q, sig)]
        n = rows
        px = torch.empty(n, dtype=torch.float64, device=dev)
        err = _native.fv_error()
        assert lib.fv_batch_price(2, *[_native.col(c) for c in cols], n, px.data_ptr(), err) == 0, err.message
        iv = torch.empty(n, dtype=torch.float64, device=dev)
        st = torch.empty(n, dtype=torch.int8, device=dev)
        call = lambda: lib.fv_batch_iv(2, 0, *[_native.col(c) for c in cols[:6]], _native.col(px), n,
                                       iv.data_ptr(), st.data_ptr(), None, err)
        for _ in range(2):
            assert call() == 0, err.message
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(5):
            call()
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / 5
        lib.fv_set_kernel_timing(1)
        _native.kernel_times(lib)
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        kt = {k: v[0] / 3 for k, v in _native.kernel_times(lib).items()}
        lib.fv_set_kernel_timing(0)
        it_ms = kt.get("k_halley_iter", 0.0)
        codes = np.bincount(st.cpu().numpy().astype(np.int64), minlength=5)[:5] / n
        out[kind] = {"ms_per_call": ms, "G_quotes_per_s": n / ms / 1e6, "kernels_ms": kt,
                     "halley_trips_per_quote_sim": trips_per_quote, "trip_class_mix_sim_ii_mixed_tt": mix,
                     "iter_ns_per_trip": it_ms * 1e6 / (trips_per_quote * n) if trips_per_quote else None,
                     "status_mix": codes.round(4).tolist()}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
