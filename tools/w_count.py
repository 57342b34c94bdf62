#!/usr/bin/env python3
"""Weighted distinct FP64 operation count of the reference's LBR path per
quote, split into the classification phase
(normalize_quote, scale, ATM test, _anchors, _region, bracket) and the solve
phase (initial_guess, the Householder(3) iteration, sigma = s / sqrt(t)), per
region -- so the dominant kernel (k_lbr_far_low_fast: the far-low solve) has
its own algorithmic work per quote for its roofline.

Runs a scratch copy of the reference (/root/reference, read-only) with the
discarded residual lines (lbr.py:429, :484) removed, on float subclasses that
record (op, operand bits); "distinct" = first occurrence per quote (an op
already seen in the classification phase is not charged again to the solve).
Weights: add/sub/mul 1, div 8, sqrt 8, exp 15, log 20, erfc 45, erfcx 24.
Run here (needs /root/reference); the result is committed as
profiles/w_phases.json and read by bench.py.

    python tools/w_count.py [rows]
"""
import json
import math
import os
import shutil
import struct
import sys
import tempfile
import types

sys.dont_write_bytecode = True
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

W = {"add": 1, "sub": 1, "mul": 1, "div": 8, "sqrt": 8, "exp": 15, "log": 20, "erfc": 45, "erfcx": 24}
STATE = {"phase": "classify", "seen": set(), "w": {}}


def note(op, a, b=0.0):
    k = (op, struct.pack("<d", float(a)), struct.pack("<d", float(b)))
    if k in STATE["seen"]:
        return
    STATE["seen"].add(k)
    STATE["w"][STATE["phase"]] = STATE["w"].get(STATE["phase"], 0.0) + W[op]


class CF(float):
    def __add__(self, o): note("add", self, o); return CF(float(self) + float(o))
    def __radd__(self, o): note("add", o, self); return CF(float(o) + float(self))
    def __sub__(self, o): note("sub", self, o); return CF(float(self) - float(o))
    def __rsub__(self, o): note("sub", o, self); return CF(float(o) - float(self))
    def __mul__(self, o): note("mul", self, o); return CF(float(self) * float(o))
    def __rmul__(self, o): note("mul", o, self); return CF(float(o) * float(self))
    def __truediv__(self, o): note("div", self, o); return CF(float(self) / float(o))
    def __rtruediv__(self, o): note("div", o, self); return CF(float(o) / float(self))
    def __pow__(self, n):
        for _ in range(int(n) - 1):
            note("mul", self, n)
        return CF(float(self) ** n)
    def __neg__(self): return CF(-float(self))
    def __abs__(self): return CF(abs(float(self)))


def counted(name, fn):
    def f(x, *a):
        note(name, x)
        return CF(fn(float(x), *a))
    return f


def load_reference():
    tmp = tempfile.mkdtemp(prefix="wcount_")
    shutil.copytree("/root/reference/pkg/src/fastvol", os.path.join(tmp, "fastvol"))
    p = os.path.join(tmp, "fastvol", "lbr.py")
    src = open(p).read()
    n = src.count("(normalized_black(")
    src = src.replace("resid = (normalized_black(min(x, 0.0), s) - beta) * scale", "resid = nan")
    src = src.replace("resid = (normalized_black(x, s) - beta) * scale", "resid = nan")
    assert src.count("resid = nan") == 2, n
    open(p, "w").write(src)
    sys.path.insert(0, tmp)
    import fastvol.distributions as D
    import fastvol.lbr as L
    return L, D


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
    L, D = load_reference()
    mathns = types.SimpleNamespace(**{k: getattr(math, k) for k in dir(math) if not k.startswith("_")})
    mathns.exp = counted("exp", math.exp)
    mathns.log = counted("log", math.log)
    mathns.sqrt = counted("sqrt", math.sqrt)
    mathns.erfc = counted("erfc", math.erfc)
    for mod in (L, D):
        mod.math = mathns
    real_erfcx = L._erfcx
    L._erfcx = counted("erfcx", lambda z: float(real_erfcx(z)))
    real_guess, real_region = L.initial_guess, L._region
    seen_region = {}

    def guess(*a, **k):
        STATE["phase"] = "solve"
        return real_guess(*a, **k)

    def region(*a, **k):
        r = real_region(*a, **k)
        seen_region["r"] = r.name
        return r
    L.initial_guess = guess
    L._region = region
    # the 2nd / 3rd normalized_black of _anchors (b_c, b_hi: lbr.py:231-238)
    # are charged to their own phases: the lazy-anchor GPU path evaluates
    # only the anchors _region's comparison chain reads (far-low: b_lo only;
    # near-low: b_lo, b_c), so the whole-call roofline can exclude the rest
    real_anchors, real_nb = L._anchors, L.normalized_black

    def anchors(*a, **k):
        outer = STATE["phase"]
        calls = [0]

        def nb(*aa, **kk):
            STATE["phase"] = ("anchor_lo", "anchor_c", "anchor_hi")[min(calls[0], 2)]
            calls[0] += 1
            try:
                return real_nb(*aa, **kk)
            finally:
                STATE["phase"] = outer
        L.normalized_black = nb
        try:
            return real_anchors(*a, **k)
        finally:
            L.normalized_black = real_nb
            STATE["phase"] = outer
    L._anchors = anchors

    import workloads as WL
    from oracle import fvoracle as O
    O.lib()
    stride = max(1, WL.C4_ROWS // rows)
    flag, F, K, t, r, sig = WL.c4_rows(np.arange(0, WL.C4_ROWS, stride, dtype=np.int64)[:rows])
    px = O.rows_price("black", flag, F, K, t, r, 0.0, sig)["price"]
    by = {}
    totals = []
    for i in range(len(flag)):
        STATE["seen"] = set()
        STATE["w"] = {}
        STATE["phase"] = "classify"
        seen_region.clear()
        L.implied_vol_lbr(CF(px[i]), int(flag[i]), CF(F[i]), CF(K[i]), CF(t[i]), CF(r[i]))
        reg = seen_region.get("r", "FINISHED")
        w = STATE["w"]
        totals.append(sum(w.values()))
        d = by.setdefault(reg, {"n": 0, "classify": 0.0, "solve": 0.0, "anchor_lo": 0.0, "anchor_c": 0.0,
                                "anchor_hi": 0.0})
        d["n"] += 1
        # b_lo / b_c / b_hi: classification work (as before), also reported apart
        d["classify"] += (w.get("classify", 0.0) + w.get("anchor_lo", 0.0) + w.get("anchor_c", 0.0)
                          + w.get("anchor_hi", 0.0))
        d["solve"] += w.get("solve", 0.0)
        d["anchor_lo"] += w.get("anchor_lo", 0.0)
        d["anchor_c"] += w.get("anchor_c", 0.0)
        d["anchor_hi"] += w.get("anchor_hi", 0.0)
    out = {"workload": "c4", "rows": len(totals), "sample": f"every {stride}th row of the C4 chain",
           "W_total_mean": float(np.mean(totals)), "by_region": {}}
    for k, d in by.items():
        out["by_region"][k] = {"share": d["n"] / len(totals), "W_classify": d["classify"] / d["n"],
                               "W_solve": d["solve"] / d["n"], "W_anchor_lo": d["anchor_lo"] / d["n"],
                               "W_anchor_c": d["anchor_c"] / d["n"], "W_anchor_hi": d["anchor_hi"] / d["n"]}
    # W of the anchors the lazy-anchor path does not evaluate: far-low quotes
    # skip b_c and b_hi, near-low quotes b_hi (lbr.py:241-248 never reads them)
    skip = 0.0
    for k, d in by.items():
        if k == "FAR_LOW":
            skip += d["anchor_c"] + d["anchor_hi"]
        elif k == "NEAR_LOW":
            skip += d["anchor_hi"]
    out["W_anchors_not_read_mean"] = skip / len(totals)
    out["W_read_mean"] = out["W_total_mean"] - out["W_anchors_not_read_mean"]
    # the first anchor of far-low quotes as well (round 2: a table bound decides
    # beta < b_lo without it for whole warps of the chain): a lower bound of the
    # work the GPU path evaluates
    fl = by.get("FAR_LOW")
    out["W_done_mean"] = out["W_read_mean"] - (fl["anchor_lo"] / len(totals) if fl else 0.0)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
