#!/usr/bin/env python3
"""A/B of the small-batch LBR path (fv_set_lbr_eager_rows): the same
device-resident call with the eager path (anchors inside the normalize pass,
far-low + near solves in one kernel) and without it, on C1 (1M), C5 (10M)
and C4 sub-chains; checks the two are bit-identical.

    python tools/eager_ab.py
"""
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import torch
    import bench
    import workloads as W
    from paper_2604_27210_b200 import _native
    lib = _native.lib_for_compute()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    lib.fv_set_stream(stream.cuda_stream)
    res = {}
    cases = [("c1", 1_000_000), ("c4", 1_000_000), ("c4", 4_000_000), ("c5", 10_000_000), ("c4", 10_000_000)]
    for wl, rows in cases:
        if wl == "c4":
            cols = bench.c4_device(0, 0, dev, ranges=[(0, rows)], n_total=rows, F=100.0)
        else:
            cols = bench.draws_device(wl, rows, 0, dev)
            kind, side = cols.pop("kind"), cols.pop("side")
        n = cols["flag"].numel()
        cols["price"] = bench.price_on_device(lib, 0, cols, n)
        if wl == "c5":
            h = {k: cols[k].cpu().numpy() for k in ("flag", "underlying", "strike", "t", "r", "price")}
            cols["price"] = torch.from_numpy(W.c5_prices(h["flag"], h["underlying"], h["strike"], h["t"], h["r"],
                                                         kind, side, h["price"])).to(dev)
        nc = bench.native_cols(cols, "price")
        out = {}
        for mode, eager in (("eager", 1 << 30), ("classic", 0)):
            lib.fv_set_lbr_eager_rows(eager)
            iv = torch.empty(n, dtype=torch.float64, device=dev)
            st = torch.empty(n, dtype=torch.int8, device=dev)
            reg = torch.empty(n, dtype=torch.int8, device=dev)
            err = _native.fv_error()

            def call():
                assert lib.fv_batch_iv(0, 1, *nc, n, iv.data_ptr(), st.data_ptr(), reg.data_ptr(), err) == 0, \
                    err.message
            for _ in range(3):
                call()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20 if n <= 4_000_000 else 8
            e0.record(stream)
            for _ in range(reps):
                call()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            out[mode] = (ms, iv.clone(), st.clone(), reg.clone())
        lib.fv_set_lbr_eager_rows(1 << 23)
        same = all(torch.equal(out["eager"][k].view(torch.int64) if k == 1 else out["eager"][k],
                               out["classic"][k].view(torch.int64) if k == 1 else out["classic"][k])
                   for k in (1, 2, 3))
        key = f"{wl}_{n}"
        res[key] = {"eager_ms": out["eager"][0], "classic_ms": out["classic"][0],
                    "eager_gqps": n / out["eager"][0] / 1e6, "classic_gqps": n / out["classic"][0] / 1e6,
                    "bit_identical": bool(same)}
        print(key, json.dumps(res[key]))
        del cols, out
        torch.cuda.empty_cache()
    json.dump(res, open(os.path.join(REPO, "gpurun_out", "eager_ab.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
