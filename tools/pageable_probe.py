#!/usr/bin/env python3
"""Where does a pageable-buffer C-ABI call spend its time?  (VERDICT r1 item
9: the drop-in Python path, numpy in / numpy out.)  50M C4 rows through
fv_batch_iv with host pointers: pinned inputs+outputs, pageable inputs with
pinned outputs, pageable inputs with pre-touched pageable outputs, and fresh
(never touched) pageable outputs -- the Python API's case -- at a few chunk
sizes.

    python tools/pageable_probe.py [rows] > gpurun_out/pageable_probe.json
"""
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import torch
    import workloads as W
    from paper_2604_27210_b200 import _native
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
    lib = _native.lib_for_compute()
    flag, F, K, t, r, sig = W.c4_params(0, n)
    from oracle import fvoracle as O          # prices only (inputs of the probe)
    O.lib()
    O.set_threads(os.cpu_count() or 1)
    px = O.rows_price("black", flag, F[:1], K, t, r[:1], 0.0, sig)["price"]
    cols_p = [np.ascontiguousarray(c) for c in (flag, F[:1], K, t, r[:1], np.zeros(1), px)]
    pinned = [torch.from_numpy(c).pin_memory() if c.size > 1 else torch.from_numpy(c) for c in cols_p]
    out = {"rows": n}

    def run(cols, iv, st, label, reps=3):
        err = _native.fv_error()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            rc = lib.fv_batch_iv(0, 1, *[_native.col(c) for c in cols], n, _native.ptr(iv), _native.ptr(st),
                                 None, err)
            ts.append(time.perf_counter() - t0)
            assert rc == 0, err.message
        out[label] = {"s": min(ts), "quotes_per_s": n / min(ts)}

    for chunk in (1 << 21, 1 << 22, 1 << 23):
        lib.fv_set_chunk_rows(chunk)
        tag = f"chunk{chunk >> 20}M"
        iv_p = torch.empty(n, dtype=torch.float64).pin_memory()
        st_p = torch.empty(n, dtype=torch.int8).pin_memory()
        run(pinned, iv_p, st_p, f"{tag}_pinned_in_pinned_out")
        run(cols_p, iv_p, st_p, f"{tag}_pageable_in_pinned_out")
        iv = np.ones(n)
        st = np.ones(n, np.int8)
        run(cols_p, iv, st, f"{tag}_pageable_in_touched_pageable_out")
        ts = []
        for _ in range(3):
            iv = np.empty(n)
            st = np.empty(n, np.int8)
            err = _native.fv_error()
            t0 = time.perf_counter()
            lib.fv_batch_iv(0, 1, *[_native.col(c) for c in cols_p], n, iv.ctypes.data, st.ctypes.data, None, err)
            ts.append(time.perf_counter() - t0)
        out[f"{tag}_pageable_in_fresh_pageable_out"] = {"s": min(ts), "quotes_per_s": n / min(ts)}
    t0 = time.perf_counter()
    a = np.empty(n)
    a[:] = 0.0
    out["first_touch_write_of_an_n_row_f64_array_s"] = time.perf_counter() - t0
    lib.fv_set_chunk_rows(1 << 22)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
