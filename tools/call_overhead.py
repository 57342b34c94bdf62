#!/usr/bin/env python3
"""Fixed cost of one device-resident C-ABI call: wall time per call (host
checks, launches, the status read-back and synchronisation) against the
device span of its kernels (fv_set_span_timing), for tiny and C1-sized
batches of LBR / Halley / price + Greeks.

    python tools/call_overhead.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2604_27210_b200 import _native  # noqa: E402


def main():
    lib = _native.lib_for_compute()
    dev = torch.device("cuda", 0)
    lib.fv_set_stream(torch.cuda.current_stream(dev).cuda_stream)
    for wl in ("c1", "c2", "c3"):
        model, method, _ = bench.workload_call(wl)
        for n in (1, 1024, 1_000_000):
            cols = bench.draws_device(wl, n, 0, dev)
            last = "sigma"
            if method >= 0:
                cols["price"] = bench.price_on_device(lib, model, cols, n)
                last = "price"
            cn = bench.native_cols(cols, last)
            outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(6)]
            st = torch.empty(n, dtype=torch.int8, device=dev)

            def call():
                e1, e2 = _native.fv_error(), _native.fv_error()
                if method >= 0:
                    return lib.fv_batch_iv(model, method, *cn, n, outs[0].data_ptr(), st.data_ptr(), None, e1)
                return lib.fv_price_greeks(model, *cn, n, *[o.data_ptr() for o in outs], st.data_ptr(), e1, e2)
            for _ in range(5):
                call()
            wall, span = [], []
            lib.fv_set_span_timing(1)
            for _ in range(50):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                call()
                wall.append(time.perf_counter() - t0)
                span.append(lib.fv_last_span_ms())
            lib.fv_set_span_timing(0)
            w, s = 1e3 * np.median(wall), np.median(span)
            print("%s n=%8d  wall %8.1f us  device span %8.1f us  host-side %6.1f us  launches %d"
                  % (wl, n, 1e3 * w, 1e3 * s, 1e3 * (w - s), lib.fv_last_launch_count()))


if __name__ == "__main__":
    main()
