#!/usr/bin/env python3
"""e2e (pinned host buffers through the C ABI) of a C1/C2/C3-style workload
at several host-pipeline chunk sizes (fv_set_chunk_rows; with the default
build the auto-sizing caps a chunk at max(n/8, 2^18) rows), plus the
device-resident call on the same rows for comparison.

    FV_LIB=... python tools/e2e_small.py c1 [rows] [chunk rows ...]
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
    wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
    chunks = [int(a) for a in sys.argv[3:]] or [65536, 131072, 262144, 524288, 1048576, 4194304]
    lib = _native.lib_for_compute()
    dev = torch.device("cuda", 0)
    lib.fv_set_stream(torch.cuda.current_stream(dev).cuda_stream)
    model, method, _ = bench.workload_call(wl)
    cols = bench.draws_device(wl, n, 0, dev)
    last = "sigma"
    if method >= 0:
        cols["price"] = bench.price_on_device(lib, model, cols, n)
        last = "price"
    h = {k: (v.cpu().pin_memory() if v.numel() > 1 else v.cpu()) for k, v in cols.items() if torch.is_tensor(v)}
    hn = bench.native_cols(h, last)
    dn = bench.native_cols(cols, last)
    outs_h = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(6)]
    st_h = torch.empty(n, dtype=torch.int8).pin_memory()
    outs_d = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(6)]
    st_d = torch.empty(n, dtype=torch.int8, device=dev)

    def call(cn, outs, st):
        err = _native.fv_error()
        if method >= 0:
            rc = lib.fv_batch_iv(model, method, *cn, n, outs[0].data_ptr(), st.data_ptr(), None, err)
        else:
            err2 = _native.fv_error()
            rc = lib.fv_price_greeks(model, *cn, n, *[o.data_ptr() for o in outs], st.data_ptr(), err, err2)
        if rc:
            raise RuntimeError(err.message)

    def timeit(f, reps=20):
        f()
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            f()
            torch.cuda.synchronize(dev)
            ts.append(time.perf_counter() - t0)
        return 1e3 * float(np.median(ts)), 1e3 * float(np.min(ts))

    med, mn = timeit(lambda: call(dn, outs_d, st_d))
    print(f"{wl} n={n} device-resident: median {med:.3f} ms  min {mn:.3f} ms")
    for c in chunks:
        lib.fv_set_chunk_rows(c)
        med, mn = timeit(lambda: call(hn, outs_h, st_h))
        print(f"{wl} n={n} chunk {c}: e2e median {med:.3f} ms  min {mn:.3f} ms  ({n / med / 1e6:.1f} M/s)")
    lib.fv_set_chunk_rows(1 << 22)


if __name__ == "__main__":
    main()
