#!/usr/bin/env python3
"""e2e (pinned host buffers through the C ABI) of the C4 100M chain at several
host-pipeline chunk sizes (fv_set_chunk_rows)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2604_27210_b200 import _native

lib = _native.lib_for_compute()
dev = torch.device("cuda", 0)
n = 100_000_000
cols = bench.c4_device(n, 0, dev)
cols["price"] = bench.price_on_device(lib, 0, cols, n)
h = {k: (v.cpu().pin_memory() if v.numel() > 1 else v.cpu()) for k, v in cols.items() if torch.is_tensor(v)}
iv = torch.empty(n, dtype=torch.float64).pin_memory()
st = torch.empty(n, dtype=torch.int8).pin_memory()
hn = bench.native_cols(h, "price")
for rows in [int(a) for a in (sys.argv[1:] or ["1048576", "2097152", "4194304", "8388608", "16777216"])]:
    lib.fv_set_chunk_rows(rows)
    err = _native.fv_error()
    lib.fv_batch_iv(0, 1, *hn, n, iv.data_ptr(), st.data_ptr(), None, err)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lib.fv_batch_iv(0, 1, *hn, n, iv.data_ptr(), st.data_ptr(), None, err)
        ts.append(time.perf_counter() - t0)
    print(rows, "rows/chunk: %.2f ms  %.3f G quotes/s" % (1e3 * min(ts), n / min(ts) / 1e9))
