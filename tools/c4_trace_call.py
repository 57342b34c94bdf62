#!/usr/bin/env python3
"""One 20M-row C4 host-buffer call (pinned) three times, printing the call
time and the bytes it moved host -> device; with an FV_HOST_TRACE=1 build
(tools/build_variants.py trace=FV_HOST_TRACE=1, FV_LIB=...) each call also
prints its host issue marks and device timeline on stderr."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2604_27210_b200 import _native
lib = _native.lib_for_compute()
dev = torch.device("cuda", 0)
n = 20_000_000
cols = bench.c4_device(n, 0, dev)
cols["price"] = bench.price_on_device(lib, 0, cols, n)
h = {k: (v.cpu().pin_memory() if v.numel() > 1 else v.cpu()) for k, v in cols.items() if torch.is_tensor(v)}
iv = torch.empty(n, dtype=torch.float64).pin_memory(); st = torch.empty(n, dtype=torch.int8).pin_memory()
hn = bench.native_cols(h, "price")
err = _native.fv_error()
for _ in range(3):
    t0 = time.perf_counter()
    lib.fv_batch_iv(0, 1, *hn, n, iv.data_ptr(), st.data_ptr(), None, err)
    print("call ms", 1e3 * (time.perf_counter() - t0), "h2d", lib.fv_last_h2d_bytes(), file=sys.stderr)
