#!/usr/bin/env python3
"""Per-stage host timestamps of a 1-row device-resident call (FV_CALL_TRACE=1 build,
FV_LIB=...): pointer classification, work + lock, launches, status kernel, synchronise."""
import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2604_27210_b200 import _native
lib = _native.lib_for_compute()
lib.fv_call_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
dev = torch.device("cuda", 0)
lib.fv_set_stream(torch.cuda.current_stream(dev).cuda_stream)
for wl in ("c3", "c1"):
    model, method, _ = bench.workload_call(wl)
    n = 1
    cols = bench.draws_device(wl, 1024, 0, dev)
    cols = {k: (v[:n].contiguous() if torch.is_tensor(v) and v.numel() > 1 else v) for k, v in cols.items()}
    last = "sigma"
    if method >= 0:
        cols["price"] = bench.price_on_device(lib, model, cols, n); last = "price"
    cn = bench.native_cols(cols, last)
    outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(6)]
    st = torch.empty(n, dtype=torch.int8, device=dev)
    e1, e2 = _native.fv_error(), _native.fv_error()
    marks = []
    walls = []
    buf = (ctypes.c_double * 16)()
    for i in range(200):
        t0 = time.perf_counter()
        if method >= 0:
            lib.fv_batch_iv(model, method, *cn, n, outs[0].data_ptr(), st.data_ptr(), None, e1)
        else:
            lib.fv_price_greeks(model, *cn, n, *[o.data_ptr() for o in outs], st.data_ptr(), e1, e2)
        walls.append((time.perf_counter() - t0) * 1e6)
        k = lib.fv_call_trace(buf, 16)
        marks.append(list(buf)[:k])
    m = np.median(np.array(marks[20:]), axis=0)
    print(wl, "wall %.1f us" % np.median(walls[20:]), "marks", ["%.1f" % x for x in m])
