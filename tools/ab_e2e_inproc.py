#!/usr/bin/env python3
"""e2e A/B of several builds of the library IN ONE PROCESS: each
variants/lib_*.so is loaded with its own ctypes handle (RTLD_LOCAL), the
workload's pinned host buffers are made once, and the builds' host-buffer
C-ABI calls alternate round by round, so box-to-box and drift noise cancel.
Prints the median and min call time per build and workload.

    [AB_LIBS=a,b] python tools/ab_e2e_inproc.py [workloads...]     (default: c4 c5 c1 c2 c3 rt)
"""
import ctypes
import glob
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402
from paper_2604_27210_b200 import _native  # noqa: E402


def load(path):
    lib = ctypes.CDLL(path)
    for name, (args, res) in _native.SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is not None:
            fn.argtypes, fn.restype = args, res
    return lib


def main():
    wls = sys.argv[1:] or ["c4", "c5", "c1", "c2", "c3", "rt"]
    paths = sorted(glob.glob(os.path.join(REPO, "variants", "lib_*.so")))
    if os.environ.get("AB_LIBS"):                     # e.g. AB_LIBS=a,b: only variants/lib_a.so, lib_b.so
        paths = [os.path.join(REPO, "variants", "lib_%s.so" % x) for x in os.environ["AB_LIBS"].split(",")]
    libs = [(os.path.basename(p)[4:-3], load(p)) for p in paths]
    # AB_CHUNKS=name:rows,...: a build's host-pipeline chunk rows (copies of one .so
    # under several names keep separate settings)
    for spec in filter(None, os.environ.get("AB_CHUNKS", "").split(",")):
        name, rows = spec.split(":")
        for nm, lib in libs:
            if nm == name:
                lib.fv_set_chunk_rows(int(rows))
    ref = _native.lib_for_compute()
    dev = torch.device("cuda", 0)
    for wl in wls:
        model, method, roundtrip = bench.workload_call(wl)
        if wl == "c4":
            n = 100_000_000
            cols = bench.c4_device(n, 0, dev)
        else:
            n = bench.default_rows(wl)
            cols = bench.draws_device(wl, n, 0, dev)
        last = "sigma"
        if method >= 0 and not roundtrip:
            cols["price"] = bench.price_on_device(ref, model, cols, n)
            last = "price"
        pin = not os.environ.get("AB_PAGEABLE")         # AB_PAGEABLE=1: pageable host buffers
        h = {k: (v.cpu().pin_memory() if (v.numel() > 1 and pin) else v.cpu()) for k, v in cols.items()
             if torch.is_tensor(v)}
        del cols
        torch.cuda.empty_cache()
        hn = bench.native_cols(h, last)
        outs = [torch.empty(n, dtype=torch.float64) for _ in range(6 if method < 0 else 2)]
        st = torch.empty(n, dtype=torch.int8)
        if pin:
            outs = [o.pin_memory() for o in outs]
            st = st.pin_memory()

        def call(lib):
            e1, e2 = _native.fv_error(), _native.fv_error()
            if roundtrip:
                rc = lib.fv_price_iv(model, method, *hn, n, outs[0].data_ptr(), outs[1].data_ptr(), st.data_ptr(),
                                     None, e1, e2)
            elif method >= 0:
                rc = lib.fv_batch_iv(model, method, *hn, n, outs[0].data_ptr(), st.data_ptr(), None, e1)
            else:
                rc = lib.fv_price_greeks(model, *hn, n, *[o.data_ptr() for o in outs], st.data_ptr(), e1, e2)
            if rc not in (0,):
                raise RuntimeError(e1.message)

        times = {name: [] for name, _ in libs}
        for name, lib in libs:
            call(lib)
        rounds = 6 if wl == "c4" else 15
        for r in range(rounds):
            order = libs if r % 2 == 0 else libs[::-1]
            for name, lib in order:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                call(lib)
                times[name].append(time.perf_counter() - t0)
        for name, _ in libs:
            ts = np.array(times[name])
            print("%-3s %-10s e2e median %.3f G/s (%.2f ms)  best %.3f G/s" %
                  (wl, name, n / np.median(ts) / 1e9, 1e3 * np.median(ts), n / ts.min() / 1e9), flush=True)
        del h, hn, outs, st
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
