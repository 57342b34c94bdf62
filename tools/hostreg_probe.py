#!/usr/bin/env python3
"""Is registering the caller's pageable numpy buffers (cudaHostRegister) for
the H2D / D2H of a host call cheaper than staging them through the library's
pinned slots (a threaded memcpy)?  VERDICT r1 item 9.  Measures, for 1 GB of
freshly written pageable memory: register + unregister, an 8-thread memcpy
into a pinned buffer, and H2D from pinned / registered / pageable memory.

    python tools/hostreg_probe.py > gpurun_out/hostreg_probe.json
"""
import json
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch


def main():
    lib = torch.cuda.cudart()
    nbytes = 1 << 30
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    out = {}
    for rep in range(2):
        a = np.empty(nbytes, dtype=np.uint8)
        a[::4096] = 1                                   # touch every page
        t0 = time.perf_counter()
        rc = lib.cudaHostRegister(a.ctypes.data, nbytes, 0)
        t1 = time.perf_counter()
        h = torch.from_numpy(a)
        dev.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        dev.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        lib.cudaHostUnregister(a.ctypes.data)
        t4 = time.perf_counter()
        out[f"rep{rep}"] = {"register_s": t1 - t0, "register_rc": int(rc), "h2d_registered_s": t3 - t2,
                            "unregister_s": t4 - t3}
    pinned = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    a = np.empty(nbytes, dtype=np.uint8)
    a[::4096] = 1
    pv = pinned.numpy()
    parts = 8
    per = nbytes // parts

    def cp(i):
        pv[i * per:(i + 1) * per] = a[i * per:(i + 1) * per]
    with ThreadPoolExecutor(parts) as ex:
        list(ex.map(cp, range(parts)))
        t0 = time.perf_counter()
        list(ex.map(cp, range(parts)))
        t1 = time.perf_counter()
    dev.copy_(pinned, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dev.copy_(pinned, non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    h = torch.from_numpy(a)
    dev.copy_(h)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    dev.copy_(h)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    out["memcpy_8threads_to_pinned_s"] = t1 - t0
    out["h2d_pinned_s"] = t3 - t2
    out["h2d_pageable_s"] = t5 - t4
    out["bytes"] = nbytes
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
