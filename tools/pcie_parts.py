#!/usr/bin/env python3
"""PCIe copy throughput against copy size with raw cudaMemcpyAsync (cuda-python,
no torch dispatch per copy): 256 MB per direction cut into parts of 0.5-64 MB,
one direction alone and both directions at once.  The host pipeline's copies
are one column of one chunk each, so this is the curve its chunk size sits on.

    python tools/pcie_parts.py > pcie_parts.txt
"""
import time

import torch
from cuda.bindings import runtime as rt


def main():
    n = 1 << 28
    h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1 = torch.cuda.Stream().cuda_stream
    s2 = torch.cuda.Stream().cuda_stream
    H2D = rt.cudaMemcpyKind.cudaMemcpyHostToDevice
    D2H = rt.cudaMemcpyKind.cudaMemcpyDeviceToHost

    def issue(dst, src, part, kind, s):
        for o in range(0, n, part):
            rt.cudaMemcpyAsync(dst + o, src + o, part, kind, s)

    def t(f):
        f()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    for part in (64 << 20, 16 << 20, 8 << 20, 4 << 20, 2 << 20, 1 << 20, 512 << 10):
        def a():
            issue(d1.data_ptr(), h1.data_ptr(), part, H2D, s1)

        def b():
            issue(h2.data_ptr(), d2.data_ptr(), part, D2H, s2)

        def c():
            for o in range(0, n, part):       # interleaved issue, as the pipeline's slots do
                rt.cudaMemcpyAsync(d1.data_ptr() + o, h1.data_ptr() + o, part, H2D, s1)
                rt.cudaMemcpyAsync(h2.data_ptr() + o, d2.data_ptr() + o, part, D2H, s2)
        # host issue rate alone (no wait): is the measurement issue-bound?
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a()
        issue_us = 1e6 * (time.perf_counter() - t0) / (n // part)
        torch.cuda.synchronize()
        ta, tb, tc = t(a), t(b), t(c)
        print("part %6d KB: H2D %5.1f GB/s  D2H %5.1f GB/s  both at once %5.1f GB/s each  (issue %.1f us/copy)"
              % (part >> 10, n / ta / 1e9, n / tb / 1e9, n / tc / 1e9, issue_us))


if __name__ == "__main__":
    main()
