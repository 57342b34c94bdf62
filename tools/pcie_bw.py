#!/usr/bin/env python3
"""PCIe link bandwidth between pinned host memory and the GPU: H2D alone,
D2H alone and both directions at once, for one large copy and for runs of
smaller copies (the host pipeline's per-column copies are 0.5-16 MB).

    python tools/pcie_bw.py > pcie_bw.txt
"""
import time

import torch


def main():
    n = 1 << 28                        # 256 MB per direction
    h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

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

    for part in (n, 16 << 20, 2 << 20, 512 << 10):
        def h2d():
            with torch.cuda.stream(s1):
                for o in range(0, n, part):
                    d1[o:o + part].copy_(h1[o:o + part], non_blocking=True)

        def d2h():
            with torch.cuda.stream(s2):
                for o in range(0, n, part):
                    h2[o:o + part].copy_(d2[o:o + part], non_blocking=True)

        def both():
            h2d()
            d2h()
        a, b, c = t(h2d), t(d2h), t(both)
        print("part %8d KB: H2D %5.1f GB/s  D2H %5.1f GB/s  both at once: %5.1f GB/s each direction"
              % (part >> 10, n / a / 1e9, n / b / 1e9, n / c / 1e9))


if __name__ == "__main__":
    main()
