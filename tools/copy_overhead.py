"""Per-copy cost of many medium H2D / D2H copies (pinned), one way and both ways."""
import time
import torch

tot = 1 << 30
h = torch.empty(tot, dtype=torch.uint8).pin_memory()
g = torch.empty(tot, dtype=torch.uint8).pin_memory()
d = torch.empty(tot, dtype=torch.uint8, device="cuda")
e = torch.empty(tot, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(nparts, both):
    part = tot // nparts
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(nparts):
        with torch.cuda.stream(s1):
            d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        if both:
            with torch.cuda.stream(s2):
                g[i * part:(i + 1) * part].copy_(e[i * part:(i + 1) * part], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for both in (False, True):
    for nparts in (1, 16, 128, 1024):
        run(nparts, both)
        t = min(run(nparts, both) for _ in range(3))
        print("both" if both else "h2d ", nparts, "parts: %.2f GB/s per direction" % (tot / t / 1e9))
