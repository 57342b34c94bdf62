import torch, time
n=1<<28  # 2 GB
h1=torch.empty(n//8*8, dtype=torch.uint8).pin_memory(); h2=torch.empty_like(h1).pin_memory()
d1=torch.empty(n, dtype=torch.uint8, device='cuda'); d2=torch.empty(n, dtype=torch.uint8, device='cuda')
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
def t(f):
    torch.cuda.synchronize(); t0=time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter()-t0
for _ in range(2):
    a=t(lambda: d1.copy_(h1, non_blocking=True)); b=t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    c=t(both)
    print('H2D %.1f GB/s  D2H %.1f GB/s  both %.1f GB/s each'%(n/a/1e9, n/b/1e9, n/c/1e9))
