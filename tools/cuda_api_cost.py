#!/usr/bin/env python3
"""Host cost of the CUDA runtime calls a device-resident C-ABI call makes (pointer
attributes, memset, a small D2H + synchronise), through cuda-python."""
import time, torch, ctypes
from cuda.bindings import runtime as rt
x = torch.empty(1024, device='cuda'); h = torch.empty(1024).pin_memory(); p = torch.empty(1024)
s = torch.cuda.current_stream().cuda_stream
def t(f, n=20000):
    f(); t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e6
print("ptrattr dev  %.2f us" % t(lambda: rt.cudaPointerGetAttributes(x.data_ptr())))
print("ptrattr pageable %.2f us" % t(lambda: rt.cudaPointerGetAttributes(p.data_ptr())))
print("getdevice %.2f us" % t(lambda: rt.cudaGetDevice()))
print("memsetAsync %.2f us" % t(lambda: rt.cudaMemsetAsync(x.data_ptr(), 0, 64, s)))
print("d2h 64B + sync %.2f us" % t(lambda: (rt.cudaMemcpyAsync(h.data_ptr(), x.data_ptr(), 64, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s), rt.cudaStreamSynchronize(s)), 5000))
print("sync idle %.2f us" % t(lambda: rt.cudaStreamSynchronize(s)))
print("python noop call %.2f us" % t(lambda: None))
