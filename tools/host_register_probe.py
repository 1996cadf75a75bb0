"""Probe: cudaHostRegister speed on the box (is pinning a pageable caller buffer per call affordable? no: ~12 GB/s)."""
import time, numpy as np, ctypes as C
from cuda.bindings import runtime as rt
import torch
torch.cuda.init()
for mb in (64, 256, 600):
    buf = np.ones(mb << 20, dtype=np.uint8)  # touched pageable memory
    p = buf.ctypes.data
    t = time.perf_counter()
    e = rt.cudaHostRegister(p, buf.nbytes, 0)
    t1 = time.perf_counter()
    e2 = rt.cudaHostUnregister(p)
    t2 = time.perf_counter()
    print(f"{mb} MB: register {1e3*(t1-t):.1f} ms ({mb/1024/(t1-t):.1f} GB/s) unregister {1e3*(t2-t1):.1f} ms", e, e2)
