#!/usr/bin/env python
"""Host memory contention check for the streamed path: 2-bit packing rate
(dm_pack_nt on all pool threads) alone, pinned H2D copy rate alone, and both
at once (does the copy engine's read of host memory slow the packers?)."""
import ctypes as C
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2601_15458_b200 as dm
    from paper_2601_15458_b200._lib import lib
    data, offs = dm.synth(1, scale=1.0)
    n = len(data)
    src = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    dst = torch.empty((n + 3) // 4, dtype=torch.uint8).pin_memory()
    raw = torch.empty(n, dtype=torch.uint8).pin_memory()
    raw.copy_(src)
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")

    def pack(reps):
        t = time.perf_counter()
        for _ in range(reps):
            lib().dm_pack_nt(C.c_char_p(src.data_ptr()), n, C.c_void_p(dst.data_ptr()))
        return n * reps / (time.perf_counter() - t) / 1e9

    def h2d(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            dev.copy_(raw, non_blocking=True)
        torch.cuda.synchronize()
        return n * reps / (time.perf_counter() - t) / 1e9

    pack(1)
    h2d(1)
    print(f"pack alone {pack(5):.1f} GB/s; pinned H2D alone {h2d(5):.1f} GB/s")
    res = {}
    th = threading.Thread(target=lambda: res.update(p=pack(5)))
    th.start()
    res["h"] = h2d(4)
    th.join()
    print(f"concurrently: pack {res['p']:.1f} GB/s, H2D {res['h']:.1f} GB/s")


if __name__ == "__main__":
    main()
