#!/usr/bin/env python
"""Host throughput of the streamed path's 2-bit packer (dm_pack_nt) on the
cfg1 residue buffer, per host-pool size (DM_HOST_THREADS is read once per
process, so each size runs in a child process)."""
import ctypes as C
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one():
    import numpy as np
    import torch
    import paper_2601_15458_b200 as dm
    from paper_2601_15458_b200._lib import lib
    data, offs = dm.synth(1, scale=float(os.environ.get("SCALE", "1.0")))
    src = torch.frombuffer(bytearray(data), dtype=torch.uint8)
    if os.environ.get("PINNED") == "1":
        src = src.pin_memory()
    dst = torch.empty((len(data) + 3) // 4, dtype=torch.uint8)
    if torch.cuda.is_available():
        dst = dst.pin_memory()
    n = len(data)
    f = lambda: lib().dm_pack_nt(C.c_char_p(src.data_ptr()), n, C.c_void_p(dst.data_ptr()))
    assert f() == 0
    best = 1e9
    for _ in range(5):
        t = time.perf_counter()
        f()
        best = min(best, time.perf_counter() - t)
    print(f"threads {os.environ.get('DM_HOST_THREADS', 'all')}: {n / best / 1e9:.1f} GB/s residues "
          f"({best * 1e3:.1f} ms for {n / 1e9:.2f} GB)", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one()
    else:
        for t in (1, 2, 4, 8, 12, 14, 16):
            subprocess.run([sys.executable, __file__, "--one"], env=dict(os.environ, DM_HOST_THREADS=str(t)))
