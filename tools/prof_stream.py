#!/usr/bin/env python
"""Streamed end-to-end path (dm_lev_pairs_packed) against the raw pinned
host->device copy bandwidth of the box; DM_TRACE=1 prints the per-chunk
host timeline of the pipeline."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--pageable", action="store_true", help="pass the Python bytes (pageable) instead of a pinned copy")
    a = ap.parse_args()
    import torch
    import paper_2601_15458_b200 as dm
    data, offs = dm.synth(1, scale=a.scale)
    nbytes = len(data)
    pinned = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        dev.copy_(pinned, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(a.reps):
        dev.copy_(pinned, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / a.reps
    print(f"pinned H2D {nbytes / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms for {nbytes / 1e9:.2f} GB)")
    del dev
    ctx = dm.default_context(0)
    src = data if a.pageable else pinned
    dm.lev_pairs_packed(src, offs, ctx)
    for _ in range(a.reps):
        t = time.perf_counter()
        _, st = dm.lev_pairs_packed(src, offs, ctx, stats=True)
        dt = time.perf_counter() - t
        print(f"packed: {dt * 1e3:.1f} ms wall, {st['total_ms']:.1f} ms stream, "
              f"{st['cells'] / dt / 1e9:.0f} GCUPS e2e")


if __name__ == "__main__":
    main()


def chunk_kernels():
    """Kernel time of one resident chunk-sized batch vs the whole batch."""
    import numpy as np
    import paper_2601_15458_b200 as dm
    data, offs = dm.synth(1, scale=1.0)
    ctx = dm.default_context(0)
    ss = dm.SeqSet(data=data, offsets=offs, ctx=ctx)
    n = (len(offs) - 1) // 2
    for k in (n, 134284, 60012):
        ia = np.arange(k, dtype=np.uint32) * 2
        dm.lev_pairs(ss, ia, ia + 1)
        _, st = dm.lev_pairs(ss, ia, ia + 1, stats=True)
        print(f"resident {k} pairs: kernels {st['kernel_ms']:.2f} ms, {st['cells'] / st['kernel_ms'] / 1e6:.0f} GCUPS")
    sub = offs[: 2 * 134284 + 1]
    sd = data[: int(sub[-1])]
    ss2 = dm.SeqSet(data=sd, offsets=sub, ctx=ctx)
    ia = np.arange(134284, dtype=np.uint32) * 2
    dm.lev_pairs(ss2, ia, ia + 1)
    _, st = dm.lev_pairs(ss2, ia, ia + 1, stats=True)
    print(f"chunk-only set 134284 pairs: kernels {st['kernel_ms']:.2f} ms")


if __name__ == "__main__" and os.environ.get("CHUNK_KERNELS"):
    chunk_kernels()
