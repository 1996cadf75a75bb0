#!/usr/bin/env python
"""Host->device upload rate of a pageable caller buffer through the library
(dm.SeqSet creation on the cfg1 residues: staged copy + census/recode/planes)
against a pinned one and torch's own pageable copy."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2601_15458_b200 as dm
    data, offs = dm.synth(1, scale=float(sys.argv[1]) if len(sys.argv) > 1 else 0.25)
    n = len(data)
    ctx = dm.default_context(0)
    for label, buf in (("pageable", data), ("pinned", torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory())):
        for _ in range(2):
            dm.SeqSet(data=buf if label == "pageable" else bytes(), offsets=offs, ctx=ctx) if label == "pageable" else None
        if label == "pageable":
            t = time.perf_counter()
            for _ in range(3):
                dm.SeqSet(data=data, offsets=offs, ctx=ctx)
            dt = (time.perf_counter() - t) / 3
            print(f"SeqSet from pageable bytes: {dt * 1e3:.1f} ms for {n / 1e6:.0f} MB ({n / dt / 1e9:.1f} GB/s incl. census/recode)")
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    src = torch.frombuffer(bytearray(data), dtype=torch.uint8)
    for _ in range(2):
        dev.copy_(src)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        dev.copy_(src)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"torch pageable H2D: {n / dt / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
