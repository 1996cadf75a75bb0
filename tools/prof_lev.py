#!/usr/bin/env python
"""Profiling driver: one dominant distance-engine launch.

N random DNA pairs of exactly L residues (a single (G, W) bucket), run
through dm_lev_pairs_device `reps` times. Prints kernel GCUPS so the same
command can be timed plainly and then captured under ncu."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=200000)
    ap.add_argument("--len", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--alphabet", default="ACGT")
    a = ap.parse_args()
    import torch
    import paper_2601_15458_b200 as dm
    from paper_2601_15458_b200._lib import check, lib
    rng = np.random.default_rng(1)
    alpha = np.frombuffer(a.alphabet.encode(), dtype=np.uint8)
    data = alpha[rng.integers(0, len(alpha), 2 * a.pairs * a.len)].tobytes()
    offs = np.arange(2 * a.pairs + 1, dtype=np.uint64) * a.len
    ctx = dm.default_context(0)
    ss = dm.SeqSet(data=data, offsets=offs, ctx=ctx)
    ia = torch.arange(a.pairs, dtype=torch.int32, device="cuda") * 2
    ib = ia + 1
    out = torch.empty(a.pairs, dtype=torch.int32, device="cuda")
    st = dm.dm_stats()
    for r in range(a.reps):
        check(lib().dm_lev_pairs_device(ctx.handle, ss.handle, C.c_void_p(ia.data_ptr()), C.c_void_p(ib.data_ptr()),
                                        a.pairs, C.c_void_p(out.data_ptr()), C.byref(st)))
        print(f"rep {r}: kernel {st.kernel_ms:.3f} ms, {st.cells / st.kernel_ms / 1e6:.1f} GCUPS "
              f"(executed {st.cells_executed / st.kernel_ms / 1e6:.1f}), launches {st.launches}")


if __name__ == "__main__":
    main()
