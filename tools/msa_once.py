#!/usr/bin/env python
"""One dm_align_sequences call on a BASELINE MSA config (profiling target):
python tools/msa_once.py <cfg> [reps]; prints wall and tree/align split."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2601_15458_b200 as dm  # noqa: E402
from paper_2601_15458_b200._lib import check, dm_align_summary, lib  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
data, offs = dm.synth(cfg, 1.0)
n = len(offs) - 1
offs_c = np.ascontiguousarray(offs, dtype=np.uint64)
ctx = dm.default_context(0)
for r in range(reps):
    rows, width, summ, st = C.c_void_p(), C.c_uint64(), dm_align_summary(), dm.dm_stats()
    t0 = time.perf_counter()
    check(lib().dm_align_sequences(ctx.handle, data, offs_c.ctypes.data_as(C.POINTER(C.c_uint64)), n,
                                   1 if cfg != 3 else 2, -10, -1, 0, None, None, 42, 0, C.byref(rows),
                                   C.byref(width), C.byref(summ), C.byref(st)))
    wall = time.perf_counter() - t0
    lib().dm_free(rows)
    print(f"cfg{cfg}: {wall * 1e3:.1f} ms (tree {st.tree_ms:.1f}, align {st.align_ms:.1f})", flush=True)
